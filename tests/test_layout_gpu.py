"""Binned layouts beyond 32768 fine bins (GPU only).

A table of 2^30 keys at C = 1 on one GPU needs 65536 fine bins of 2^14
buckets; the level-2 partition then fans out 256 ways instead of 128 and the
fine-bin histogram runs in two smem ranges.  The reference has no such size
cliff (core.py:96-101).  These cases reach that layout with few keys and a
large hash range (load factor << 1), and check the CUDA path against the
oracle without materialising V-sized host arrays: offsets through their
nonzero degrees, edges as (bucket, key) multisets, multiplicities by direct
counting (tests/oracles.py:25-29), comparisons from the degrees.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")
torch = pytest.importorskip("torch")


def check_sparse(keys, queries, v, key_bits=32):
    table = hg.build(keys, 1.0, hash_range=v, key_bits=key_bits)
    h = O.hash_keys(O.KIND_MURMUR, 0, keys, v)
    ub, cnt = np.unique(h, return_counts=True)
    off = table.offset_device.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    assert int(off[0]) == 0 and int(off[-1]) == len(keys)
    deg = off[1:] - off[:-1]
    nz = torch.nonzero(deg).flatten()
    assert np.array_equal(nz.cpu().numpy(), ub)
    assert np.array_equal(deg[nz].cpu().numpy(), cnt)
    # edges: (bucket, key) multiset
    edges = table.keys_device.cpu().numpy().view(np.uint32 if key_bits == 32 else np.uint64)
    owner = np.repeat(ub, cnt)
    got = np.lexsort((edges, owner))
    want_order = np.lexsort((keys, h))
    assert np.array_equal(edges[got], keys[want_order])
    res = hg.intersect(table, queries)
    mult = O.count_occurrences(keys, queries)
    assert np.array_equal(res.multiplicities, mult)
    hq = O.hash_keys(O.KIND_MURMUR, 0, queries, v)
    pos = np.searchsorted(ub, hq)
    pos_ok = (pos < len(ub)) & (ub[np.minimum(pos, len(ub) - 1)] == hq)
    comps = int(np.where(pos_ok, cnt[np.minimum(pos, len(ub) - 1)], 0).sum())
    assert (res.matched_positions, res.total_matches, res.comparisons) == (
        int(np.count_nonzero(mult)), int(mult.sum()), comps)


@pytest.mark.parametrize("v", [(1 << 29) + 12345, 1 << 30])
def test_more_than_32768_fine_bins(v):
    """V = 2^29 + 12345 (32769 fine bins, Lemire reduction) and V = 2^30
    (65536 fine bins, mask): 256-way level 2, split histogram."""
    keys = O.generate_keys(32, 1 << 21, 7)
    queries = np.concatenate([keys[::2], O.generate_keys(32, 1 << 20, 0x51)])
    check_sparse(keys, queries, v)


def test_more_than_32768_fine_bins_u64():
    keys = O.generate_keys(32, 1 << 20, 7, key_bits=64)
    queries = np.concatenate([keys[::2], O.generate_keys(32, 1 << 19, 0x51, key_bits=64)])
    check_sparse(keys, queries, 1 << 30, key_bits=64)
