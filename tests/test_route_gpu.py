"""hg_route (the one-pass routing of the distributed path) for P = 1..13 on one
GPU: every destination row holds exactly the reference's row as a multiset
(multishard.py:294-310 restated by the oracle), `order` maps each routed slot
back to its input key, and the peer-memory mode (P separate destination
buffers standing in for the ranks' symmetric buffers) fills the same rows."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")


@pytest.mark.parametrize("P,n,kb", [(1, 100_003, 32), (2, 300_000, 32), (3, 77_777, 32), (5, 300_000, 64),
                                    (8, 1 << 20, 32), (8, 200_001, 64), (13, 250_000, 32)])
def test_route_rows_and_order(P, n, kb):
    import torch

    from paper_2104_00792_b200.distributed import DeviceOps
    from paper_2104_00792_b200.multishard import ShardConfig

    rng = np.random.default_rng(P * 1000 + n)
    keys = O.generate_keys(32, n, P, key_bits=64) if kb == 64 else rng.integers(1, 1 << 24, size=n, dtype=np.uint64).astype(np.uint32)
    fam = hg.HashFamily()
    hr, bins_g, bin_size = ShardConfig(shards=P).resolve(n)
    kk = keys.astype(np.uint32) if kb == 32 else keys  # oracle plans on the (truncated) 32-bit view for u32
    splits = O.plan_splits(np.array_split(kk, P), hr, bins_g) if kb == 32 else None
    ops = DeviceOps(kb)
    dk = ops.to_local(keys)
    counts = ops.bin_histogram(dk, hr, bins_g, bin_size, fam)
    sp = ops.split_plan(counts, bins_g, n, P)
    if splits is not None:
        assert np.array_equal(sp.cpu().numpy(), splits)
    send = ops.segment_sums(counts, sp).cpu().numpy()
    rows = np.concatenate([[0], np.cumsum(send)])
    grouped, order = ops.route(dk, hr, bin_size, sp, P, fam, rows[:-1], want_order=True)
    g = grouped.cpu().numpy().view(np.uint32 if kb == 32 else np.uint64)
    o = order.cpu().numpy().view(np.uint32).astype(np.int64)
    assert np.array_equal(np.sort(o), np.arange(n))  # a permutation
    assert np.array_equal(g, keys[o])  # order points at the routed key
    if kb == 32:
        dest = O.dest_of_hash(O.hash_keys(0, 0, kk, hr), sp.cpu().numpy(), bin_size)
        for d in range(P):
            assert np.array_equal(np.sort(g[rows[d]:rows[d + 1]]), np.sort(kk[dest == d]))
    # peer mode: P destination buffers, this "rank" the only sender (dest_base 0)
    bufs = [ops.empty_keys(int(send[d])) for d in range(P)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    base = torch.zeros(P, dtype=torch.int64, device="cuda")
    ops.route(dk, hr, bin_size, sp, P, fam, rows[:-1], ptrs, base)
    for d in range(P):
        got = bufs[d].cpu().numpy().view(np.uint32 if kb == 32 else np.uint64)
        assert np.array_equal(np.sort(got), np.sort(g[rows[d]:rows[d + 1]]))
