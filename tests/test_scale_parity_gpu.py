"""Parity at the configurations the bench measures (GPU only).

Each case runs the product path at full size and compares it with the CPU
oracle on the same inputs:

* offsets: exact, over every bucket (oracle: bincount of the reference hash,
  hashing.py:98-114 / core.py:96-99);
* edges, every bucket: two per-bucket signatures of the key multiset (the sum
  of the keys and the sum of fmix32 of the keys, float64 sums that are exact
  below 2^53), oracle vs device layout;
* edges, sampled: `canonical` (test_acceptance.py:44-51) exactly equal on 64
  randomly chosen 2^14-bucket windows (the fine-bin size of the bench layout);
* multiplicities: every query exact against an unhashed count of the input
  (tests/oracles.py:25-29 restated: a direct-address count for k <= 28, sorted
  unique counts for 64-bit keys);
* matched / total / comparisons: exact (comparisons = sum_h deg_a(h) deg_q(h),
  query.py:153-155).

Sizes: 2^28 uint32 keys and queries at C = 1 (F = 16,384 fine bins, 128
level-1 bins: the bench layout), the same at C = 4, the high-duplicate C3
stream (2^28 keys from 2^16 values), and 2^26 uint64 keys (two-level u64
partition, local build, probe and unpartition).
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")

# bench.py's default workload (C5 at P=1, C=1): the oracle's answer, also
# committed in bench.py as the step's checksum.
BENCH_EXPECTED = {"matched": 169_672_492, "total": 268_422_361, "comparisons": 517_428_761}


def _fmix32_u64(keys):
    x = (keys.astype(np.uint64) ^ (keys.astype(np.uint64) >> np.uint64(32))).astype(np.uint32)
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x85EBCA6B)
    x ^= x >> np.uint32(13)
    x *= np.uint32(0xC2B2AE35)
    x ^= x >> np.uint32(16)
    return x


def _weights(keys):
    """Per-key weights of the bucket signatures: low word, high word (64-bit
    keys), fmix32 of the folded key -- as float64 (per-bucket sums stay exact)."""
    k64 = keys.astype(np.uint64)
    yield (k64 & np.uint64(0xFFFFFFFF)).astype(np.float64)
    if keys.dtype == np.uint64:
        yield (k64 >> np.uint64(32)).astype(np.float64)
    yield _fmix32_u64(keys).astype(np.float64)


def _multiplicities(keys, queries, k):
    if keys.dtype == np.uint32 and k <= 28:
        cnt = np.bincount(keys, minlength=(1 << k) + 1)
        return cnt[np.minimum(queries, np.uint32(1 << k))] * (queries <= (1 << k))
    u, c = np.unique(keys, return_counts=True)
    i = np.searchsorted(u, queries)
    i = np.minimum(i, len(u) - 1)
    return np.where(u[i] == queries, c[i], 0)


def check_scale(keys, queries, lf, k, key_bits, seed_windows=0):
    """Build + query on the GPU, then every check listed in the module doc."""
    import torch

    kb = key_bits
    n = len(keys)
    kd = torch.from_numpy(keys.view(np.int32 if kb == 32 else np.int64)).cuda()
    qd = torch.from_numpy(queries.view(np.int32 if kb == 32 else np.int64)).cuda()
    table = hg.build(kd, lf, key_bits=kb)
    res = hg.intersect(table, qd)
    v = table.hash_range
    assert v == O.hash_range_for(n, lf)
    off_dev = table.offset_device.cpu().numpy().view(np.uint32).astype(np.int64)
    edges = table.keys_device.cpu().numpy().view(keys.dtype)
    mult_dev = res.multiplicities_device.cpu().numpy().view(np.uint32).astype(np.int64)
    del kd, qd, table
    torch.cuda.empty_cache()

    # offsets, every bucket
    h = O.hash_keys(O.KIND_MURMUR, 0, keys, v)
    deg = np.bincount(h, minlength=v)
    assert off_dev[0] == 0 and off_dev[-1] == n
    assert np.array_equal(np.diff(off_dev), deg), "offsets differ from the oracle"
    # bucket multisets, every bucket (signatures)
    owner = np.repeat(np.arange(v, dtype=np.int64), deg)
    for wa, wb in zip(_weights(edges), _weights(keys)):
        a = np.bincount(owner, weights=wa, minlength=v)
        b = np.bincount(h, weights=wb, minlength=v)
        assert np.array_equal(a, b), "a bucket's key multiset differs from the oracle"
        del a, b
    del owner
    # bucket multisets, sampled windows: canonical equality
    rng = np.random.default_rng(seed_windows)
    win = 1 << 14
    nwin = max(1, -(-v // win))
    chosen = np.unique(rng.integers(0, nwin, size=min(64, nwin)))
    pick = np.zeros(nwin, dtype=bool)
    pick[chosen] = True
    sel = pick[h >> 14]
    ho, ko = h[sel], keys[sel]
    o = np.lexsort((ko, ho))
    ho, ko = ho[o], ko[o]
    for w in chosen:
        b0, b1 = int(w) * win, min(v, (int(w) + 1) * win)
        lo, hi = off_dev[b0], off_dev[b1]
        got_owner = np.repeat(np.arange(b0, b1, dtype=np.int64), np.diff(off_dev[b0:b1 + 1]))
        got = edges[lo:hi]
        g = np.lexsort((got, got_owner))
        a0, a1 = np.searchsorted(ho, b0), np.searchsorted(ho, b1)
        assert np.array_equal(got[g], ko[a0:a1]), f"window {w}: canonical bucket contents differ"
    del sel, ho, ko
    # multiplicities and aggregates
    mult = _multiplicities(keys, queries, k)
    assert np.array_equal(mult_dev, mult), "multiplicities differ from the oracle"
    hq = O.hash_keys(O.KIND_MURMUR, 0, queries, v)
    comps = int(np.dot(deg.astype(np.int64), np.bincount(hq, minlength=v).astype(np.int64)))
    agg = (int(np.count_nonzero(mult)), int(mult.sum(dtype=np.int64)), comps)
    assert (res.matched_positions, res.total_matches, res.comparisons) == agg
    return agg


def test_bench_workload_c1_u32_2p28():
    """bench.py's step: 2^28 keys from {1..2^28} (seed 0), 2^28 queries (seed
    0x51), C = 1 -- F = 16,384 fine bins, 128 level-1 bins, 296-CTA chunks."""
    keys = O.generate_keys(28, 1 << 28, 0)
    queries = O.generate_keys(28, 1 << 28, 0x51)
    spec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 28, 1 << 28, 0)
    dev = hg.generate_device(spec, 0, 1 << 28)
    assert np.array_equal(dev[::4099].cpu().numpy().view(np.uint32), keys[::4099])  # the bench's device stream
    del dev
    agg = check_scale(keys, queries, 1.0, 28, 32, seed_windows=1)
    assert agg == (BENCH_EXPECTED["matched"], BENCH_EXPECTED["total"], BENCH_EXPECTED["comparisons"])
    import bench

    assert bench.EXPECTED[(28, 28, 1.0, 32)] == BENCH_EXPECTED


def test_c4_load_factor_u32_2p28():
    """C = 4 (V = 2^26, ~4 keys per bucket) at the bench size."""
    keys = O.generate_keys(28, 1 << 28, 0)
    queries = O.generate_keys(28, 1 << 28, 0x51)
    check_scale(keys, queries, 4.0, 28, 32, seed_windows=2)


def test_c3_high_duplicate_u32_2p28():
    """BASELINE C3: 2^28 keys drawn from 2^16 values (~4096 copies each),
    queries from the same domain (oversized fine bins + deep-bucket probe)."""
    keys = O.generate_keys(16, 1 << 28, 0)
    queries = O.generate_keys(16, 1 << 28, 0x51)
    check_scale(keys, queries, 1.0, 16, 32, seed_windows=3)


def test_u64_two_level_2p26():
    """64-bit keys at 2^26 (full SplitMix64 words): F = 8,192 fine bins, so
    the u64 two-level partition, local build, probe and unpartition all run.
    Half the queries are table keys (hits), half fresh words (misses)."""
    n = 1 << 26
    keys = O.generate_keys(64, n, 0, key_bits=64)
    rng = np.random.default_rng(7)
    queries = np.concatenate([keys[rng.integers(0, n, size=n // 2)], O.generate_keys(64, n // 2, 0x51, key_bits=64)])
    rng.shuffle(queries)
    check_scale(keys, queries, 1.0, 64, 64, seed_windows=4)
