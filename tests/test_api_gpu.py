"""The reference test suite's behaviours, exercised through the drop-in API on
the GPU (restated from pkg/tests/test_core.py, test_query.py and
test_multishard.py of the reference: hand examples, edge cases, errors,
immutability, worker-count independence, plan invariants)."""

from collections import Counter

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")
IDENT = hg.HashFamily.identity()
MURMUR = hg.HashFamily.murmur32()


def bucket_map(keys, family, v):
    out = {}
    for k in keys:
        out.setdefault(hg.hash_key(family, int(k), v), Counter())[int(k) & 0xFFFFFFFF] += 1
    return out


# ---------------------------------------------------------------- core (test_core.py)

def test_hand_example_identity():
    t = hg.build([0, 2, 2, 5], 1.0, IDENT)
    assert t.hash_range == 4
    assert t.offset.tolist() == [0, 1, 2, 4, 4]
    assert t.bucket(0).entries.tolist() == [0]
    assert t.bucket(1).entries.tolist() == [5]
    assert sorted(t.bucket(2).entries.tolist()) == [2, 2]
    assert t.bucket(3).entries.tolist() == []


def test_empty_and_single():
    t = hg.build([], 1.0, MURMUR)
    assert t.hash_range == 1 and t.offset.tolist() == [0, 0] and len(t.keys) == 0
    t = hg.build([42], 1.0, IDENT)
    assert t.offset.tolist() == [0, 1] and t.keys.tolist() == [42]


@pytest.mark.parametrize("n", [0, 1, 2, 1000, 1 << 20])
@pytest.mark.parametrize("lf", [0.5, 1.0, 2.0])
@pytest.mark.parametrize("family", [IDENT, MURMUR])
def test_csr_well_formed(n, lf, family):
    rng = np.random.default_rng(n + int(lf * 10))
    keys = rng.integers(0, 1 << 24, size=n, dtype=np.uint32)
    t = hg.build(keys, lf, family)
    assert t.hash_range == max(1, int(np.ceil(n / lf)))
    off = t.offset
    assert off[0] == 0 and off[-1] == n and np.all(np.diff(off) >= 0)
    if n:
        owner = np.repeat(np.arange(t.hash_range), np.diff(off))
        assert np.array_equal(hg.hash_array(family, t.keys, t.hash_range), owner)
        assert np.array_equal(np.sort(t.keys), np.sort(keys))


@pytest.mark.parametrize("family", [IDENT, MURMUR])
def test_buckets_match_bruteforce(family):
    rng = np.random.default_rng(23)
    keys = rng.integers(0, 5000, size=4000, dtype=np.uint32)
    t = hg.build(keys, 1.0, family)
    ref = bucket_map(keys, family, t.hash_range)
    for h in range(t.hash_range):
        assert Counter(t.bucket(h).entries.tolist()) == ref.get(h, Counter())


def test_worker_count_accepted_and_independent():
    rng = np.random.default_rng(37)
    keys = rng.integers(0, 1 << 16, size=1 << 15, dtype=np.uint32)
    base = hg.build(keys, 1.0, MURMUR, worker_count=1)
    for w in (2, 8):
        other = hg.build(keys, 1.0, MURMUR, worker_count=w)
        assert np.array_equal(base.offset, other.offset)
        assert np.array_equal(O.canonical(base.offset, base.keys)[1], O.canonical(other.offset, other.keys)[1])


def test_all_duplicates_single_bucket():
    keys = np.full(100_000, 123456, dtype=np.uint32)
    t = hg.build(keys, 1.0, MURMUR)
    deg = np.diff(t.offset)
    assert deg.max() == 100_000 and deg.sum() == 100_000
    assert t.contains(123456) == 100_000


def test_positions_permutation():
    rng = np.random.default_rng(43)
    keys = rng.integers(0, 100, size=500, dtype=np.uint32)
    t, counters, pos = hg.build_traced(keys, 1.0, MURMUR, worker_count=4)
    assert sorted(pos.tolist()) == list(range(500))
    assert np.array_equal(t.keys, keys[pos])
    assert (counters.hashed, counters.counted, counters.placed, counters.total) == (500, 500, 500, 1500)


def test_bucket_index_errors_contains_and_immutability():
    t = hg.build([0, 2, 2, 5], 1.0, IDENT)
    with pytest.raises(IndexError):
        t.bucket(4)
    with pytest.raises(IndexError):
        t.bucket(-1)
    assert t.contains(2) == 2 and t.contains(9) == 0
    assert hg.build([], 1.0, IDENT).contains(0) == 0
    with pytest.raises(ValueError):
        t.keys[0] = 9
    with pytest.raises(ValueError):
        t.offset[0] = 9
    with pytest.raises(AttributeError):
        t.hash_range = 3


def test_build_rejects_bad_config():
    for kwargs in (dict(load_factor=0.0), dict(load_factor=-2.0), dict(worker_count=0), dict(hash_range=0)):
        with pytest.raises(hg.ConfigError):
            hg.build([1], **{"family": MURMUR, **kwargs})
    with pytest.raises(hg.ConfigError):
        hg.build(np.zeros((2, 2), np.uint32))


def test_explicit_hash_range_and_uint64_truncation():
    t = hg.build([1, 2, 3, 4], 1.0, IDENT, hash_range=2)
    assert sorted(t.bucket(0).entries.tolist()) == [2, 4] and sorted(t.bucket(1).entries.tolist()) == [1, 3]
    # like the reference, 64-bit input is coerced to uint32 (core.py:84-88)
    t = hg.build(np.array([1, (1 << 32) + 1, (1 << 40) + 7], dtype=np.uint64), 1.0, IDENT)
    assert sorted(t.keys.tolist()) == [1, 1, 7]


# ---------------------------------------------------------------- query (test_query.py)

def test_query_hand_example_and_empties():
    t = hg.build([0, 2, 2, 5], 1.0, IDENT)
    r = hg.intersect(t, [2, 7, 0])
    assert r.multiplicities.tolist() == [2, 0, 1] and r.matched_positions == 2 and r.total_matches == 3
    r = hg.intersect(hg.build([1, 2, 3], 1.0, MURMUR), [])
    assert len(r.multiplicities) == 0 and r.matched_positions == 0 and r.total_matches == 0
    r = hg.intersect(hg.build([], 1.0, MURMUR), [1, 2, 3])
    assert r.multiplicities.tolist() == [0, 0, 0] and r.comparisons == 0


@pytest.mark.parametrize("family", [IDENT, MURMUR])
@pytest.mark.parametrize("lf", [0.5, 1.0, 2.0])
def test_zero_iff_absent(family, lf):
    rng = np.random.default_rng(59)
    keys = rng.integers(0, 300, size=500, dtype=np.uint32)
    qs = rng.integers(0, 600, size=400, dtype=np.uint32)
    r = hg.intersect(hg.build(keys, lf, family), qs)
    present = set(keys.tolist())
    assert [(m == 0) for m in r.multiplicities.tolist()] == [q not in present for q in qs.tolist()]


def test_symmetry_and_duplicates():
    rng = np.random.default_rng(67)
    a = rng.integers(0, 2000, size=3000, dtype=np.uint32)
    b = rng.integers(0, 2000, size=1700, dtype=np.uint32)
    assert hg.intersect(hg.build(a), b).total_matches == hg.intersect(hg.build(b), a).total_matches
    r = hg.intersect(hg.build([7, 7, 7], 1.0, MURMUR), [7, 7])
    assert r.multiplicities.tolist() == [3, 3] and r.total_matches == 6


def test_intersect_buckets_and_composition():
    ta = hg.build([2, 2], 1.0, IDENT, hash_range=1)
    tb = hg.build([2], 1.0, IDENT, hash_range=1)
    r = hg.intersect_buckets(ta.bucket(0), tb.bucket(0))
    assert r.counts.tolist() == [2] and r.total_matches == 2 and r.comparisons == 2
    t = hg.build([1, 2, 3, 4], 1.0, IDENT)
    with pytest.raises(hg.ConfigError):
        hg.intersect_buckets(t.bucket(0), t.bucket(1))
    rng = np.random.default_rng(71)
    keys = rng.integers(0, 500, size=2000, dtype=np.uint32)
    qs = rng.integers(0, 500, size=1500, dtype=np.uint32)
    table = hg.build(keys, 1.0, MURMUR)
    qt = hg.build(qs, 1.0, MURMUR, hash_range=table.hash_range)
    res = hg.intersect(table, qs)
    matches = comps = 0
    for h in range(table.hash_range):
        rb = hg.intersect_buckets(table.bucket(h), qt.bucket(h))
        matches += rb.total_matches
        comps += rb.comparisons
    assert (res.total_matches, res.comparisons) == (matches, comps)


def test_intersect_tables_validation_and_timed():
    t1 = hg.build([1, 2, 3], 1.0, MURMUR)
    qt = hg.build([1, 2], 1.0, MURMUR, hash_range=7)
    with pytest.raises(hg.ConfigError):
        hg.intersect_tables(t1, qt, np.arange(2))
    qt = hg.build([1, 2], 1.0, hg.HashFamily.murmur32(5), hash_range=t1.hash_range)
    with pytest.raises(hg.ConfigError):
        hg.intersect_tables(t1, qt, np.arange(2))
    keys = np.arange(1, 1 << 12, dtype=np.uint32)
    res, times = hg.intersect_timed(hg.build(keys), keys)
    assert res.matched_positions == len(keys)
    assert times.table_build_ns >= 0 and times.intersect_ns >= 0
    assert times.total_ns == times.table_build_ns + times.intersect_ns


def test_comparisons_quadratic_in_duplicate_rate():
    n = 1 << 16
    per = {}
    for d in (8, 16, 32):
        rng = np.random.default_rng(79)
        keys = rng.integers(1, n + 1, size=n, dtype=np.uint32)
        qs = rng.integers(1, n + 1, size=n, dtype=np.uint32)
        r = hg.intersect(hg.build(keys, 1.0, MURMUR, hash_range=n // d), qs)
        per[d] = r.comparisons / r.hash_values
    for d in (8, 16):
        assert 3.0 <= per[2 * d] / per[d] <= 5.0


# ---------------------------------------------------------------- multishard (test_multishard.py)

def test_plan_examples_and_invariance():
    plan = hg.plan_partition([[0, 1], [2, 3]], hash_range=4, bins_g=4, family=IDENT)
    assert plan.bin_size == 1 and plan.bin_splits.tolist() == [0, 2, 4]
    assert plan.shard_of(np.array([0, 1, 2, 3])).tolist() == [0, 0, 1, 1]
    plan = hg.plan_partition([[5, 6, 7]], hash_range=100, bins_g=10, family=IDENT)
    assert plan.bin_splits.tolist() == [0, 10]
    rng = np.random.default_rng(97)
    keys = rng.integers(0, 1 << 16, size=20_000, dtype=np.uint32)
    a = hg.plan_partition(np.array_split(keys, 4), 1 << 16, 256, MURMUR)
    sh = keys.copy()
    rng.shuffle(sh)
    b = hg.plan_partition(np.array_split(sh, 4), 1 << 16, 256, MURMUR)
    c = hg.plan_partition([sh, [], [], []], 1 << 16, 256, MURMUR)
    assert np.array_equal(a.bin_splits, b.bin_splits) and np.array_equal(a.bin_splits, c.bin_splits)


def test_plan_balance_uniform_keys():
    rng = np.random.default_rng(89)
    keys = rng.integers(1, 1 << 20, size=1 << 20, dtype=np.uint32)
    hr = 1 << 20
    plan = hg.plan_partition(np.array_split(keys, 8), hash_range=hr, bins_g=round(hr ** 0.5), family=MURMUR)
    counts = np.bincount(plan.shard_of(hg.hash_array(MURMUR, keys, hr)), minlength=8)
    assert np.all(np.abs(counts - len(keys) / 8) <= 0.05 * len(keys) / 8)


def test_plan_rejects_bad_config():
    for args in (([[1], [2]], 4, 1), ([[1], [2]], 0, 4), ([], 4, 4)):
        with pytest.raises(hg.ConfigError):
            hg.plan_partition(args[0], hash_range=args[1], bins_g=args[2], family=IDENT)


def test_reorganize_and_exchange():
    plan = hg.plan_partition([[0, 1], [2, 3]], hash_range=4, bins_g=4, family=IDENT)
    sb = hg.reorganize([0, 1, 2, 3], plan, IDENT)
    assert sorted(sb.row(0).tolist()) == [0, 1] and sorted(sb.row(1).tolist()) == [2, 3]
    empty = hg.reorganize([], plan, IDENT)
    assert empty.row(0).tolist() == [] and empty.row(1).tolist() == []
    allone = hg.reorganize([3, 3, 3, 3], plan, IDENT)
    assert allone.row(0).tolist() == [] and allone.row(1).tolist() == [3, 3, 3, 3]
    a, b, c, d = (np.array([v], dtype=np.uint32) for v in (10, 11, 12, 13))
    s0 = hg.SendBuffers(np.array([0, 1, 2]), np.concatenate([a, b]))
    s1 = hg.SendBuffers(np.array([0, 1, 2]), np.concatenate([c, d]))
    fabric = hg.ExchangeFabric(2)
    received = hg.exchange(fabric, [s0, s1])
    assert received[0].tolist() == [10, 12] and received[1].tolist() == [11, 13]
    assert fabric.keys_moved == 4 and fabric.bytes_moved == 16
    with pytest.raises(hg.ConfigError):
        hg.SendBuffers(np.array([0, 3]), np.array([1], dtype=np.uint32))


def test_build_sharded_cases_and_report():
    cfg = hg.ShardConfig(shards=2, family=IDENT, hash_range=4, bins_g=4)
    table, report = hg.build_sharded([[0, 1], [2, 3]], cfg)
    assert sorted(table.shards[0].keys.tolist()) == [0, 1] and sorted(table.shards[1].keys.tolist()) == [2, 3]
    assert report.total_keys == 4 and report.shard_received_counts == [2, 2]
    assert hg.query_sharded(table, [3, 9]).multiplicities.tolist() == [1, 0]
    table, report = hg.build_sharded([[], []], hg.ShardConfig(shards=2))
    assert report.total_keys == 0 and report.build_throughput == 0.0
    assert hg.query_sharded(table, [1, 2, 3]).multiplicities.tolist() == [0, 0, 0]
    rng = np.random.default_rng(139)
    keys = rng.integers(0, 1 << 12, size=1 << 12, dtype=np.uint32)
    _, report = hg.build_sharded(list(np.array_split(keys, 2)), hg.ShardConfig(shards=2))
    assert set(report.phases) == {"partition", "preprocess", "all_to_all", "table_construction"}
    assert sum(st.time_ns for st in report.phases.values()) <= report.total_time_ns
    assert report.bytes_exchanged == 4 * report.total_keys and report.build_throughput > 0
    d = report.to_json_dict()
    assert d["schema"] == "phase-report-v1" and set(d["passes"]) == set(report.passes)
    assert hg.work_audit(report, len(keys), 2).ok
    assert not hg.work_audit(report, 10, 2).ok
    with pytest.raises(hg.ConfigError):
        hg.build_sharded([[1], [2]], hg.ShardConfig(shards=2, bins_g=1))
    with pytest.raises(hg.ConfigError):
        hg.build_sharded([[1]], hg.ShardConfig(shards=2))


@pytest.mark.parametrize("shards", [1, 2, 4, 8, 16])
def test_query_sharded_matches_oracle(shards):
    rng = np.random.default_rng(127 + shards)
    keys = rng.integers(0, 1 << 15, size=1 << 15, dtype=np.uint32)
    qs = rng.integers(0, 1 << 15, size=1 << 14, dtype=np.uint32)
    table, _ = hg.build_sharded(list(np.array_split(keys, shards)), hg.ShardConfig(shards=shards, family=MURMUR))
    assert np.array_equal(hg.query_sharded(table, qs).multiplicities, O.count_occurrences(keys, qs))
    one = hg.query_sharded(table, qs, worker_count=1)
    res, times = hg.query_sharded_timed(table, qs, worker_count=8)
    assert np.array_equal(one.multiplicities, res.multiplicities) and one.comparisons == res.comparisons
    assert times.total_ns >= 0


def test_query_sharded_large_case():
    rng = np.random.default_rng(149)
    keys = rng.integers(1, 1 << 22, size=1 << 22, dtype=np.uint32)
    qs = rng.integers(1, 1 << 22, size=1 << 18, dtype=np.uint32)
    table, report = hg.build_sharded(list(np.array_split(keys, 16)), hg.ShardConfig(shards=16, family=MURMUR))
    assert sum(report.shard_received_counts) == len(keys)
    assert np.array_equal(hg.query_sharded(table, qs).multiplicities, O.count_occurrences(keys, qs))


def test_cuda_tensor_inputs_stay_on_device():
    import torch

    keys = torch.arange(1, 1 << 18, device="cuda", dtype=torch.int32)
    t = hg.build(keys)
    assert t.keys_device.is_cuda and t.offset_device.is_cuda
    r = hg.intersect(t, keys)
    assert r.multiplicities_device.is_cuda and r.matched_positions == keys.numel()
    h = hg.hash_array(MURMUR, keys, 1000)
    assert h.is_cuda and h.dtype == torch.int64


@pytest.mark.parametrize("lf", [1.0, 2.0, 4.0, 8.0])
def test_query_takes_binned_path_at_every_load_factor(lf):
    """The query workspace is sized for any table density, so denser tables
    (C > 1, BASELINE's C5 sweep) still run the binned query -- not the direct
    Alg. 1 fallback -- and give the oracle's answers."""
    from paper_2104_00792_b200 import _lib

    rng = np.random.default_rng(int(lf * 10))
    n = 1 << 20
    keys = rng.integers(1, 1 << 21, size=n, dtype=np.uint64).astype(np.uint32)
    queries = rng.integers(1, 1 << 21, size=n, dtype=np.uint64).astype(np.uint32)
    table = hg.build(keys, lf)
    _lib.timing_enable(True)
    _lib.timing_collect()
    res = hg.intersect(table, queries)
    names = {name for name, _ in _lib.timing_collect()}
    _lib.timing_enable(False)
    assert "hg_local_probe" in names and "hg_place_pos" not in names, names
    assert np.array_equal(res.multiplicities, O.count_occurrences(keys, queries))
