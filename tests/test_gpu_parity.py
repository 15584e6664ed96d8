"""CUDA path vs the reference's golden outputs and the CPU oracle (GPU only).

Parity rules (north star): offsets exact; edges equal as per-bucket multisets
(`canonical`); multiplicities and aggregate counters exact; plans, received
counts and (stable) send buffers exact.
"""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")


def fam(kind, seed):
    return hg.HashFamily(hg.HashKind(int(kind)), int(seed))


def assert_table_equal(table, offset, placed):
    assert np.array_equal(table.offset, offset)
    a = O.canonical(table.offset, table.keys)
    b = O.canonical(offset, placed)
    assert np.array_equal(a[1], b[1])


def test_hash_array_golden():
    cases, shared = load_golden("hashing")
    probe = shared["probe"]
    for c in cases[1:]:
        got = hg.hash_array(fam(c["kind"], c["seed"]), probe, int(c["v"]))
        assert got.dtype == np.int64
        assert np.array_equal(got, c["out"].astype(np.int64)), (int(c["kind"]), int(c["seed"]), int(c["v"]))


def test_build_golden():
    cases, _ = load_golden("build")
    for c in cases:
        table, counters, positions = hg.build_traced(c["keys"], float(c["load_factor"]), fam(c["kind"], c["seed"]),
                                                     hash_range=int(c["hash_range"]))
        assert table.hash_range == int(c["hash_range"])
        assert_table_equal(table, c["offset"], c["placed"])
        n = len(c["keys"])
        assert (counters.hashed, counters.counted, counters.placed) == (n, n, n)
        assert sorted(positions.tolist()) == list(range(n))
        assert np.array_equal(table.keys, c["keys"][positions])


def test_query_golden():
    cases, _ = load_golden("query")
    for c in cases:
        table = hg.build(c["keys"], float(c["load_factor"]), fam(c["kind"], c["seed"]), hash_range=int(c["hash_range"]))
        res = hg.intersect(table, c["queries"])
        assert np.array_equal(res.multiplicities, c["multiplicities"])
        assert res.matched_positions == int(c["matched"])
        assert res.total_matches == int(c["total"])
        assert res.comparisons == int(c["comparisons"])
        assert res.hash_values == int(c["hash_values"])
        # the two-step path (build_query_table + intersect_tables) agrees
        qt, pos = hg.build_query_table(table, c["queries"])
        res2 = hg.intersect_tables(table, qt, pos)
        assert np.array_equal(res2.multiplicities, c["multiplicities"])
        assert res2.comparisons == int(c["comparisons"])


def test_sharded_golden():
    cases, _ = load_golden("sharded")
    for c in cases:
        p = int(c["p"])
        parts = [c[f"in{d}"] for d in range(p)]
        cfg = hg.ShardConfig(shards=p, load_factor=float(c["load_factor"]), bins_g=int(c["bins_in"]),
                             family=fam(c["kind"], c["seed"]), hash_range=int(c["hr_in"]))
        table, report = hg.build_sharded(parts, cfg)
        assert report.hash_range == int(c["hash_range"]) and report.bins_g == int(c["bins_g"])
        assert table.plan.bin_size == int(c["bin_size"])
        assert np.array_equal(table.plan.bin_splits, c["splits"])
        assert report.shard_received_counts == c["received"].tolist()
        assert report.search_steps == int(c["search_steps"])
        assert report.bytes_exchanged == int(c["bytes_exchanged"])
        for d in range(p):
            assert_table_equal(table.shards[d], c[f"off{d}"], c[f"keys{d}"])
            sb = hg.reorganize(parts[d], table.plan, fam(c["kind"], c["seed"]))
            assert np.array_equal(sb.offsets, c[f"send_off{d}"])
            assert np.array_equal(sb.keys, c[f"send_keys{d}"])  # stable rows: exact
        res = hg.query_sharded(table, c["queries"])
        assert np.array_equal(res.multiplicities, c["multiplicities"])
        assert (res.matched_positions, res.total_matches, res.comparisons, res.hash_values) == (
            int(c["matched"]), int(c["total"]), int(c["comparisons"]), int(c["hash_values"]))


def test_workload_golden():
    cases, _ = load_golden("workload")
    for c in cases:
        if "keys" in c:
            spec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, int(c["k"]), int(c["count"]), int(c["seed"]))
            assert np.array_equal(hg.generate(spec), c["keys"])


@pytest.mark.parametrize("n,lf,kind,seed,dom", [
    (1 << 20, 1.0, 0, 0, 1 << 24),
    (1 << 20, 0.5, 0, 12345, 1 << 20),
    (1 << 20, 4.0, 1, 0, 1 << 30),
    (3_000_001, 1.0, 0, 0xDEADBEEF, 1 << 21),
    ((1 << 20) + 17, 1.0, 0, 7, 64),  # high-duplicate
])
def test_random_vs_oracle(n, lf, kind, seed, dom):
    rng = np.random.default_rng(n + kind)
    keys = rng.integers(1, dom + 1, size=n, dtype=np.uint64).astype(np.uint32)
    queries = np.concatenate([rng.choice(keys, size=n // 3),
                              rng.integers(1, dom + 1, size=n // 3, dtype=np.uint64).astype(np.uint32)])
    f = fam(kind, seed)
    table = hg.build(keys, lf, f)
    v = table.hash_range
    off, placed, _ = O.build_csr(keys, v, kind, seed, workers=8)
    assert_table_equal(table, off, placed)
    res = hg.intersect(table, queries)
    mult, matched, total, comp, hv = O.query(off, placed, queries, kind, seed, workers=8)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons, res.hash_values) == (matched, total, comp, hv)


@pytest.mark.parametrize("p", [1, 2, 3, 8, 16])
def test_sharded_random_vs_oracle(p):
    rng = np.random.default_rng(300 + p)
    keys = rng.integers(1, 1 << 20, size=(1 << 18) + p, dtype=np.uint32)
    queries = rng.integers(1, 1 << 20, size=1 << 16, dtype=np.uint32)
    parts = np.array_split(keys, p)
    table, report = hg.build_sharded(parts, hg.ShardConfig(shards=p))
    ref = O.build_sharded(parts, p)
    assert np.array_equal(table.plan.bin_splits, ref["splits"])
    assert report.shard_received_counts == ref["received"]
    assert report.search_steps == ref["search_steps"]
    for d in range(p):
        assert_table_equal(table.shards[d], *ref["tables"][d])
    res = hg.query_sharded(table, queries)
    mult, matched, total, comp, hv = O.query_sharded(ref, queries)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.total_matches, res.comparisons, res.hash_values) == (total, comp, hv)


def test_u64_keys_vs_restatement():
    rng = np.random.default_rng(64)
    keys = rng.integers(0, 1 << 63, size=(1 << 18), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    keys[: 1 << 12] = keys[1 << 12: 1 << 13]
    queries = np.concatenate([keys[: 1 << 14], rng.integers(0, 1 << 63, size=1 << 14, dtype=np.uint64)])
    for kind, seed, v in [(0, 0, 1 << 18), (0, 99, 100_003), (1, 0, 77_777)]:
        table = hg.build(keys, 1.0, fam(kind, seed), hash_range=v, key_bits=64)
        off, placed, _ = O.build_csr(keys, v, kind, seed)
        assert_table_equal(table, off, placed)
        res = hg.intersect(table, queries)
        mult, matched, total, comp, hv = O.query(off, placed, queries, kind, seed)
        assert np.array_equal(res.multiplicities, mult)
        assert (res.matched_positions, res.total_matches, res.comparisons) == (matched, total, comp)
        got = hg.hash_array(fam(kind, seed), keys[:4096], v, key_bits=64)
        assert np.array_equal(got, O.hash_keys(kind, seed, keys[:4096], v))


def test_full_size_properties():
    """At the C1 size (2^24 keys, 2^24 queries): size-independent invariants."""
    import torch

    spec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 24, 1 << 24, 0)
    qspec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 24, 1 << 24, 0x51)
    keys = hg.generate_device(spec)
    queries = hg.generate_device(qspec)
    table = hg.build(keys)
    off = table.offset
    assert off[0] == 0 and off[-1] == 1 << 24 and np.all(np.diff(off) >= 0)
    # edges hold the input multiset: compare sorted device arrays
    assert torch.equal(torch.sort(table.keys_device)[0], torch.sort(keys)[0])
    # every edge sits in the bucket its key hashes to
    h = hg.hash_array(table.family, table.keys_device, table.hash_range)
    owner = torch.repeat_interleave(torch.arange(table.hash_range, device=h.device),
                                    torch.from_numpy(np.diff(off)).to(h.device))
    assert torch.equal(h, owner)
    res = hg.intersect(table, queries)
    # SURVEY §8(d) measured 10,601,263 of 2^24 C1 queries hit
    assert res.matched_positions == 10_601_263
    self_res = hg.intersect(table, keys)
    assert self_res.matched_positions == 1 << 24
    _, counts = torch.unique(keys, return_counts=True)
    assert self_res.total_matches == int((counts.to(torch.int64) ** 2).sum())


@pytest.mark.parametrize("n,dom,lf", [((1 << 20) + 3, 1 << 22, 1.0), (1 << 21, 1 << 12, 1.0), (1 << 20, 1 << 30, 0.5),
                                      (1 << 20, 1 << 20, 4.0), (1 << 20, 1 << 20, 16.0)])
def test_binned_and_direct_paths_agree(monkeypatch, n, dom, lf):
    """The v2 binned kernels (default for >= 2^16 keys) and the direct Alg. 1
    kernels (HG_FORCE_DIRECT) produce identical offsets and bucket multisets."""
    rng = np.random.default_rng(n ^ dom)
    keys = rng.integers(1, dom + 1, size=n, dtype=np.uint64).astype(np.uint32)
    queries = rng.integers(1, dom + 1, size=n // 2, dtype=np.uint64).astype(np.uint32)
    t_binned = hg.build(keys, lf)
    r_binned = hg.intersect(t_binned, queries)
    monkeypatch.setenv("HG_FORCE_DIRECT", "1")
    t_direct = hg.build(keys, lf)
    r_direct = hg.intersect(t_direct, queries)
    monkeypatch.delenv("HG_FORCE_DIRECT")
    assert_table_equal(t_binned, t_direct.offset, t_direct.keys)
    assert np.array_equal(r_binned.multiplicities, r_direct.multiplicities)
    assert (r_binned.matched_positions, r_binned.total_matches, r_binned.comparisons) == (
        r_direct.matched_positions, r_direct.total_matches, r_direct.comparisons)
    # and both match the oracle
    mult = O.count_occurrences(keys, queries)
    assert np.array_equal(r_binned.multiplicities, mult)


def test_all_identical_keys_large():
    """Every key in one bucket: the oversized-bin path (global counters)."""
    n = 1 << 20
    keys = np.full(n, 123456, dtype=np.uint32)
    table = hg.build(keys)
    deg = np.diff(table.offset)
    assert deg.max() == n and deg.sum() == n
    assert table.contains(123456) == n
    res = hg.intersect(table, np.array([123456, 5, 123456], dtype=np.uint32))
    assert res.multiplicities.tolist() == [n, 0, n]


@pytest.mark.parametrize("n,values,lf", [(1 << 20, 1 << 8, 1.0), (1 << 22, 1 << 12, 1.0), ((1 << 20) + 5, 3, 2.0),
                                         (1 << 22, 1 << 17, 1.0)])  # last: > 256 deep keys per bin (map overflow)
def test_high_duplicate_build_and_query(n, values, lf):
    """C3-shaped inputs (many copies of few values): deep buckets go through the
    probe's per-bin map and oversized fine bins through the global build."""
    rng = np.random.default_rng(values)
    domain = rng.integers(0, 1 << 32, size=values, dtype=np.uint64).astype(np.uint32)
    keys = domain[rng.integers(0, values, size=n)]
    queries = np.concatenate([domain[rng.integers(0, values, size=n // 2)],
                              rng.integers(0, 1 << 32, size=n // 8, dtype=np.uint64).astype(np.uint32)])
    table = hg.build(keys, lf)
    off, placed, _ = O.build_csr(keys, table.hash_range)
    assert_table_equal(table, off, placed)
    res = hg.intersect(table, queries)
    assert np.array_equal(res.multiplicities, O.count_occurrences(keys, queries))
    _, matched, total, comp, _ = O.query(off, placed, queries)
    assert (res.matched_positions, res.total_matches, res.comparisons) == (matched, total, comp)


def test_c1_exact_vs_oracle():
    """BASELINE C1 at full size (2^24 uint32 keys and 2^24 queries from the
    reference's SplitMix64 streams, C = 1), bit-exact against the CPU
    restatement: offsets equal, every bucket the same multiset, every
    multiplicity and aggregate counter equal."""
    spec = hg.WorkloadSpec(hg.WorkloadKind.RANDOM_WITH_REPLACEMENT, 24, 1 << 24, 0)
    keys = O.generate_keys(24, 1 << 24, 0)
    queries = O.generate_keys(24, 1 << 24, 0x51)
    assert np.array_equal(hg.generate(spec), keys)
    table = hg.build(keys)
    off, placed, _ = O.build_csr(keys, table.hash_range)
    assert_table_equal(table, off, placed)
    res = hg.intersect(table, queries)
    mult, matched, total, comp, _ = O.query(off, placed, queries)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons) == (matched, total, comp)
    assert matched == 10_601_263  # SURVEY §8(d), measured with the reference


@pytest.mark.parametrize("v", [(1 << 32) - 1, (1 << 31) + 1, (1 << 31) + 12345, 3, 5, 641, (1 << 20) * 3 + 1])
@pytest.mark.parametrize("kind", [0, 1])
def test_hash_mod_extreme_ranges(v, kind):
    """hash mod V for non-power-of-two V through the invariant-multiplier
    reduction (hg_common.cuh mod_gm32): the largest 32-bit V, V just above 2^31
    (the second shift at its maximum), tiny V; the inputs include the ends of
    the 32-bit range (identity hash: the reduced value is the key itself)."""
    rng = np.random.default_rng(v % 1000003 + kind)
    keys = np.concatenate([rng.integers(0, 1 << 32, size=(1 << 20) - 6, dtype=np.uint64),
                           np.array([0, 1, v - 1, v % (1 << 32), 0xFFFFFFFE, 0xFFFFFFFF], dtype=np.uint64)]
                          ).astype(np.uint32)
    got = hg.hash_array(fam(kind, 99), keys, v)
    assert np.array_equal(got, O.hash_keys(kind, 99, keys, v).astype(np.int64))


@pytest.mark.parametrize("v,kind", [((1 << 20) * 3, 0), ((1 << 20) + 1, 1), ((1 << 21) - 1, 0), (12345, 1)])
def test_non_power_of_two_ranges_vs_oracle(v, kind):
    """Binned and direct builds and queries at non-power-of-two ranges."""
    n = 1 << 20
    rng = np.random.default_rng(v)
    keys = np.concatenate([rng.integers(0, 1 << 32, size=n - 4, dtype=np.uint64),
                           np.array([0, 1, 0xFFFFFFFE, 0xFFFFFFFF], dtype=np.uint64)]).astype(np.uint32)
    queries = np.concatenate([keys[::5], rng.integers(0, 1 << 32, size=n // 5, dtype=np.uint64).astype(np.uint32)])
    f = fam(kind, 99)
    table = hg.build(keys, 1.0, f, hash_range=v)
    off, placed, _ = O.build_csr(keys, v, kind, 99, workers=8)
    assert_table_equal(table, off, placed)
    res = hg.intersect(table, queries)
    mult, matched, total, comp, hv = O.query(off, placed, queries, kind, 99, workers=8)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons) == (matched, total, comp)
