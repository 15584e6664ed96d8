"""Pin the CPU oracle against outputs of the reference itself (CPU only).

The fixtures in tests/golden were produced by running the unmodified reference
(tests/golden/make_golden.py); the known-answer values below are the
reference test suite's own (test_hashing.py:22-36, test_core.py:23-31,
test_query.py:22-27, test_multishard.py:27-32, test_workload.py:24-43).
"""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

FMIX_KAT = {
    0x00000000: 0x00000000,
    0x00000001: 0x514E28B7,
    0x00000002: 0x30F4C306,
    0x00000007: 0x18C9AEC4,
    0x0000002A: 0x087FCD5C,
    0xDEADBEEF: 0x0DE5C6A9,
    0xFFFFFFFF: 0x81F16F39,
}


def test_fmix32_known_answers():
    for k, v in FMIX_KAT.items():
        assert O.fmix32_scalar(k) == v
        assert O.hash_scalar(O.KIND_MURMUR, 0, k, 1 << 32) == v
        assert int(O.hash_keys(O.KIND_MURMUR, 0, np.array([k], np.uint32), 1 << 32)[0]) == v


def test_hash_matches_reference_golden():
    cases, shared = load_golden("hashing")
    probe = shared["probe"]
    raw = cases[0]
    assert [O.fmix32_scalar(int(k)) for k in raw["keys"]] == raw["out"].tolist()
    for c in cases[1:]:
        got = O.hash_keys(int(c["kind"]), int(c["seed"]), probe, int(c["v"]))
        assert np.array_equal(got, c["out"].astype(np.int64)), (int(c["kind"]), int(c["seed"]), int(c["v"]))
        # the scalar form agrees on a prefix
        for k, h in zip(probe[:50], c["out"][:50]):
            assert O.hash_scalar(int(c["kind"]), int(c["seed"]), int(k), int(c["v"])) == int(h)


def test_hash_range_for_examples():
    assert O.hash_range_for(0, 1.0) == 1
    assert O.hash_range_for(4, 0.5) == 8
    assert O.hash_range_for(10, 3.0) == 4
    assert O.hash_range_for(5, 2.0) == 3
    with pytest.raises(ValueError):
        O.hash_range_for(10, 1e-308)


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_build_matches_reference_golden(workers):
    cases, _ = load_golden("build")
    for c in cases:
        off, placed, pos = O.build_csr(c["keys"], int(c["hash_range"]), int(c["kind"]), int(c["seed"]), workers)
        # the restatement is stable, so it reproduces the reference bit for bit
        assert np.array_equal(off, c["offset"])
        assert np.array_equal(placed, c["placed"])
        assert np.array_equal(pos, c["positions"])


def test_build_hand_example():
    off, placed, _ = O.build_csr(np.array([0, 2, 2, 5], np.uint32), 4, O.KIND_IDENTITY)
    assert off.tolist() == [0, 1, 2, 4, 4]
    assert placed.tolist() == [0, 5, 2, 2]


@pytest.mark.parametrize("workers", [1, 4])
def test_query_matches_reference_golden(workers):
    cases, _ = load_golden("query")
    for c in cases:
        v = int(c["hash_range"])
        off, placed, _ = O.build_csr(c["keys"], v, int(c["kind"]), int(c["seed"]))
        mult, matched, total, comp, hv = O.query(off, placed, c["queries"], int(c["kind"]), int(c["seed"]), workers)
        assert np.array_equal(mult, c["multiplicities"])
        assert (matched, total, comp, hv) == (int(c["matched"]), int(c["total"]), int(c["comparisons"]), int(c["hash_values"]))
        assert np.array_equal(mult, O.count_occurrences(c["keys"], c["queries"]))


def test_sharded_matches_reference_golden():
    cases, _ = load_golden("sharded")
    for c in cases:
        p = int(c["p"])
        parts = [c[f"in{d}"] for d in range(p)]
        s = O.build_sharded(parts, p, float(c["load_factor"]), int(c["bins_in"]), int(c["hr_in"]),
                            int(c["kind"]), int(c["seed"]))
        assert (s["hash_range"], s["bins_g"], s["bin_size"]) == (int(c["hash_range"]), int(c["bins_g"]), int(c["bin_size"]))
        assert np.array_equal(s["splits"], c["splits"])
        assert s["received"] == c["received"].tolist()
        assert s["search_steps"] == int(c["search_steps"])
        for d, (off, keys) in enumerate(s["tables"]):
            assert np.array_equal(off, c[f"off{d}"])
            assert np.array_equal(keys, c[f"keys{d}"])
        for d, a in enumerate(parts):
            offs, grouped, _ = O.reorganize(a, s["splits"], s["hash_range"], s["bin_size"], int(c["kind"]), int(c["seed"]))
            assert np.array_equal(offs, c[f"send_off{d}"])
            assert np.array_equal(grouped, c[f"send_keys{d}"])
        mult, matched, total, comp, hv = O.query_sharded(s, c["queries"], int(c["kind"]), int(c["seed"]))
        assert np.array_equal(mult, c["multiplicities"])
        assert (matched, total, comp, hv) == (int(c["matched"]), int(c["total"]), int(c["comparisons"]), int(c["hash_values"]))


def test_plan_hand_example():
    splits = O.plan_splits([np.array([0, 1], np.uint32), np.array([2, 3], np.uint32)], 4, 4, O.KIND_IDENTITY)
    assert splits.tolist() == [0, 2, 4]
    assert O.dest_of_hash(np.array([0, 1, 2, 3]), splits, 1).tolist() == [0, 0, 1, 1]


def test_splitmix_golden():
    assert O.splitmix64_at(0, np.arange(4)).tolist() == [
        16294208416658607535, 7960286522194355700, 487617019471545679, 17909611376780542444]
    cases, _ = load_golden("workload")
    for c in cases:
        if "idx" in c:
            assert np.array_equal(O.splitmix64_at(int(c["seed"]), c["idx"]), c["out"])
        else:
            got = O.generate_keys(int(c["k"]), int(c["count"]), int(c["seed"]))
            assert np.array_equal(got, c["keys"])
            # array_split slices address the same stream
            half = int(c["count"]) // 2
            tail = O.generate_keys(int(c["k"]), int(c["count"]) - half, int(c["seed"]), start=half)
            assert np.array_equal(tail, c["keys"][half:])


def test_u64_restatement_reduces_to_structure():
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 1 << 63, size=5000, dtype=np.uint64)
    keys[:100] = keys[100:200]  # duplicates
    v = 4096
    off, placed, pos = O.build_csr(keys, v, O.KIND_MURMUR, 3)
    assert np.array_equal(placed, keys[pos])
    h = O.hash_keys(O.KIND_MURMUR, 3, placed, v)
    assert np.array_equal(h, np.repeat(np.arange(v), np.diff(off)))
    q = np.concatenate([keys[:300], rng.integers(0, 1 << 63, size=300, dtype=np.uint64)])
    mult = O.query(off, placed, q, O.KIND_MURMUR, 3)[0]
    assert np.array_equal(mult, O.count_occurrences(keys, q))
    assert O.hash_scalar(O.KIND_MURMUR, 3, int(keys[7]), v, key_bits=64) == int(O.hash_keys(O.KIND_MURMUR, 3, keys[7:8], v)[0])
