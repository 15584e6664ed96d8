"""Seeded random configurations through the CUDA path vs the oracle (GPU only).

Each case draws a key count, key width, hash kind and seed, a hash range from
"one bucket" to "far sparser than the keys", a key distribution (uniform over
a small or large domain, a few hot keys mixed in, all-identical runs) and a
query set (present, absent and hot keys), so the binned path's layouts (one
or two levels, 128- or 256-way level 2), probe depth classes (slots, linear
tail, sorted search, map), oversized-bin build, slice map, hash table and hot
bin work items all meet inputs nobody hand-picked.  Checked like every parity
test: offsets exact, buckets equal as multisets, multiplicities and
matched / total / comparisons exact; the two-step query agrees.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")


def draw(seed):
    rng = np.random.default_rng(1000 + seed)
    key_bits = 64 if rng.random() < 0.3 else 32
    n = int(2 ** rng.uniform(16, 21))
    dom_bits = int(rng.choice([8, 12, 16, 20, 28, 32]))
    kind = O.KIND_IDENTITY if rng.random() < 0.2 else O.KIND_MURMUR
    hi = (1 << dom_bits) if dom_bits < 64 else None
    keys = rng.integers(0, hi, size=n, dtype=np.uint64)
    if key_bits == 64 and rng.random() < 0.5:
        keys = keys * np.uint64(0x9E3779B97F4A7C15)
    style = rng.integers(0, 3)
    if style == 1:  # a few hot keys
        hot = rng.integers(0, 1 << 31, size=4, dtype=np.uint64)
        m = rng.random(n) < 0.3
        keys[m] = hot[rng.integers(0, 4, size=int(m.sum()))]
    elif style == 2:  # an all-identical run
        keys[: n // 3] = np.uint64(rng.integers(0, 1 << 31))
    keys = keys.astype(np.uint32) if key_bits == 32 else keys
    q = int(2 ** rng.uniform(14, 21))
    queries = np.concatenate([rng.choice(keys, size=q // 2),
                              rng.integers(0, 1 << 32, size=q - q // 2, dtype=np.uint64).astype(keys.dtype)])
    rng.shuffle(queries)
    v = max(1, int(n * 2 ** rng.uniform(-12, 6)))
    seed_h = int(rng.integers(0, 1 << 32))
    return keys, queries, v, kind, seed_h, key_bits


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_vs_oracle(seed):
    keys, queries, v, kind, seed_h, key_bits = draw(seed)
    fam = hg.HashFamily(hg.HashKind(kind), seed_h)
    table = hg.build(keys, 1.0, family=fam, hash_range=v, key_bits=key_bits)
    off, placed, _ = O.build_csr(keys, v, kind=kind, seed=seed_h, workers=O.default_workers())
    assert np.array_equal(table.offset, off)
    assert np.array_equal(O.canonical(table.offset, table.keys)[1], O.canonical(off, placed)[1])
    res = hg.intersect(table, queries)
    mult, matched, total, comp, _ = O.query(off, placed, queries, kind=kind, seed=seed_h, workers=O.default_workers())
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons) == (matched, total, comp)
    if seed % 3 == 0:  # the reference's two-step query on the same inputs
        qt, pos = hg.build_query_table(table, queries)
        two = hg.intersect_tables(table, qt, pos)
        assert np.array_equal(two.multiplicities, mult)
        assert (two.matched_positions, two.total_matches, two.comparisons) == (matched, total, comp)
