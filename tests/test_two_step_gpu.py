"""The reference's two-step query through the binned path (GPU only).

build_query_table (query.py:84-95) runs a traced binned build: positions come
from the partition's own position maps (k_repart), not from global atomics;
intersect_tables (query.py:120-179) probes the trace's grouped query keys and
returns the counts to query order through the trace's position maps (or, for
positions it did not produce, probes the query table's fine-bin slices and
scatters).  Parity: the same multiplicities
and matched / total / comparisons as the oracle's two-step query, positions a
permutation with keys[positions] == the table's keys.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2104_00792_b200")


def two_step(keys, queries, v, key_bits=32, copy_positions=False):
    table = hg.build(keys, 1.0, hash_range=v, key_bits=key_bits)
    qt, positions = hg.build_query_table(table, queries)
    assert positions.dtype == np.int64 and not positions.flags.writeable
    assert np.array_equal(np.sort(positions), np.arange(len(queries)))
    assert np.array_equal(np.asarray(queries)[positions], qt.keys)
    off_q, placed_q, _ = O.build_csr(queries, v)
    assert np.array_equal(qt.offset, off_q)
    assert np.array_equal(O.canonical(qt.offset, qt.keys)[1], O.canonical(off_q, placed_q)[1])
    pos = positions.copy() if copy_positions else positions
    res = hg.intersect_tables(table, qt, pos)
    off, placed, _ = O.build_csr(keys, v)
    mult, matched, total, comp, _ = O.query(off, placed, queries)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons) == (matched, total, comp)
    return res


@pytest.mark.parametrize("log2", [16, 18, 21])
def test_two_step_traced(log2):
    n = 1 << log2
    keys = O.generate_keys(log2, n, 0)
    queries = O.generate_keys(log2, n + 12345, 0x51)
    two_step(keys, queries, n)


def test_two_step_foreign_positions_scatter():
    n = 1 << 20
    keys = O.generate_keys(20, n, 0)
    queries = O.generate_keys(20, n, 0x51)
    two_step(keys, queries, n, copy_positions=True)


@pytest.mark.parametrize("d", [4, 128, 4096])
def test_two_step_dense(d):
    n = 1 << 20
    keys = O.generate_keys(20, n, 0)
    queries = O.generate_keys(20, n, 0x51)
    two_step(keys, queries, n // d)


def test_two_step_hot_queries():
    n = 1 << 20
    keys = O.generate_keys(20, n, 0)
    queries = np.concatenate([np.full(n // 2, 7, np.uint32), O.generate_keys(20, n // 2, 0x51)])
    two_step(keys, queries, n)


def test_two_step_u64():
    n = 1 << 19
    keys = O.generate_keys(32, n, 0, key_bits=64)
    queries = np.concatenate([keys[::3], O.generate_keys(32, n, 0x51, key_bits=64)])
    two_step(keys, queries, n, key_bits=64)


def test_build_traced_binned_positions():
    n = 1 << 20
    keys = O.generate_keys(20, n, 3)
    table, counters, positions = hg.build_traced(keys)
    assert np.array_equal(keys[positions], table.keys)
    assert np.array_equal(np.sort(positions), np.arange(n))
    off, placed, _ = O.build_csr(keys, table.hash_range)
    assert np.array_equal(table.offset, off)


@pytest.mark.parametrize("log2_t,log2_q", [(18, 21), (21, 17), (20, 20)])
def test_two_step_layouts(log2_t, log2_q):
    """Query tables larger than the table (the trace's fine bins nest inside
    the probe's), smaller and equal: the probe reads the trace's grouped keys
    at the table's probe layout (at C = 1 both pick the same fine bins)."""
    keys = O.generate_keys(log2_t, 1 << log2_t, 0)
    queries = O.generate_keys(log2_t, 1 << log2_q, 0x51)
    two_step(keys, queries, 1 << log2_t)


@pytest.mark.parametrize("log2_q", [15, 17])
def test_two_step_coarser_trace(log2_q):
    """A dense table (4 keys per bucket: smaller fine bins) with a sparser
    query table: the trace's fine bins are coarser than the table's probe
    layout, so the probe runs at the trace's layout over its grouped keys
    (table slices above the smem capacity take the map / hash-table paths)."""
    n = 1 << 20
    keys = O.generate_keys(20, n, 0)
    queries = np.concatenate([O.generate_keys(20, (1 << log2_q) - 1000, 0x51), keys[:1000]])
    two_step(keys, queries, n // 4)
