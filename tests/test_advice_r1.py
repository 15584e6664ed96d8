"""Regression tests for the round-1 advisor findings."""

import numpy as np
import pytest

import oracle as O

hg = pytest.importorskip("paper_2104_00792_b200")
IDENT = hg.HashFamily.identity()


class _Table32:
    key_bits = 32


def test_wide_queries_rejected_for_32bit_table_cpu():
    """64-bit query keys that do not fit 32 bits are refused, not truncated
    (a KEY8 file or --key-bits 64 workload against an HGR1 table)."""
    from paper_2104_00792_b200 import query as Q

    with pytest.raises(hg.ConfigError):
        Q._query_keys(_Table32(), np.array([1, 1 << 40], dtype=np.uint64))
    with pytest.raises(hg.ConfigError):
        Q._query_keys(_Table32(), np.array([-1], dtype=np.int64))


@pytest.mark.gpu
def test_wide_queries_fit_or_refuse_gpu():
    import torch

    t = hg.build(np.array([1, 2, 3], dtype=np.uint32))
    # 64-bit arrays whose values fit 32 bits still query (reference-compatible)
    res = hg.intersect(t, np.array([1, 4], dtype=np.uint64))
    assert res.multiplicities.tolist() == [1, 0]
    with pytest.raises(hg.ConfigError):
        hg.intersect(t, torch.tensor([1, 1 << 33], dtype=torch.int64, device="cuda"))


@pytest.mark.gpu
def test_intersect_at_hash_range_2_32_top_bucket():
    """v = 2^32 (accepted, like the reference): bucket 2^32-1 must read
    offsets[2^32], not wrap to offsets[0] (k_intersect indexed with h + 1 in
    32 bits)."""
    v = 1 << 32
    keys = np.array([0xFFFFFFFF, 5, 0xFFFFFFFF], dtype=np.uint32)
    table = hg.build(keys, 1.0, IDENT, hash_range=v)
    res = hg.intersect(table, np.array([0xFFFFFFFF, 7, 5], dtype=np.uint32))
    assert res.multiplicities.tolist() == [2, 0, 1]
    assert (res.matched_positions, res.total_matches) == (2, 3)
    assert res.comparisons == 2 + 0 + 1
    qt, pos = hg.build_query_table(table, np.array([0xFFFFFFFF], dtype=np.uint32))
    r2 = hg.intersect_tables(table, qt, pos)
    assert r2.multiplicities.tolist() == [2] and r2.comparisons == 2


@pytest.mark.gpu
@pytest.mark.parametrize("shards", [1024, 2000, 4096])
def test_reorganize_many_shards(shards):
    """>= 1024 destinations need the opt-in dynamic shared memory limit."""
    rng = np.random.default_rng(shards)
    keys = rng.integers(0, 1 << 32, size=1 << 16, dtype=np.uint64).astype(np.uint32)
    hr = 1 << 20
    plan = hg.plan_partition([keys[i::shards] for i in range(shards)], hash_range=hr, bins_g=1 << 13)
    sb = hg.reorganize(keys, plan)
    dest = O.dest_of_hash(O.hash_keys(0, 0, keys, hr), plan.bin_splits, plan.bin_size)
    for d in (0, shards // 2, shards - 1):
        assert np.array_equal(sb.row(d), keys[dest == d])


@pytest.mark.gpu
def test_query_agg_accumulates_on_every_path():
    """hg_query's agg is accumulated (caller zeroes) on the binned and the
    direct path alike, so shard queries can sum into one buffer."""
    import torch

    from paper_2104_00792_b200 import _device as D
    from paper_2104_00792_b200 import _lib
    from paper_2104_00792_b200.query import query_device  # noqa: F401

    for n in (1 << 10, 1 << 18):  # direct, binned
        keys = O.generate_keys(20, n, 0)
        table = hg.build(keys)
        qd = D.to_device_keys(O.generate_keys(20, n, 0x51), 32)
        agg = torch.zeros(3, dtype=torch.int64, device="cuda")
        mult = torch.empty(n, dtype=torch.int32, device="cuda")
        ws = D.workspace(_lib.load().hg_query_workspace_size(n, table.hash_range, table.num_keys, 32))
        for _ in range(2):
            _lib.call("hg_query", D.ptr(table.offset_device), D.ptr(table.keys_device), table.num_keys, D.ptr(qd), n,
                      32, 0, 0, table.hash_range, D.ptr(mult), D.ptr(agg), D.ptr(ws), ws.numel(), D.stream_ptr())
        one = hg.intersect(table, qd)
        got = agg.cpu().numpy()
        assert got.tolist() == [2 * one.matched_positions, 2 * one.total_matches, 2 * one.comparisons], n
