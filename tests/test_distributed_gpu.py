"""The NCCL path of paper_2104_00792_b200.distributed on the one GPU a test box
has (world_size 1, so every collective is local): device ops, all_reduce of the
bin counters, alltoallv of keys and multiplicities, against the oracle."""

import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29731")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("n,dom,lf", [(1 << 20, 1 << 22, 1.0), (300_001, 1 << 10, 0.5)])
def test_distributed_single_rank_matches_oracle(nccl_group, n, dom, lf, transport):
    from paper_2104_00792_b200 import HashFamily
    from paper_2104_00792_b200.distributed import DistConfig, build_distributed, query_distributed

    rng = np.random.default_rng(n)
    keys = rng.integers(1, dom + 1, size=n, dtype=np.uint64).astype(np.uint32)
    qs = rng.integers(1, dom + 1, size=n // 2, dtype=np.uint64).astype(np.uint32)
    table = build_distributed(keys, DistConfig(load_factor=lf, family=HashFamily.murmur32(9), transport=transport))
    ref = O.build_sharded([keys], 1, load_factor=lf, kind=0, seed=9)
    assert np.array_equal(table.plan.bin_splits, ref["splits"])
    off, placed = ref["tables"][0]
    assert np.array_equal(table.shard.offset, off)
    assert np.array_equal(O.canonical(table.shard.offset, table.shard.keys)[1], O.canonical(off, placed)[1])
    res = query_distributed(table, qs)
    mult, matched, total, comp, hv = O.query_sharded(ref, qs, 0, 9)
    assert np.array_equal(res.multiplicities, mult)
    assert (res.matched_positions, res.total_matches, res.comparisons, res.hash_values) == (matched, total, comp, hv)


def test_p2p_repeated_calls_reuse_buffers(nccl_group):
    """Back-to-back p2p builds/queries of different sizes reuse (and grow) the
    symmetric buffers; every result still equals the oracle."""
    from paper_2104_00792_b200 import HashFamily
    from paper_2104_00792_b200.distributed import DistConfig, build_distributed, query_distributed

    for i, n in enumerate([1 << 16, 1 << 18, 5000, 1 << 18]):
        rng = np.random.default_rng(100 + i)
        keys = rng.integers(1, 1 << 20, size=n, dtype=np.uint64).astype(np.uint32)
        qs = rng.integers(1, 1 << 20, size=n, dtype=np.uint64).astype(np.uint32)
        table = build_distributed(keys, DistConfig(transport="p2p"))
        res = query_distributed(table, qs)
        assert np.array_equal(res.multiplicities, O.count_occurrences(keys, qs))
