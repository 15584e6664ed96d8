"""Multi-process (world_size 2 and 3) check of the one-process-per-GPU path on
CPU: paper_2104_00792_b200.distributed orchestrates the four phases over a
gloo process group, with the compute steps supplied by an oracle-backed ops
object (the CUDA kernels are covered by the GPU tests).  The result must equal
the reference's single-process sharded build and query on the same shards."""

import os
import pickle
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

FAMILY = None  # set per test via args


class OracleTable:
    def __init__(self, offset, keys, v):
        self.offset, self.keys, self.hash_range, self.key_bits = offset, keys, v, 32


class OracleOps:
    """CPU stand-in for DeviceOps built on the numpy restatement (test only)."""

    key_bits = 32

    def __init__(self, kind, seed):
        self.kind, self.seed = kind, seed

    def device(self):
        return torch.device("cpu")

    def to_local(self, keys):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.uint32)).view(np.int32).copy())

    @staticmethod
    def _np(t):
        return t.numpy().view(np.uint32)

    def bin_histogram(self, keys, hr, bins_g, bin_size, family):
        return torch.from_numpy(O.bin_histogram(self._np(keys), hr, bins_g, self.kind, self.seed).astype(np.int64))

    def split_plan(self, counts, bins_g, total, shards):
        return torch.from_numpy(O.splits_from_bins(counts.numpy(), total, shards))

    def reorganize(self, keys, hr, bin_size, splits, shards, family, want_order=False, steps=None):
        k = self._np(keys)
        if len(k):
            dest = O.dest_of_hash(O.hash_keys(self.kind, self.seed, k, hr), splits.numpy(), bin_size)
        else:
            dest = np.zeros(0, np.int64)
        offs = np.zeros(shards + 1, dtype=np.int64)
        np.cumsum(np.bincount(dest, minlength=shards), out=offs[1:])
        order = np.argsort(dest, kind="stable")
        grouped = torch.from_numpy(k[order].view(np.int32).copy())
        return torch.from_numpy(offs), grouped, torch.from_numpy(order.astype(np.int32))

    def build(self, keys, v, family, load_factor):
        off, placed, _ = O.build_csr(self._np(keys), v, self.kind, self.seed)
        return OracleTable(off, placed, v)

    def query(self, table, queries):
        mult, matched, total, comp, _ = O.query(table.offset, table.keys, self._np(queries), self.kind, self.seed)
        return (torch.from_numpy(mult.astype(np.uint32).view(np.int32)),
                torch.tensor([matched, total, comp], dtype=torch.int64))

    def scatter(self, src, order, n):
        out = torch.zeros(n, dtype=torch.int32)
        out[order.long()] = src
        return out

    def zeros_i64(self, n):
        return torch.zeros(n, dtype=torch.int64)

    def empty_keys(self, n):
        return torch.empty(n, dtype=torch.int32)

    def empty_u32(self, n):
        return torch.empty(n, dtype=torch.int32)


def _worker(rank, world, port, outdir, parts, queries, kind, seed, lf):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_00792_b200 import HashFamily, HashKind
        from paper_2104_00792_b200.distributed import DistConfig, build_distributed, query_distributed

        fam = HashFamily(HashKind(kind), seed)
        ops = OracleOps(kind, seed)
        table = build_distributed(parts[rank], DistConfig(load_factor=lf, family=fam), ops=ops)
        res = query_distributed(table, queries[rank], ops=ops)
        out = dict(splits=table.plan.bin_splits.copy(), received=table.received_count,
                   offset=table.shard.offset, keys=table.shard.keys, hash_range=table.plan.hash_range,
                   mult=res.multiplicities_device.numpy().view(np.uint32).astype(np.int64),
                   agg=res._agg_device.numpy().copy(), hv=res.hash_values)
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(out, f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,dom,kind,seed,lf", [
    (2, 20_000, 1 << 14, 0, 0, 1.0),
    (3, 9_001, 1 << 10, 0, 12345, 0.5),
    (2, 5_000, 50, 1, 0, 2.0),
])
def test_build_and_query_distributed_match_reference(world, n, dom, kind, seed, lf):
    rng = np.random.default_rng(n + world)
    keys = rng.integers(1, dom + 1, size=n, dtype=np.uint64).astype(np.uint32)
    qs = rng.integers(1, dom + 1, size=n // 2, dtype=np.uint64).astype(np.uint32)
    parts = [np.ascontiguousarray(p) for p in np.array_split(keys, world)]
    qparts = [np.ascontiguousarray(p) for p in np.array_split(qs, world)]
    port = 29600 + (n + world * 7) % 300
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, d, parts, qparts, kind, seed, lf), nprocs=world, join=True)
        outs = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(world)]
    ref = O.build_sharded(parts, world, load_factor=lf, kind=kind, seed=seed)
    for r, o in enumerate(outs):
        assert np.array_equal(o["splits"], ref["splits"])
        assert o["received"] == ref["received"][r]
        off, placed = ref["tables"][r]
        assert np.array_equal(o["offset"], off)
        assert np.array_equal(O.canonical(o["offset"], o["keys"])[1], O.canonical(off, placed)[1])
        assert np.array_equal(o["mult"], O.count_occurrences(keys, qparts[r]))
    mult, matched, total, comp, hv = O.query_sharded(ref, qs, kind, seed)
    agg = outs[0]["agg"]
    assert (int(agg[0]), int(agg[1]), int(agg[2])) == (matched, total, comp)
    assert outs[0]["hv"] == hv
