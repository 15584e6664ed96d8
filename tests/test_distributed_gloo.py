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

    def segment_sums(self, local_counts, splits):
        cs = np.concatenate([[0], np.cumsum(local_counts.numpy())])
        sp = splits.numpy()
        return torch.from_numpy((cs[sp[1:]] - cs[sp[:-1]]).astype(np.int64))

    def route(self, keys, hr, bin_size, splits, shards, family, row_offsets, dest_ptrs=None, dest_base=None,
              want_order=False):
        offs, grouped, order = self.reorganize(keys, hr, bin_size, splits, shards, family, want_order=True)
        offs = offs.numpy()
        assert np.array_equal(offs[:-1], np.asarray(row_offsets))  # counts from the histogram == real row sizes
        # hg_route's claims race: any order inside a row is valid -- shuffle rows to prove nothing depends on it
        rng = np.random.default_rng(len(grouped))
        perm = np.concatenate([offs[d] + rng.permutation(offs[d + 1] - offs[d]) for d in range(shards)]).astype(np.int64)
        perm = torch.from_numpy(perm)
        return grouped[perm], (order[perm] if want_order else None)

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


# ---- fused peer-memory exchange: slot arithmetic (no GPU, no process group)

def _emulate_p2p(rows_per_sender, rank_of_dest_layouts):
    """Place every sender's row d at dest_base into receiver d's buffer, as
    hg_reorganize_place_peers does, and return the receive buffers."""
    P = len(rows_per_sender)
    mat = np.array([[len(rows_per_sender[s][d]) for d in range(P)] for s in range(P)])
    from paper_2104_00792_b200.distributed import peer_layout

    lays = [peer_layout(mat, r) for r in range(P)]
    recv = [np.full(lays[d]["n_recv"], -1, dtype=np.int64) for d in range(P)]
    for s in range(P):
        for d in range(P):
            row = rows_per_sender[s][d]
            b = lays[s]["dest_base"][d]
            assert np.all(recv[d][b:b + len(row)] == -1), "overlapping peer writes"
            recv[d][b:b + len(row)] = row
    return mat, lays, recv


@pytest.mark.parametrize("P,seed", [(1, 0), (2, 1), (3, 2), (8, 3), (8, 4)])
def test_peer_layout_equals_alltoallv(P, seed):
    rng = np.random.default_rng(seed)
    rows = [[rng.integers(0, 1 << 30, size=int(rng.integers(0, 50) if rng.random() > 0.2 else 0)) for _ in range(P)]
            for _ in range(P)]
    mat, lays, recv = _emulate_p2p(rows, None)
    for d in range(P):
        # ExchangeFabric.gather(d): senders' rows in rank order (multishard.py:137-166)
        expect = np.concatenate([rows[s][d] for s in range(P)]) if P else np.zeros(0)
        assert np.array_equal(recv[d], expect)
        assert lays[d]["n_recv"] == mat[:, d].sum()
        assert lays[d]["capacity"] == mat.sum(axis=0).max()
    # reverse direction: receiver d's element i of sender s's segment goes back
    # to s's grouped position back_base[s] + (i - recv_bounds[s])
    back = [np.full(mat[s].sum(), -1, dtype=np.int64) for s in range(P)]
    for d in range(P):
        rb, bb = lays[d]["recv_bounds"], lays[d]["back_base"]
        for s in range(P):
            seg = recv[d][rb[s]:rb[s + 1]]
            back[s][bb[s]:bb[s] + len(seg)] = seg
    for s in range(P):
        grouped = np.concatenate([rows[s][d] for d in range(P)])
        assert np.array_equal(back[s], grouped)
        assert lays[s]["n_send_max"] == mat.sum(axis=1).max()
