"""One process per GPU: the paper's multi-GPU HashGraph over torch.distributed.

This is the production form of the partitioned build (Alg. 2,
multishard.py:336-471) and query (multishard.py:485-542): every rank owns one
shard and one GPU; the reference's in-memory ExchangeFabric becomes NCCL
collectives over NVLink / NVSwitch:

  Phase 1  hg_bin_histogram on the local keys -> all_reduce(SUM) of the BINS_G
           counters (the paper's "Reduce") -> hg_split_plan,
           run identically on every rank (replaces the "BCast")
  Phase 2  hg_reorganize: stable per-destination CSR of the local keys
  Phase 3  all_to_all of the P x P send counts, then all_to_all_single
           (alltoallv) of the keys ("AllToAll ... D2D")
  Phase 4  local build with V_d = ceil(N_d / C) over the received keys

A query routes its keys with the same plan (forward alltoallv), answers them on
the owning shard and returns the uint32 multiplicities with the reverse
alltoallv; the sender scatters them back to query order.

Every compute step goes through an `ops` object.  The default, `DeviceOps`,
launches the libhashgraph_b200 kernels; multi-process CPU tests substitute an
oracle-backed implementation to check the orchestration over gloo.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .core import HashGraph, build_device
from .errors import ConfigError
from .hashing import HashFamily, family_code, hash_range_for
from .multishard import PartitionPlan, ShardConfig, bin_histogram_device, reorganize_device, split_plan_device
from .query import QueryResult, query_device


@dataclass(frozen=True)
class DistConfig:
    """ShardConfig for one-process-per-GPU runs: shards = world size."""

    load_factor: float = 1.0
    bins_g: int = 0
    family: HashFamily = HashFamily()
    hash_range: int = 0
    key_bits: int = 32

    def shard_config(self, world: int) -> ShardConfig:
        return ShardConfig(shards=world, load_factor=self.load_factor, bins_g=self.bins_g, family=self.family,
                           hash_range=self.hash_range)


class DeviceOps:
    """Compute steps of the distributed path, on the current CUDA device."""

    def __init__(self, key_bits: int = 32):
        self.key_bits = key_bits

    def device(self):
        return D.device()

    def to_local(self, keys):
        if not D.is_tensor(keys):
            keys = D.coerce_host_keys(keys, self.key_bits)
        return D.to_device_keys(keys, self.key_bits)

    def bin_histogram(self, keys, hash_range, bins_g, bin_size, family):
        return bin_histogram_device([keys], hash_range, bins_g, bin_size, family, self.key_bits)

    def split_plan(self, counts, bins_g, total, shards):
        return split_plan_device(counts, bins_g, total, shards)

    def reorganize(self, keys, hash_range, bin_size, splits, shards, family, want_order=False, steps=None):
        return reorganize_device(keys, hash_range, bin_size, splits, shards, family, self.key_bits, want_order, steps)

    def build(self, keys, v, family, load_factor):
        off, edges, _ = build_device(keys, v, family, self.key_bits)
        return HashGraph(off, edges, v, family, float(load_factor), self.key_bits, keys.numel())

    def query(self, table, queries):
        return query_device(table, queries)

    def scatter(self, src, order, n):
        out = D.torch().zeros(n, dtype=D.torch().int32, device=src.device)
        if src.numel():
            _lib.call("hg_scatter_u32", D.ptr(src), D.ptr(order), src.numel(), D.ptr(out), D.stream_ptr())
        return out

    def zeros_i64(self, n):
        return D.torch().zeros(n, dtype=D.torch().int64, device=D.device())

    def empty_keys(self, n):
        return D.empty(n, self.key_bits)

    def empty_u32(self, n):
        return D.torch().empty(n, dtype=D.torch().int32, device=D.device())

    def synchronize(self):
        D.torch().cuda.synchronize()


@dataclass
class DistTable:
    """This rank's shard of a partitioned HashGraph plus the global plan."""

    plan: PartitionPlan
    shard: object  # HashGraph (or the test ops' table type)
    family: HashFamily
    rank: int
    world: int
    received_count: int
    splits_device: object = field(repr=False, default=None)
    phase_ns: dict = field(default_factory=dict)
    bytes_sent: int = 0


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised (launch one process per GPU with torchrun)")
    return dist


def _alltoallv(dist, out, inp, out_splits, in_splits, group):
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)
    return out


def _exchange_counts(dist, ops, send_counts_i64, world, group):
    """All-to-all of the per-destination counts: returns recv counts (host list)."""
    recv = ops.zeros_i64(world)
    dist.all_to_all_single(recv, send_counts_i64, group=group)
    return recv


def build_distributed(local_keys, config: DistConfig = DistConfig(), group=None, ops=None):
    """The four-phase build with this rank's keys; returns a DistTable.

    Collective: every rank of `group` must call it.  Phase times are measured
    with host wall clock around synchronised phases only when
    `config` asks for them via `ops` timing; by default the call is enqueue-
    heavy with two host syncs (the counts exchange sizes the receive buffer).
    """
    dist = _dist()
    ops = ops or DeviceOps(config.key_bits)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = D.torch()
    keys = ops.to_local(local_keys)
    n_local = keys.numel()
    tot = t.tensor([n_local], dtype=t.int64, device=ops.device())
    dist.all_reduce(tot, group=group)
    total = int(tot.item())
    cfg = config.shard_config(world)
    hr, bins_g, bin_size = cfg.resolve(total)
    t0 = time.perf_counter_ns()

    # Phase 1: local bin histogram -> global sum -> identical split plan everywhere
    counts = ops.bin_histogram(keys, hr, bins_g, bin_size, config.family)
    dist.all_reduce(counts, group=group)
    splits = ops.split_plan(counts, bins_g, total, world)
    t1 = time.perf_counter_ns()

    # Phase 2: per-destination CSR
    rows, grouped, _ = ops.reorganize(keys, hr, bin_size, splits, world, config.family)
    send_counts = rows[1:] - rows[:-1]
    t2 = time.perf_counter_ns()

    # Phase 3: counts exchange, then the keys alltoallv
    recv_counts = _exchange_counts(dist, ops, send_counts.contiguous(), world, group)
    send_h = [int(x) for x in send_counts.cpu().tolist()]
    recv_h = [int(x) for x in recv_counts.cpu().tolist()]
    n_recv = sum(recv_h)
    received = ops.empty_keys(n_recv)
    _alltoallv(dist, received, grouped, recv_h, send_h, group)
    t3 = time.perf_counter_ns()

    # Phase 4: local table with V_d = ceil(N_d / C)
    v_d = hash_range_for(n_recv, config.load_factor)
    shard = ops.build(received, v_d, config.family, config.load_factor)
    t4 = time.perf_counter_ns()

    plan = PartitionPlan(world, hr, bins_g, bin_size, splits.cpu().numpy())
    kb = 4 if config.key_bits == 32 else 8
    return DistTable(plan=plan, shard=shard, family=config.family, rank=rank, world=world, received_count=n_recv,
                     splits_device=splits,
                     phase_ns={"partition": t1 - t0, "preprocess": t2 - t1, "all_to_all": t3 - t2,
                               "table_construction": t4 - t3},
                     bytes_sent=kb * (n_local - send_h[rank]))


def query_distributed(table: DistTable, local_queries, group=None, ops=None):
    """Answer this rank's queries against the partitioned table (collective).

    Returns a QueryResult whose multiplicities are positional for this rank's
    queries; the aggregate counters are summed over all ranks (the reference's
    query_sharded totals, multishard.py:531-541)."""
    dist = _dist()
    ops = ops or DeviceOps(getattr(table.shard, "key_bits", 32))
    t = D.torch()
    world, rank = table.world, table.rank
    plan = table.plan
    q = ops.to_local(local_queries)
    nq = q.numel()
    splits = table.splits_device if table.splits_device is not None else plan.splits_device()
    rows, grouped, order = ops.reorganize(q, plan.hash_range, plan.bin_size, splits, world, table.family,
                                          want_order=True)
    send_counts = rows[1:] - rows[:-1]
    recv_counts = _exchange_counts(dist, ops, send_counts.contiguous(), world, group)
    send_h = [int(x) for x in send_counts.cpu().tolist()]
    recv_h = [int(x) for x in recv_counts.cpu().tolist()]
    incoming = ops.empty_keys(sum(recv_h))
    _alltoallv(dist, incoming, grouped, recv_h, send_h, group)
    mult_in, agg = ops.query(table.shard, incoming)
    back = ops.empty_u32(nq)
    _alltoallv(dist, back, mult_in, send_h, recv_h, group)
    mult = ops.scatter(back, order, nq)
    agg = agg.clone()
    dist.all_reduce(agg, group=group)
    hv = t.tensor([table.shard.hash_range], dtype=t.int64, device=agg.device)
    dist.all_reduce(hv, group=group)
    return QueryResult(mult, agg, int(hv.item()))
