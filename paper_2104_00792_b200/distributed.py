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

`transport="p2p"` replaces Phase 2 + Phase 3 by one kernel: after a P x P
all_gather of the send counts (the only host sync), hg_reorganize_place_peers
stores every key straight into its owner's receive buffer -- a symmetric
allocation (torch symmetric memory) mapped into every rank over NVLink /
NVSwitch -- at the slot the alltoallv would have produced (senders in rank
order, input order inside a sender), so the exchange overlaps the scatter
tile by tile and no staging copy of the keys exists.  Queries go out the same
way and hg_return_peers writes each answer straight into the sender's buffer
at the key's grouped position.  Device barriers on the symmetric handle
order the buffer reuse; small collectives (counts, bin sums, aggregates) stay
on NCCL.

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
    transport: str = "nccl"  # "nccl" (all_to_all_single) or "p2p" (fused peer-memory scatter)

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

    # ---- one-pass routing (both transports) and the fused peer-memory exchange
    def segment_sums(self, local_counts, splits):
        """Per-destination key counts from this rank's bin histogram: sum of
        local_counts[splits[d]:splits[d+1]] (no second pass over the keys)."""
        t = D.torch()
        cs = t.cat([t.zeros(1, dtype=t.int64, device=local_counts.device), local_counts.to(t.int64).cumsum(0)])
        return cs[splits[1:]] - cs[splits[:-1]]

    def route(self, keys, hash_range, bin_size, splits, shards, family, row_offsets, dest_ptrs=None, dest_base=None,
              want_order=False):
        """hg_route: keys to their destination rows, locally (returns grouped)
        or straight into peer buffers (dest_ptrs); returns (grouped, order)."""
        t = D.torch()
        n = keys.numel()
        kind, seed = family_code(family)
        grouped = None if dest_ptrs is not None else self.empty_keys(n)
        order = t.empty(n, dtype=t.int32, device=keys.device) if want_order else None
        cursors = t.empty(shards, dtype=t.int64, device=keys.device)
        _lib.call("hg_route", D.ptr(keys), n, self.key_bits, kind, seed, hash_range, bin_size, D.ptr(splits), shards,
                  D.ptr(_dev_i64(self, row_offsets)), D.ptr(dest_ptrs), D.ptr(dest_base), D.ptr(grouped), D.ptr(order),
                  D.ptr(cursors), D.stream_ptr())
        return grouped, order

    def return_peers(self, vals, recv_bounds, back_ptrs, back_base, shards):
        _lib.call("hg_return_peers", D.ptr(vals), vals.numel(), D.ptr(recv_bounds), D.ptr(back_ptrs),
                  D.ptr(back_base), shards, D.stream_ptr())

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
    transport: str = "nccl"


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised (launch one process per GPU with torchrun)")
    return dist


def _alltoallv(dist, out, inp, out_splits, in_splits, group):
    dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=group)
    return out


def peer_layout(counts, rank: int) -> dict:
    """Slot arithmetic of the fused exchange from the all-gathered P x P count
    matrix (counts[s, d] = keys sender s routes to destination d).  It equals
    the layout of all_to_all_single / ExchangeFabric.gather (multishard.py:
    137-166): receiver d holds the rows of senders 0..P-1 in rank order.

      dest_base[d]    this rank's first slot in destination d's receive buffer
      recv_bounds[s]  sender s's segment start in this rank's receive buffer (P+1)
      back_base[s]    where this rank's answers for sender s start in s's grouped order
      n_recv          keys this rank receives; capacity: max receive size over ranks
      n_send_max      max keys any rank sends (the reverse buffers' size)"""
    c = np.asarray(counts, dtype=np.int64)
    col_pre = np.cumsum(c, axis=0) - c  # [s, d]: sum over s' < s of c[s', d]
    row_pre = np.cumsum(c, axis=1) - c  # [s, d]: sum over d' < d of c[s, d']
    n_recv = int(c[:, rank].sum())
    return {
        "dest_base": col_pre[rank].copy(),
        "recv_bounds": np.concatenate([col_pre[:, rank], [n_recv]]),
        "back_base": row_pre[:, rank].copy(),
        "n_recv": n_recv,
        "capacity": int(c.sum(axis=0).max()) if c.size else 0,
        "n_send_max": int(c.sum(axis=1).max()) if c.size else 0,
    }


class PeerBuffers:
    """Symmetric receive buffers for the fused exchange, grown on demand.

    Allocation and rendezvous are collective: every rank calls `get` with the
    same (name, size), which the all-gathered count matrix guarantees."""

    def __init__(self, group=None):
        self.group = group
        self._bufs = {}
        self._ok = None

    def available(self) -> bool:
        """Whether symmetric memory works on every rank (decided once, agreed by
        an all_reduce MIN so no rank takes the peer path alone)."""
        if self._ok is None:
            import warnings

            import torch.distributed as dist

            t = D.torch()
            # Capability is decided locally first (import + a local symmetric
            # allocation, no collective), agreed by all_reduce(MIN), and only
            # then does any rank enter the collective rendezvous: a rank that
            # cannot use peer memory never leaves the others blocked in it.
            try:
                import torch.distributed._symmetric_memory as symm_mem

                symm_mem.empty(1 << 10, dtype=t.int32, device=D.device())
                ok = 1
            except Exception as e:  # no symmetric-memory support: NCCL alltoallv instead
                warnings.warn(f"peer-memory exchange unavailable ({e}); using NCCL all_to_all")
                ok = 0
            flag = t.tensor([ok], dtype=t.int32, device=D.device())
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
            self._ok = bool(int(flag.item()))
            if self._ok:
                self.get("probe", 1 << 10, t.int32)  # collective: every rank agreed to enter
        return self._ok

    def get(self, name: str, n: int, dtype):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        t = D.torch()
        cur = self._bufs.get(name)
        if cur is None or cur[0].numel() < n or cur[0].dtype != dtype:
            cap = max(1 << 16, n + n // 8)  # headroom so small run-to-run changes reuse the mapping
            buf = symm_mem.empty(cap, dtype=dtype, device=D.device())
            handle = symm_mem.rendezvous(buf, group=self.group or dist.group.WORLD)
            ptrs = t.tensor(list(handle.buffer_ptrs), dtype=t.int64, device=D.device())
            cur = self._bufs[name] = (buf, handle, ptrs)
        return cur


_PEER_BUFFERS = {}


def _peer_buffers(group) -> PeerBuffers:
    key = id(group)
    if key not in _PEER_BUFFERS:
        _PEER_BUFFERS[key] = PeerBuffers(group)
    return _PEER_BUFFERS[key]


def _gather_counts(dist, ops, send_counts, world, group):
    """All-gather of every rank's per-destination counts -> host P x P matrix."""
    t = D.torch()
    out = t.zeros(world * world, dtype=t.int64, device=send_counts.device)
    dist.all_gather_into_tensor(out, send_counts.to(t.int64).contiguous(), group=group)
    return out.cpu().numpy().reshape(world, world)


def _dev_i64(ops, arr):
    t = D.torch()
    return t.tensor(np.asarray(arr, dtype=np.int64), dtype=t.int64, device=ops.device())


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
    local_counts = ops.bin_histogram(keys, hr, bins_g, bin_size, config.family)
    counts = local_counts.clone()
    dist.all_reduce(counts, group=group)
    splits = ops.split_plan(counts, bins_g, total, world)
    t1 = time.perf_counter_ns()

    # Phase 2 + 3: per-destination counts are segment sums of the local
    # histogram; one all_gather gives every rank the P x P matrix (the only
    # host sync), then one routing pass -- straight into the owners' symmetric
    # buffers (p2p) or into a local grouped buffer for the NCCL alltoallv
    mat = _gather_counts(dist, ops, ops.segment_sums(local_counts, splits), world, group)
    lay = peer_layout(mat, rank)
    send_h = [int(x) for x in mat[rank]]
    n_recv = lay["n_recv"]
    row_off = np.concatenate([[0], np.cumsum(mat[rank])[:-1]])
    t2 = time.perf_counter_ns()
    if config.transport == "p2p" and _peer_buffers(group).available():
        buf, handle, ptrs = _peer_buffers(group).get("keys", lay["capacity"], keys.dtype)
        handle.barrier()  # every rank is done reading its buffer from the previous exchange
        ops.route(keys, hr, bin_size, splits, world, config.family, row_off, ptrs, _dev_i64(ops, lay["dest_base"]))
        handle.barrier()  # all peer stores have landed
        received = buf[:n_recv]
    else:
        grouped, _ = ops.route(keys, hr, bin_size, splits, world, config.family, row_off)
        received = ops.empty_keys(n_recv)
        _alltoallv(dist, received, grouped, [int(x) for x in mat[:, rank]], send_h, group)
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
                     bytes_sent=kb * (n_local - send_h[rank]), transport=config.transport)


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
    local_counts = ops.bin_histogram(q, plan.hash_range, plan.bins_g, plan.bin_size, table.family)
    mat = _gather_counts(dist, ops, ops.segment_sums(local_counts, splits), world, group)
    lay = peer_layout(mat, rank)
    row_off = np.concatenate([[0], np.cumsum(mat[rank])[:-1]])
    if getattr(table, "transport", "nccl") == "p2p" and _peer_buffers(group).available():
        pb = _peer_buffers(group)
        qbuf, handle, qptrs = pb.get("queries", lay["capacity"], q.dtype)
        bbuf, _, bptrs = pb.get("answers", lay["n_send_max"], t.int32)
        handle.barrier()  # previous users of both buffers are done
        _, order = ops.route(q, plan.hash_range, plan.bin_size, splits, world, table.family, row_off, qptrs,
                             _dev_i64(ops, lay["dest_base"]), want_order=True)
        handle.barrier()  # queries landed
        mult_in, agg = ops.query(table.shard, qbuf[:lay["n_recv"]])
        ops.return_peers(mult_in, _dev_i64(ops, lay["recv_bounds"]), bptrs, _dev_i64(ops, lay["back_base"]), world)
        handle.barrier()  # answers landed in every sender's grouped order
        mult = ops.scatter(bbuf[:nq], order, nq)
    else:
        grouped, order = ops.route(q, plan.hash_range, plan.bin_size, splits, world, table.family, row_off,
                                   want_order=True)
        send_h = [int(x) for x in mat[rank]]
        recv_h = [int(x) for x in mat[:, rank]]
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
