"""Partitioned build across P shards (mirrors multishard.py of the reference).

This module is the single-process drop-in: P shard inputs in, P local tables
out, all driven from the calling thread.  With one GPU per shard visible (or
an explicit `devices=` list) shard d lives on GPU d; otherwise the P shards
are "virtual shards" of the current GPU (the analogue of the reference's shard
threads, multishard.py:414-419).  Every phase is the same sm_100a kernel:

  Phase 1  hg_bin_histogram (per device, summed on shard 0's) + hg_split_plan
  Phase 2  hg_reorganize   (stable per-destination CSR, search-step counter)
  Phase 3  row copies into each owner's receive buffer, ascending sender order
           (device-to-device over NVLink between GPUs; one concatenation on
           one GPU)
  Phase 4  hg_build with the local range V_d = ceil(N_d / C)

The one-process-per-GPU version over NCCL / symmetric memory is
`paper_2104_00792_b200.distributed`.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .core import BuildCounters, HashGraph, build_device
from .errors import ConfigError
from .hashing import HashFamily, family_code, hash_range_for
from .query import QueryResult, QueryStageTimes, query_device

PHASE_NAMES = ("partition", "preprocess", "all_to_all", "table_construction")

PASS_NAMES = (
    "hash",
    "bin_count",
    "dest_search",
    "buffer_place",
    "exchange",
    "local_hash",
    "local_count",
    "local_place",
)


@dataclass(frozen=True)
class ShardConfig:
    """Build configuration; zero means "derive it" (multishard.py:53-80)."""

    shards: int
    load_factor: float = 1.0
    bins_g: int = 0
    family: HashFamily = HashFamily()
    hash_range: int = 0

    def __post_init__(self) -> None:
        if self.shards < 1:
            raise ConfigError(f"shard count must be >= 1, got {self.shards}")
        if self.load_factor <= 0:
            raise ConfigError(f"load factor must be positive, got {self.load_factor}")
        if self.bins_g < 0:
            raise ConfigError(f"bins_g must be >= 0, got {self.bins_g}")
        if self.hash_range < 0:
            raise ConfigError(f"hash_range must be >= 0, got {self.hash_range}")

    def resolve(self, total_keys: int) -> tuple[int, int, int]:
        """(hash_range, bins_g, bin_size) for an input of total_keys."""
        hr = self.hash_range or hash_range_for(total_keys, self.load_factor)
        bins = self.bins_g or max(self.shards, round(math.sqrt(hr)))
        if bins < self.shards:
            raise ConfigError(f"bins_g={bins} is less than shard count {self.shards}")
        return hr, bins, -(-hr // bins)


@dataclass(frozen=True)
class PartitionPlan:
    """Hash-range ownership from global bin counts (multishard.py:83-113).

    Shard d owns hash values [bin_splits[d] * bin_size, bin_splits[d+1] * bin_size).
    """

    shards: int
    hash_range: int
    bins_g: int
    bin_size: int
    bin_splits: np.ndarray

    def __post_init__(self) -> None:
        s = np.asarray(self.bin_splits, dtype=np.int64)
        object.__setattr__(self, "bin_splits", s)
        if len(s) != self.shards + 1 or s[0] != 0 or s[-1] != self.bins_g:
            raise ConfigError(f"malformed bin splits {s}")
        if np.any(np.diff(s) < 0):
            raise ConfigError(f"bin splits not monotone: {s}")
        s.flags.writeable = False

    @property
    def boundaries(self) -> np.ndarray:
        return self.bin_splits * self.bin_size

    def shard_of(self, hashes: np.ndarray) -> np.ndarray:
        """Destination shard of each global hash value (host helper on host arrays)."""
        return np.searchsorted(self.boundaries, hashes, side="right") - 1

    def splits_device(self):
        """bin_splits as an int64 tensor on the current device."""
        return D.torch().from_numpy(np.array(self.bin_splits, dtype=np.int64)).to(D.device())


class SendBuffers:
    """One shard's outgoing keys as a CSR with one row per destination (multishard.py:116-134).

    Held in HBM (`offsets_device` int64[P+1], `keys_device`); `offsets` /
    `keys` / `row()` materialise numpy views for host inspection.
    """

    def __init__(self, offsets, keys, *, key_bits: int = 32, _device=None):
        if _device is not None:
            self.offsets_device, self.keys_device, off_host = _device
            self._offsets = np.asarray(off_host, dtype=np.int64)
            self.key_bits = key_bits
            self._keys = None
            return
        off = np.asarray(offsets, dtype=np.int64)
        ks = np.asarray(keys)
        key_bits = 64 if ks.dtype == np.uint64 else 32
        ks = ks.astype(np.uint64 if key_bits == 64 else np.uint32)
        if off[0] != 0 or off[-1] != len(ks):
            raise ConfigError("send buffer offsets do not cover the key array")
        if np.any(np.diff(off) < 0):
            raise ConfigError("send buffer offsets not monotone")
        self._offsets = off
        self._keys = ks
        self.key_bits = key_bits
        self.offsets_device = None
        self.keys_device = D.to_device_keys(ks, key_bits)

    @property
    def offsets(self) -> np.ndarray:
        return self._offsets

    @property
    def keys(self) -> np.ndarray:
        if self._keys is None:
            self._keys = D.to_numpy_keys(self.keys_device, self.key_bits)
        return self._keys

    @property
    def shards(self) -> int:
        return len(self._offsets) - 1

    def row(self, d: int) -> np.ndarray:
        return self.keys[self._offsets[d]:self._offsets[d + 1]]

    def row_device(self, d: int):
        return self.keys_device[int(self._offsets[d]):int(self._offsets[d + 1])]


@dataclass
class ExchangeFabric:
    """All-to-all between virtual shards on one device (multishard.py:137-166)."""

    shards: int
    posted: list = field(default_factory=list)
    keys_moved: int = 0
    bytes_moved: int = 0

    def __post_init__(self) -> None:
        if not self.posted:
            self.posted = [None] * self.shards

    def post(self, shard: int, buffers: SendBuffers) -> None:
        assert buffers.shards == self.shards, "send CSR row count != shard count"
        self.posted[shard] = buffers

    def gather_device(self, shard: int):
        """Row `shard` of every sender, ascending sender order, as one device array."""
        rows = []
        for s in range(self.shards):
            sb = self.posted[s]
            assert sb is not None, f"shard {s} has not posted its buffers"
            rows.append(sb.row_device(shard))
        kb = rows[0].element_size() if rows else 4
        total = sum(r.numel() for r in rows)
        # one device-side concatenation (a single copy kernel) instead of P
        # separate cudaMemcpyAsync calls
        out = D.torch().cat(rows) if rows else D.torch().empty(0, dtype=D.torch().int32, device=D.device())
        self.keys_moved += total
        self.bytes_moved += kb * total
        return out

    def gather(self, shard: int) -> np.ndarray:
        sb = self.posted[0]
        return D.to_numpy_keys(self.gather_device(shard), sb.key_bits if sb is not None else 32)


@dataclass(frozen=True)
class ShardedHashGraph:
    """P local tables plus the plan that routes keys to them (multishard.py:169-180)."""

    plan: PartitionPlan
    shards: list
    family: HashFamily
    received_counts: list

    @property
    def total_keys(self) -> int:
        return sum(self.received_counts)

    @property
    def devices(self) -> list:
        """The CUDA device holding each shard's table."""
        return [sh.keys_device.device for sh in self.shards]


@dataclass
class PhaseStats:
    time_ns: int = 0
    keys_touched: int = 0
    search_steps: int = 0
    bytes_exchanged: int = 0


@dataclass
class PhaseReport:
    """Per-phase device times and deterministic counters (multishard.py:183-240).

    Phase times are CUDA-event device times of each phase over all shards.
    """

    shards: int
    total_keys: int
    hash_range: int
    bins_g: int
    load_factor: float
    family: HashFamily
    phases: dict
    passes: dict
    search_steps: int
    bytes_exchanged: int
    shard_received_counts: list
    total_time_ns: int
    build_throughput: float

    def to_json_dict(self) -> dict:
        kind = self.family.kind
        return {
            "schema": "phase-report-v1",
            "shards": self.shards,
            "total_keys": self.total_keys,
            "hash_range": self.hash_range,
            "bins_g": self.bins_g,
            "load_factor": self.load_factor,
            "family": kind.name.lower() if hasattr(kind, "name") else str(kind),
            "seed": self.family.seed,
            "total_time_ns": self.total_time_ns,
            "build_throughput_keys_per_sec": self.build_throughput,
            "phases": {
                name: {
                    "time_ns": st.time_ns,
                    "keys_touched": st.keys_touched,
                    "search_steps": st.search_steps,
                    "bytes_exchanged": st.bytes_exchanged,
                }
                for name, st in self.phases.items()
            },
            "passes": dict(self.passes),
            "search_steps": self.search_steps,
            "bytes_exchanged": self.bytes_exchanged,
            "shard_received_counts": list(self.shard_received_counts),
        }


@dataclass(frozen=True)
class AuditVerdict:
    ok: bool
    violations: list


# --------------------------------------------------------------------------- device phases


def _inputs_to_device(per_shard_inputs, key_bits=32):
    out = []
    for k in per_shard_inputs:
        if not D.is_tensor(k):
            k = D.coerce_host_keys(k, key_bits)
        out.append(D.to_device_keys(k, key_bits))
    return out


def bin_histogram_device(arrays, hash_range, bins_g, bin_size, family, key_bits=32, counts=None):
    """Phase 1 histogram of every shard into one uint64[bins_g] device array."""
    t = D.torch()
    if counts is None:
        counts = t.zeros(bins_g, dtype=t.int64, device=D.device())
    kind, seed = family_code(family)
    for a in arrays:
        if a.numel():
            _lib.call("hg_bin_histogram", D.ptr(a), a.numel(), key_bits, kind, seed, hash_range, bins_g, bin_size,
                      D.ptr(counts), D.stream_ptr())
    return counts


def split_plan_device(counts, bins_g, total, shards):
    t = D.torch()
    splits = t.empty(shards + 1, dtype=t.int64, device=D.device())
    _lib.call("hg_split_plan", D.ptr(counts), bins_g, total, shards, D.ptr(splits), D.stream_ptr())
    return splits


def reorganize_device(keys_dev, hash_range, bin_size, splits_dev, shards, family, key_bits=32,
                      want_order=False, steps=None, keep_workspace=False):
    """Phase 2 on device: (row_offsets int64[P+1] device, grouped keys, order u32 | None)
    (+ the workspace, whose tile bases hg_reorganize_gather reuses, with keep_workspace)."""
    t = D.torch()
    n = keys_dev.numel()
    kind, seed = family_code(family)
    rows = t.empty(shards + 1, dtype=t.int64, device=D.device())
    grouped = t.empty(n, dtype=keys_dev.dtype, device=D.device())
    order = t.empty(n, dtype=t.int32, device=D.device()) if want_order else None
    ws = D.workspace(_lib.load().hg_reorganize_workspace_size(n, shards))
    _lib.call("hg_reorganize", D.ptr(keys_dev), n, key_bits, kind, seed, hash_range, bin_size, D.ptr(splits_dev),
              shards, D.ptr(rows), D.ptr(grouped), D.ptr(order), D.ptr(steps), D.ptr(ws), ws.numel(),
              D.stream_ptr())
    if keep_workspace:
        return rows, grouped, order, ws
    return rows, grouped, order


# --------------------------------------------------------------------------- public API


def plan_partition(per_shard_inputs, hash_range: int, bins_g: int, family: HashFamily = HashFamily()) -> PartitionPlan:
    """Phase 1 as a standalone operation (multishard.py:266-291)."""
    shards = len(per_shard_inputs)
    if shards < 1:
        raise ConfigError("need at least one shard input")
    if hash_range < 1:
        raise ConfigError(f"hash range must be >= 1, got {hash_range}")
    if bins_g < shards:
        raise ConfigError(f"bins_g={bins_g} is less than shard count {shards}")
    bin_size = -(-hash_range // bins_g)
    arrays = _inputs_to_device(per_shard_inputs)
    total = sum(a.numel() for a in arrays)
    counts = bin_histogram_device(arrays, hash_range, bins_g, bin_size, family)
    splits = split_plan_device(counts, bins_g, total, shards)
    return PartitionPlan(shards, hash_range, bins_g, bin_size, splits.cpu().numpy())


def reorganize(shard_keys, plan: PartitionPlan, family: HashFamily = HashFamily()) -> SendBuffers:
    """Phase 2 as a standalone operation: stable per-destination CSR (multishard.py:313-318)."""
    (dk,) = _inputs_to_device([shard_keys])
    rows, grouped, _ = reorganize_device(dk, plan.hash_range, plan.bin_size, plan.splits_device(), plan.shards,
                                         family)
    return SendBuffers(None, None, _device=(rows, grouped, rows.cpu().numpy()))


def exchange(fabric: ExchangeFabric, all_buffers) -> list:
    """Phase 3 as a standalone operation (multishard.py:321-333)."""
    if len(all_buffers) != fabric.shards:
        raise ConfigError(f"expected {fabric.shards} send buffers, got {len(all_buffers)}")
    for s, sb in enumerate(all_buffers):
        fabric.post(s, sb)
    received = [fabric.gather(d) for d in range(fabric.shards)]
    total_sent = sum(len(sb.keys) for sb in all_buffers)
    assert total_sent == sum(len(r) for r in received), "exchange lost or duplicated keys"
    return received


# Phase 3 between shards of one device is one concatenation; the per-row copy
# path that runs between GPUs can be forced on one GPU (tests).
_EXCHANGE_BY_ROWS = False


def shard_devices(shards: int, devices=None) -> list:
    """The CUDA device of every shard.

    `devices=None` places shard d on GPU d when the process sees exactly
    `shards` GPUs (more than one), the analogue of the reference's one thread
    per shard (multishard.py:414-419) on real hardware; otherwise every shard
    is a virtual shard on the current GPU.  An explicit list (ints or
    torch.device, one per shard, repeats allowed) overrides that."""
    t = D.torch()
    cur = t.cuda.current_device()
    if devices is None:
        n = t.cuda.device_count()
        return list(range(shards)) if shards > 1 and n == shards else [cur] * shards
    out = []
    for d in devices:
        idx = d.index if isinstance(d, t.device) else int(d)
        if idx is None:
            idx = cur
        if not 0 <= idx < t.cuda.device_count():
            raise ConfigError(f"device {d!r} is not a visible CUDA device")
        out.append(idx)
    if len(out) != shards:
        raise ConfigError(f"got {len(out)} devices for {shards} shards")
    return out


def build_sharded(per_shard_inputs, config: ShardConfig, key_bits: int = 32, devices=None):
    """The four-phase build (multishard.py:336-471), one shard per GPU or as
    virtual shards of one GPU (see `shard_devices`).

    All shards are driven from this host thread; every phase is enqueued on
    the shards' devices (their current streams).

    * Virtual shards (one device): the shard inputs are concatenated once and
      Phases 1-3 are ONE histogram, one split and ONE stable reorganize over
      the concatenation -- its row d is exactly the exchange's gather(d)
      (senders ascending, each in input order), so the exchange is a view.
    * One shard per GPU: per-device histograms summed on shard 0's device,
      the plan copied to every device, a stable reorganize per sender, and
      each sender's row copied straight into the owner's receive buffer
      (device-to-device over NVLink/NVSwitch with peer access, ordered after
      the sender's Phase 2 and before the owner's Phase 4 by stream events).

    Then a local build per shard with V_d = ceil(N_d / C).  The only host
    sync is the send-row matrix the receive buffers are sized from.  Like
    the reference (whose clock starts after input coercion, multishard.py:
    348, 414), `total_time_ns` starts once the inputs are on the devices.

    Returns (ShardedHashGraph, PhaseReport)."""
    p = config.shards
    if len(per_shard_inputs) != p:
        raise ConfigError(f"got {len(per_shard_inputs)} shard inputs for {p} shards")
    t = D.require_cuda()
    devs = shard_devices(p, devices)
    if len(set(devs)) == 1 and not _EXCHANGE_BY_ROWS:
        return _build_sharded_one_device(per_shard_inputs, config, key_bits, devs[0])
    return _build_sharded_devices(per_shard_inputs, config, key_bits, devs)


def _report(config, n, hr, bins_g, phase_ns, search_steps, keys_moved, bytes_moved, received_counts, total_ns):
    assert keys_moved == n, "exchange conservation violated"
    passes = {name: n for name in PASS_NAMES}
    phases = {
        "partition": PhaseStats(time_ns=phase_ns[0], keys_touched=2 * n),
        "preprocess": PhaseStats(time_ns=phase_ns[1], keys_touched=2 * n, search_steps=search_steps),
        "all_to_all": PhaseStats(time_ns=phase_ns[2], keys_touched=n, bytes_exchanged=bytes_moved),
        "table_construction": PhaseStats(time_ns=phase_ns[3], keys_touched=3 * n),
    }
    return PhaseReport(
        shards=config.shards, total_keys=n, hash_range=hr, bins_g=bins_g, load_factor=config.load_factor,
        family=config.family, phases=phases, passes=passes, search_steps=search_steps,
        bytes_exchanged=bytes_moved, shard_received_counts=received_counts, total_time_ns=total_ns,
        build_throughput=(n / (total_ns / 1e9)) if (n and total_ns) else 0.0,
    )


def _local_tables(received, config, key_bits):
    """Phase 4 (multishard.py:403-409): one local build per shard with its
    own range V_d = ceil(N_d / C).  Virtual shards sharing one GPU reuse one
    workspace and call the library directly: a 2^20-key shard builds in tens
    of microseconds, so per-call host overhead is what a loop over shards
    would otherwise spend."""
    t = D.torch()
    devs = {r.device for r in received}
    if len(received) > 1 and len(devs) == 1:
        lib = _lib.load()
        kind, seed = family_code(config.family)
        dev = next(iter(devs))
        with D.on(dev):
            vds = [hash_range_for(r.numel(), config.load_factor) for r in received]
            ws = D.workspace(max(lib.hg_build_workspace_size(r.numel(), v, key_bits) for r, v in zip(received, vds)))
            stream = D.stream_ptr()
            tables = []
            for r, v_d in zip(received, vds):
                off = t.empty(v_d + 1, dtype=t.int32, device=dev)
                edges = t.empty(r.numel(), dtype=r.dtype, device=dev)
                _lib.call("hg_build", r.data_ptr(), r.numel(), key_bits, kind, seed, v_d, off.data_ptr(),
                          edges.data_ptr(), None, ws.data_ptr(), ws.numel(), stream)
                tables.append(HashGraph(off, edges, v_d, config.family, float(config.load_factor), key_bits,
                                        r.numel()))
        return tables
    tables = []
    for r in received:
        v_d = hash_range_for(r.numel(), config.load_factor)
        off, edges, _ = build_device(r, v_d, config.family, key_bits)  # on r's device
        tables.append(HashGraph(off, edges, v_d, config.family, float(config.load_factor), key_bits, r.numel()))
    return tables


def _concat_inputs(per_shard_inputs, key_bits):
    """The shard inputs as one contiguous device array (one H2D for host inputs)."""
    t = D.torch()
    if all(D.is_cuda_tensor(k) for k in per_shard_inputs):
        parts = _inputs_to_device(per_shard_inputs, key_bits)
        sizes = [a.numel() for a in parts]
        flat = t.cat(parts) if len(parts) > 1 else parts[0]
        return flat, sizes
    host = []
    for k in per_shard_inputs:
        if D.is_tensor(k):
            k = D.to_numpy_keys(k, key_bits) if k.is_cuda else k.numpy().view(D.np_key_dtype(key_bits))
        host.append(D.coerce_host_keys(k, key_bits))
    sizes = [len(a) for a in host]
    flat = np.concatenate(host) if len(host) > 1 else host[0]
    return D.to_device_keys(flat, key_bits), sizes


def _build_sharded_one_device(per_shard_inputs, config, key_bits, dev):
    t = D.torch()
    p = config.shards
    with D.on(dev):
        flat, sizes = _concat_inputs(per_shard_inputs, key_bits)
        n = flat.numel()
        hr, bins_g, bin_size = config.resolve(n)
        t.cuda.current_stream().synchronize()  # inputs resident (the host->device copy is asynchronous) before the clock
        wall0 = time.perf_counter_ns()
        ev = [t.cuda.Event(enable_timing=True) for _ in range(4)]
        steps = t.zeros(1, dtype=t.int64, device=D.device())
        ev[0].record()
        counts = bin_histogram_device([flat], hr, bins_g, bin_size, config.family, key_bits)
        splits = split_plan_device(counts, bins_g, n, p)
        ev[1].record()
        rows, grouped, _ = reorganize_device(flat, hr, bin_size, splits, p, config.family, key_bits, steps=steps)
        ev[2].record()
        rows_host = rows.cpu().numpy()  # the one host sync: the local ranges
        received = [grouped[int(rows_host[d]):int(rows_host[d + 1])] for d in range(p)]  # gather(d), as views
        tables = _local_tables(received, config, key_bits)
        ev[3].record()
        ev[3].synchronize()
        total_ns = time.perf_counter_ns() - wall0
        splits_host = splits.cpu().numpy()
        search_steps = int(steps.cpu().item())

    def ns(a, b):
        return int(a.elapsed_time(b) * 1e6)

    received_counts = [int(r.numel()) for r in received]
    plan = PartitionPlan(p, hr, bins_g, bin_size, splits_host)
    table = ShardedHashGraph(plan, tables, config.family, received_counts)
    # the exchange is the reorganize's row layout itself: no device time of its own
    phase_ns = [ns(ev[0], ev[1]), ns(ev[1], ev[2]), 0, ns(ev[2], ev[3])]
    report = _report(config, n, hr, bins_g, phase_ns, search_steps, n, (key_bits // 8) * n, received_counts,
                     total_ns)
    return table, report


def _build_sharded_devices(per_shard_inputs, config, key_bits, devs):
    t = D.torch()
    p = config.shards
    distinct = sorted(set(devs))
    home = devs[0]
    arrays = []
    for d, k in zip(devs, per_shard_inputs):
        with D.on(d):
            arrays.append(_inputs_to_device([k], key_bits)[0])
    n = sum(a.numel() for a in arrays)
    hr, bins_g, bin_size = config.resolve(n)
    for d in distinct:  # inputs resident before the clock starts (reference: after coercion)
        t.cuda.synchronize(d)
    wall0 = time.perf_counter_ns()

    def events():
        out = {}
        for d in distinct:
            with D.on(d):
                out[d] = t.cuda.Event(enable_timing=True)
        return out

    ev = [events() for _ in range(5)]

    def mark(k):
        for d in distinct:
            with D.on(d):
                ev[k][d].record()

    mark(0)
    # Phase 1: one histogram per device, summed on the home device; the plan
    # is computed there and copied to every device
    counts = {}
    for d, a in zip(devs, arrays):
        with D.on(d):
            counts[d] = bin_histogram_device([a], hr, bins_g, bin_size, config.family, key_bits, counts.get(d))
    with D.on(home):
        total = counts[home]
        for d in distinct:
            if d != home:
                total = total + counts[d].to(home)
        splits_home = split_plan_device(total, bins_g, n, p)
    splits = {d: (splits_home if d == home else splits_home.to(d)) for d in distinct}
    mark(1)
    # Phase 2: stable per-destination rows on each sender's device
    steps = {}
    sends = []
    for d, a in zip(devs, arrays):
        with D.on(d):
            if d not in steps:
                steps[d] = t.zeros(1, dtype=t.int64, device=D.device())
            sends.append(reorganize_device(a, hr, bin_size, splits[d], p, config.family, key_bits,
                                           steps=steps[d])[:2])
    mark(2)
    # one host sync: row sizes decide the receive buffers
    rows_host = np.stack([r.cpu().numpy() for r, _ in sends])
    fabric = ExchangeFabric(p)
    for s_, (rows, grouped) in enumerate(sends):
        fabric.post(s_, SendBuffers(None, None, key_bits=key_bits, _device=(rows, grouped, rows_host[s_])))
    ev3 = events()
    for d in distinct:
        with D.on(d):
            ev3[d].record()
    # Phase 3: owner j receives row j of every sender, ascending sender order
    received = []
    for j, dj in enumerate(devs):
        with D.on(dj):
            sizes = rows_host[:, j + 1] - rows_host[:, j]
            recv = t.empty(int(sizes.sum()), dtype=D.storage_dtype(key_bits), device=D.device())
            o = 0
            for s_ in range(p):
                m = int(sizes[s_])
                if m:
                    recv[o:o + m].copy_(fabric.posted[s_].row_device(j), non_blocking=True)
                o += m
            fabric.keys_moved += int(sizes.sum())
            fabric.bytes_moved += (key_bits // 8) * int(sizes.sum())
            received.append(recv)
    mark(3)
    # Phase 4: local build on each owner's device
    tables = _local_tables(received, config, key_bits)
    mark(4)
    for d in distinct:
        ev[4][d].synchronize()
    total_ns = time.perf_counter_ns() - wall0
    plan = PartitionPlan(p, hr, bins_g, bin_size, splits_home.cpu().numpy())
    received_counts = [int(r.numel()) for r in received]
    search_steps = sum(int(x.cpu().item()) for x in steps.values())

    def ns(a, b):  # a phase's device time: the mean over the shards' devices (multishard.py:436-447)
        return int(np.mean([a[d].elapsed_time(b[d]) for d in distinct]) * 1e6)

    phase_ns = [ns(ev[0], ev[1]), ns(ev[1], ev[2]), ns(ev3, ev[3]), ns(ev[3], ev[4])]
    table = ShardedHashGraph(plan, tables, config.family, received_counts)
    report = _report(config, n, hr, bins_g, phase_ns, search_steps, fabric.keys_moved, fabric.bytes_moved,
                     received_counts, total_ns)
    return table, report


def query_sharded(table: ShardedHashGraph, queries, worker_count: int = 1) -> QueryResult:
    """Count each query key's occurrences across all shards (multishard.py:474-482)."""
    result, _ = _query_sharded(table, queries, worker_count, timed=False)
    return result


def query_sharded_timed(table: ShardedHashGraph, queries, worker_count: int = 1):
    """query_sharded() plus the routing+build vs intersect split (multishard.py:485-542)."""
    return _query_sharded(table, queries, worker_count, timed=True)


def _query_sharded(table: ShardedHashGraph, queries, worker_count: int, timed: bool):
    """Queries are routed on shard 0's device with the table's plan (stable
    rows), each row is answered on its shard's device into its slice of one
    grouped answer array, and hg_reorganize_gather returns the answers to
    input order there (recomputing each query's row slot, coalesced stores)."""
    if worker_count < 1:
        raise ConfigError(f"worker count must be >= 1, got {worker_count}")
    t = D.require_cuda()
    plan = table.plan
    p = plan.shards
    key_bits = table.shards[0].key_bits if table.shards else 32
    home = table.shards[0].keys_device.device if table.shards else D.device()
    with D.on(home):
        (q,) = _inputs_to_device([queries], key_bits)
        nq = q.numel()
        ev = [t.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        splits_dev = plan.splits_device()
        rows, grouped, _, rws = reorganize_device(q, plan.hash_range, plan.bin_size, splits_dev, p, table.family,
                                                  key_bits, keep_workspace=True)
        rows_h = rows.cpu().numpy()
        mult = t.zeros(nq, dtype=t.int32, device=D.device())
        answers = t.zeros(nq + 4, dtype=t.int32, device=D.device())  # grouped (row) order
        agg = t.zeros(3, dtype=t.int64, device=D.device())
        hash_values = 0
        ev[1].record()
        for d, shard in enumerate(table.shards):
            lo, hi = int(rows_h[d]), int(rows_h[d + 1])
            hash_values += shard.hash_range
            if hi == lo:
                continue
            m_d, a_d = query_device(shard, grouped[lo:hi])  # on the shard's device
            if m_d.device != mult.device:
                m_d, a_d = m_d.to(mult.device), a_d.to(mult.device)
            answers[lo:hi].copy_(m_d)
            agg += a_d
        if nq:
            kind, seed = family_code(table.family)
            _lib.call("hg_reorganize_gather", D.ptr(q), nq, key_bits, kind, seed, plan.hash_range, plan.bin_size,
                      D.ptr(splits_dev), p, D.ptr(rows), D.ptr(answers), D.ptr(mult), D.ptr(rws), rws.numel(),
                      D.stream_ptr())
        ev[2].record()
    result = QueryResult(mult, agg, hash_values)
    if not timed:
        return result, None
    ev[2].synchronize()
    times = QueryStageTimes(int(ev[0].elapsed_time(ev[1]) * 1e6), int(ev[1].elapsed_time(ev[2]) * 1e6))
    return result, times


def work_audit(report: PhaseReport, total_keys: int, shards: int) -> AuditVerdict:
    """Counted work against the linear-cost model (multishard.py:545-563)."""
    violations = []
    bound = total_keys * shards
    if report.search_steps > bound:
        violations.append(f"dest_search steps {report.search_steps} exceed N*P = {bound}")
    for name in PASS_NAMES:
        touched = report.passes.get(name)
        if touched is None:
            violations.append(f"missing pass counter {name!r}")
        elif name != "dest_search" and touched > total_keys:
            violations.append(f"pass {name!r} touched {touched} keys, bound is N = {total_keys}")
    return AuditVerdict(ok=not violations, violations=violations)
