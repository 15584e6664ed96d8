"""Batch querying by table intersection on the GPU (mirrors query.py of the reference).

`intersect` runs the whole query (query-side table over the table's hash range
plus the per-bucket IntersectArray) in libhashgraph_b200 and returns a
`QueryResult` whose arrays stay in HBM until read: `multiplicities` (int64
numpy, positional) and the aggregate counters are materialised on first
access; `multiplicities_device` is the uint32 device array.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .core import Bucket, HashGraph, _build, as_device_table, build_device, build_traced
from .errors import ConfigError
from .hashing import family_code, same_family


class QueryResult:
    """Per-position multiplicities plus aggregate counters (query.py:30-38)."""

    __slots__ = ("multiplicities_device", "_agg_device", "hash_values", "_mult", "_agg", "_n")

    def __init__(self, multiplicities_device=None, agg_device=None, hash_values: int = 0, *,
                 multiplicities=None, matched_positions=None, total_matches=None, comparisons=None):
        self.multiplicities_device = multiplicities_device
        self._agg_device = agg_device
        self.hash_values = int(hash_values)
        self._mult = None if multiplicities is None else np.asarray(multiplicities, dtype=np.int64)
        self._agg = None
        if matched_positions is not None:
            self._agg = (int(matched_positions), int(total_matches), int(comparisons))
        self._n = (multiplicities_device.numel() if multiplicities_device is not None else len(self._mult))

    @property
    def multiplicities(self) -> np.ndarray:
        if self._mult is None:
            m = self.multiplicities_device
            self._mult = D.widen_u32_to_numpy(m) if m.numel() else np.zeros(0, np.int64)
        return self._mult

    def _aggregates(self):
        if self._agg is None:
            a = self._agg_device.cpu().numpy().view(np.uint64)
            self._agg = (int(a[0]), int(a[1]), int(a[2]))
        return self._agg

    @property
    def matched_positions(self) -> int:
        return self._aggregates()[0]

    @property
    def total_matches(self) -> int:
        return self._aggregates()[1]

    @property
    def comparisons(self) -> int:
        return self._aggregates()[2]

    def __len__(self) -> int:
        return self._n

    def __repr__(self) -> str:
        return f"QueryResult(n={self._n}, hash_values={self.hash_values})"


@dataclass(frozen=True)
class QueryStageTimes:
    """Device-time split of a query: query-table build vs intersect (query.py:41-50)."""

    table_build_ns: int
    intersect_ns: int

    @property
    def total_ns(self) -> int:
        return self.table_build_ns + self.intersect_ns


@dataclass(frozen=True)
class BucketIntersection:
    """Result of intersecting one bucket pair (query.py:53-59)."""

    counts: np.ndarray
    total_matches: int
    comparisons: int


def intersect_buckets(a: Bucket, b: Bucket) -> BucketIntersection:
    """Count, for each key in b, its occurrences in a (query.py:62-81).

    A per-bucket inspection helper over two host `Bucket` views (the reference
    uses it in tests); whole-table intersections run on the GPU.
    """
    if a.hash_value != b.hash_value:
        raise ConfigError(f"bucket hash values differ: {a.hash_value} != {b.hash_value}")
    ea, eb = np.asarray(a.entries), np.asarray(b.entries)
    srt = np.sort(ea)
    counts = (np.searchsorted(srt, eb, side="right") - np.searchsorted(srt, eb, side="left")).astype(np.int64)
    return BucketIntersection(counts, int(counts.sum()), len(ea) * len(eb))


class QueryTableTrace:
    """What intersect_tables needs to return counts to query order without a
    scatter: the traced build's workspace (hg_build_traced_workspace_size:
    both partition levels' position maps and every grouped key's slot), the
    device positions, and the host positions array handed to the caller
    (identity-checked, read-only)."""

    __slots__ = ("workspace", "positions_device", "positions_host")

    def __init__(self, workspace, positions_device, positions_host):
        self.workspace = workspace
        self.positions_device = positions_device
        self.positions_host = positions_host


def build_query_table(table, queries):
    """Query-side table with the input table's hash range (query.py:84-95).

    The build runs traced: the returned table keeps its trace (about 20 bytes
    per query key of device memory) so that intersect_tables(table, qt,
    positions) with these very positions streams the counts back to query
    order; positions is the usual read-only int64 array."""
    key_bits = getattr(table, "key_bits", 32)
    if key_bits not in (32, 64):
        raise ConfigError(f"key_bits must be 32 or 64, got {key_bits}")
    qt, _, pos, ws = _build(queries, 1.0, table.family, 1, table.hash_range, key_bits, True, keep_trace=True)
    positions = D.frozen(D.widen_u32_to_numpy(pos) if pos is not None and pos.numel() else np.zeros(0, np.int64))
    if pos is not None and pos.numel():
        object.__setattr__(qt, "_trace", QueryTableTrace(ws, pos, positions))
    return qt, positions


def _check_pair(table, query_table, worker_count):
    if query_table.hash_range != table.hash_range:
        raise ConfigError(f"hash ranges differ: {query_table.hash_range} != {table.hash_range}")
    if not same_family(query_table.family, table.family):
        raise ConfigError("hash families differ between table and query table")
    if worker_count < 1:
        raise ConfigError(f"worker count must be >= 1, got {worker_count}")
    if table.hash_range > 1 << 32:
        raise ConfigError(f"hash range {table.hash_range} exceeds the 2^32 intersection limit")


def intersect_tables(table, query_table, positions, worker_count: int = 1) -> QueryResult:
    """Intersect corresponding buckets of a prebuilt query table (query.py:120-179)."""
    _check_pair(table, query_table, worker_count)
    ta, tb = as_device_table(table), as_device_table(query_table)
    with D.on(ta.keys_device):
        return _intersect_tables_device(ta, tb, positions)


def _intersect_tables_device(ta, tb, positions):
    t = D.torch()
    trace = getattr(tb, "_trace", None)
    if trace is not None and positions is trace.positions_host:  # the positions build_query_table returned
        pos = trace.positions_device
    else:
        trace = None
        if D.is_cuda_tensor(positions):
            pos = positions.to(t.int32)
        else:
            pos = t.from_numpy(np.asarray(positions, dtype=np.int64).astype(np.uint32).view(np.int32)).to(D.device())
    nb = tb.num_keys
    mult = t.zeros(nb, dtype=t.int32, device=D.device())
    agg = t.zeros(3, dtype=t.int64, device=D.device())
    kind, seed = family_code(ta.family)
    ws = D.workspace(_lib.load().hg_intersect_tables_workspace_size(nb, ta.hash_range, ta.num_keys, ta.key_bits))
    tw = trace.workspace if trace is not None else None
    _lib.call("hg_intersect_tables", D.ptr(ta.offset_device), D.ptr(ta.keys_device), ta.num_keys,
              D.ptr(tb.offset_device), D.ptr(tb.keys_device), D.ptr(pos), nb, ta.key_bits, kind, seed, ta.hash_range,
              D.ptr(tw), tw.numel() if tw is not None else 0, D.ptr(mult), D.ptr(agg), D.ptr(ws),
              ws.numel(), D.stream_ptr())
    return QueryResult(mult, agg, ta.hash_range)


def query_device(table: HashGraph, queries_dev):
    """Enqueue the whole query on the current stream; returns (mult u32, agg u64[3])."""
    t = D.torch()
    q = queries_dev.numel()
    kind, seed = family_code(table.family)
    with D.on(table.keys_device):  # the table's device and its current stream
        if queries_dev.device != table.keys_device.device:
            queries_dev = queries_dev.to(table.keys_device.device)
        mult = t.empty(q, dtype=t.int32, device=queries_dev.device)
        agg = t.zeros(3, dtype=t.int64, device=queries_dev.device)
        ws = D.workspace(_lib.load().hg_query_workspace_size(q, table.hash_range, table.num_keys, table.key_bits))
        _lib.call("hg_query", D.ptr(table.offset_device), D.ptr(table.keys_device), table.num_keys,
                  D.ptr(queries_dev), q, table.key_bits, kind, seed, table.hash_range, D.ptr(mult), D.ptr(agg),
                  D.ptr(ws), ws.numel(), D.stream_ptr())
    return mult, agg


def _query_keys(table: HashGraph, queries):
    """Queries on the device at the table's key width.

    A 32-bit table refuses 64-bit queries that do not fit in 32 bits (a KEY8
    file or 64-bit workload against an HGR1 table): the reference's silent
    uint32 truncation (core.py:84-88) would report spurious matches for them.
    Narrower queries against a 64-bit table are widened (lossless)."""
    if table.key_bits == 32:
        wide = None
        if D.is_tensor(queries) and queries.element_size() == 8:
            wide = queries
        elif not D.is_tensor(queries):
            arr = np.asarray(queries)
            if arr.dtype.kind in "iu" and arr.dtype.itemsize == 8 and arr.size:
                lo, hi = int(arr.min()), int(arr.max())
                if lo < 0 or hi > 0xFFFFFFFF:
                    raise ConfigError("64-bit query keys do not fit the table's 32-bit keys (build the table "
                                      "with key_bits=64)")
        if wide is not None and wide.numel():
            t = D.torch()
            w = wide.view(t.int64) if wide.dtype != t.int64 else wide
            if bool(((w < 0) | (w > 0xFFFFFFFF)).any()):
                raise ConfigError("64-bit query keys do not fit the table's 32-bit keys (build the table "
                                  "with key_bits=64)")
    return D.to_device_keys(queries, table.key_bits)


def intersect(table, queries, worker_count: int = 1) -> QueryResult:
    """Count each query key's occurrences in the table (query.py:182-190)."""
    if worker_count < 1:
        raise ConfigError(f"worker count must be >= 1, got {worker_count}")
    ta = as_device_table(table)
    if ta.hash_range > 1 << 32:
        raise ConfigError(f"hash range {ta.hash_range} exceeds the 2^32 intersection limit")
    with D.on(ta.keys_device):
        qd = _query_keys(ta, queries)
        mult, agg = query_device(ta, qd)
    return QueryResult(mult, agg, ta.hash_range)


def intersect_timed(table, queries, worker_count: int = 1):
    """intersect() plus the build-vs-intersect split, in device nanoseconds (query.py:193-202).

    Runs the same fused query as intersect(); the library records a split
    event once the query-side table (the binned grouping of the queries) is
    complete, so table_build_ns covers that and intersect_ns the probe and the
    return to query order."""
    if worker_count < 1:
        raise ConfigError(f"worker count must be >= 1, got {worker_count}")
    D.require_cuda()
    ta = as_device_table(table)
    if ta.hash_range > 1 << 32:
        raise ConfigError(f"hash range {ta.hash_range} exceeds the 2^32 intersection limit")
    with D.on(ta.keys_device):
        return _intersect_timed_device(ta, queries)


def _intersect_timed_device(ta, queries):
    t = D.torch()
    qd = _query_keys(ta, queries)
    nb = qd.numel()
    mult = t.zeros(nb, dtype=t.int32, device=qd.device)
    agg = t.zeros(3, dtype=t.int64, device=qd.device)
    kind, seed = family_code(ta.family)
    ws = D.workspace(_lib.load().hg_query_workspace_size(nb, ta.hash_range, ta.num_keys, ta.key_bits))
    ev = [t.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[1].record()  # creates the split event; the library re-records it at the split point
    ev[0].record()
    _lib.call("hg_query_timed", D.ptr(ta.offset_device), D.ptr(ta.keys_device), ta.num_keys, D.ptr(qd), nb,
              ta.key_bits, kind, seed, ta.hash_range, D.ptr(mult), D.ptr(agg), D.ptr(ws), ws.numel(),
              ev[1].cuda_event, D.stream_ptr())
    ev[2].record()
    ev[2].synchronize()
    build_ns = int(ev[0].elapsed_time(ev[1]) * 1e6) if nb else 0
    inter_ns = int(ev[1].elapsed_time(ev[2]) * 1e6) if nb else 0
    return QueryResult(mult, agg, ta.hash_range), QueryStageTimes(build_ns, inter_ns)
