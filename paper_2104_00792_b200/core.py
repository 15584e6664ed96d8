"""Single-shard table: the CSR HashGraph built on the GPU (mirrors core.py of the reference).

`HashGraph` keeps its arrays in HBM (`offset_device` uint32[V+1],
`keys_device` uint32/uint64[N]); the reference-facing attributes `offset`
(int64[V+1]) and `keys` are read-only numpy copies materialised on first
access, so code written against the reference keeps working unchanged.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .errors import ConfigError, SnapshotFormatError
from .hashing import HashFamily, HashKind, family_code, hash_key, hash_range_for

MASK32 = 0xFFFFFFFF


@dataclass(frozen=True)
class Bucket:
    """Read-only view of the keys stored under one hash value (core.py:34-42)."""

    hash_value: int
    entries: np.ndarray

    def __len__(self) -> int:
        return len(self.entries)


@dataclass(frozen=True)
class BuildCounters:
    """Keys touched by each build pass (core.py:45-55)."""

    hashed: int
    counted: int
    placed: int

    @property
    def total(self) -> int:
        return self.hashed + self.counted + self.placed


class HashGraph:
    """The CSR pair plus the parameters that produced it; immutable (core.py:58-81)."""

    __slots__ = ("offset_device", "keys_device", "hash_range", "family", "load_factor", "key_bits",
                 "_num_keys", "_offset", "_keys", "_frozen", "_trace")

    def __init__(self, offset_device, keys_device, hash_range: int, family, load_factor: float,
                 key_bits: int = 32, num_keys: int | None = None):
        object.__setattr__(self, "offset_device", offset_device)
        object.__setattr__(self, "keys_device", keys_device)
        object.__setattr__(self, "hash_range", int(hash_range))
        object.__setattr__(self, "family", family)
        object.__setattr__(self, "load_factor", float(load_factor))
        object.__setattr__(self, "key_bits", int(key_bits))
        object.__setattr__(self, "_num_keys", int(keys_device.numel() if num_keys is None else num_keys))
        object.__setattr__(self, "_offset", None)
        object.__setattr__(self, "_keys", None)
        object.__setattr__(self, "_trace", None)  # QueryTableTrace of a build_query_table table
        object.__setattr__(self, "_frozen", True)

    def __setattr__(self, name, value):
        raise AttributeError(f"HashGraph is immutable (cannot set {name!r})")

    @property
    def num_keys(self) -> int:
        return self._num_keys

    @property
    def offset(self) -> np.ndarray:
        if self._offset is None:
            object.__setattr__(self, "_offset", D.frozen(D.widen_u32_to_numpy(self.offset_device)))
        return self._offset

    @property
    def keys(self) -> np.ndarray:
        if self._keys is None:
            object.__setattr__(self, "_keys", D.frozen(D.to_numpy_keys(self.keys_device, self.key_bits)))
        return self._keys

    def bucket(self, h: int) -> Bucket:
        if not 0 <= h < self.hash_range:
            raise IndexError(f"hash value {h} outside [0, {self.hash_range})")
        lo, hi = (int(x) for x in self.offset_device[h:h + 2].cpu().numpy().view(np.uint32))
        entries = D.to_numpy_keys(self.keys_device[lo:hi], self.key_bits)
        return Bucket(h, D.frozen(entries))

    def contains(self, key: int) -> int:
        """Number of occurrences of `key` in the table (0 when absent)."""
        h = hash_key(self.family, key, self.hash_range, self.key_bits)
        entries = self.bucket(h).entries
        mask = MASK32 if self.key_bits == 32 else (1 << 64) - 1
        return int(np.count_nonzero(entries == entries.dtype.type(key & mask)))

    def __repr__(self) -> str:
        return (f"HashGraph(num_keys={self.num_keys}, hash_range={self.hash_range}, family={self.family!r}, "
                f"load_factor={self.load_factor}, key_bits={self.key_bits}, device={self.keys_device.device})")


def as_device_table(table) -> HashGraph:
    """Accept our HashGraph or any reference-shaped table (offset/keys numpy)."""
    if isinstance(table, HashGraph):
        return table
    D.require_cuda()
    offset = np.asarray(table.offset, dtype=np.int64)
    keys = np.asarray(table.keys)
    key_bits = 64 if keys.dtype == np.uint64 else 32
    if offset[-1] >= 1 << 32:
        raise ConfigError("device tables hold fewer than 2^32 keys")
    off_dev = D.torch().from_numpy(offset.astype(np.uint32).view(np.int32)).to(D.device())
    keys_dev = D.to_device_keys(keys, key_bits)
    return HashGraph(off_dev, keys_dev, table.hash_range, table.family, table.load_factor, key_bits)


def _resolve_range(n: int, load_factor: float, hash_range) -> int:
    if hash_range is None:
        return hash_range_for(n, load_factor)
    if load_factor <= 0:
        raise ConfigError(f"load factor must be positive, got {load_factor}")
    if hash_range < 1:
        raise ConfigError(f"hash range must be >= 1, got {hash_range}")
    return int(hash_range)


def build_device(keys_dev, v: int, family, key_bits: int = 32, want_positions: bool = False, keep_trace: bool = False):
    """Launch the GPU build over device keys: (offset u32[v+1], edges, positions u32 | None).

    Enqueue-only on the current stream.  With positions the binned path runs
    traced (hg_build_traced_workspace_size); keep_trace also returns the
    workspace, which then holds the trace hg_intersect_tables reuses."""
    t = D.torch()
    n = keys_dev.numel()
    kind, seed = family_code(family)
    with D.on(keys_dev):  # the keys' device and its current stream
        offsets = t.empty(v + 1, dtype=t.int32, device=keys_dev.device)
        edges = t.empty(n, dtype=keys_dev.dtype, device=keys_dev.device)
        positions = t.empty(n, dtype=t.int32, device=keys_dev.device) if want_positions else None
        size = (_lib.load().hg_build_traced_workspace_size if want_positions else
                _lib.load().hg_build_workspace_size)(n, v, key_bits)
        ws = D.workspace(size)
        _lib.call("hg_build", D.ptr(keys_dev), n, key_bits, kind, seed, v, D.ptr(offsets), D.ptr(edges),
                  D.ptr(positions), D.ptr(ws), ws.numel(), D.stream_ptr())
    if keep_trace:
        return offsets, edges, positions, ws
    return offsets, edges, positions


def build(keys, load_factor: float = 1.0, family: HashFamily = HashFamily(), worker_count: int = 1,
          hash_range: int | None = None, key_bits: int = 32) -> HashGraph:
    """Build a table over `keys` on the GPU (core.py:164-180).

    `worker_count` is validated like the reference but has no effect: the
    parallelism is the GPU's.  `key_bits=64` builds over uint64 keys.
    """
    table, _, _ = _build(keys, load_factor, family, worker_count, hash_range, key_bits, False)
    return table


def build_traced(keys, load_factor: float = 1.0, family: HashFamily = HashFamily(), worker_count: int = 1,
                 hash_range: int | None = None, key_bits: int = 32):
    """build() plus counters and positions (core.py:183-209).

    positions[p] is the input index of the key stored at keys[p] (int64 numpy).
    """
    table, counters, pos = _build(keys, load_factor, family, worker_count, hash_range, key_bits, True)
    positions = D.widen_u32_to_numpy(pos) if pos is not None and pos.numel() else np.zeros(0, np.int64)
    return table, counters, positions


def _build(keys, load_factor, family, worker_count, hash_range, key_bits, want_positions, keep_trace=False):
    if key_bits not in (32, 64):
        raise ConfigError(f"key_bits must be 32 or 64, got {key_bits}")
    if not D.is_tensor(keys):
        keys = D.coerce_host_keys(keys, key_bits)  # validate shape before range checks
    if worker_count < 1:
        raise ConfigError(f"worker count must be >= 1, got {worker_count}")
    n = D.key_count(keys)
    v = _resolve_range(n, load_factor, hash_range)
    dk = D.to_device_keys(keys, key_bits)
    if keep_trace:
        offsets, edges, positions, trace = build_device(dk, v, family, key_bits, want_positions, True)
    else:
        offsets, edges, positions = build_device(dk, v, family, key_bits, want_positions)
        trace = None
    table = HashGraph(offsets, edges, v, family, float(load_factor), key_bits, n)
    counters = BuildCounters(hashed=n, counted=n, placed=n)
    if keep_trace:
        return table, counters, positions, trace
    return table, counters, positions


# ---------------------------------------------------------------- snapshots (core.py:27-28, 212-255)
#
# HGR1 is the reference's byte format: b"HGR1", header <QQBId (V, N, family
# kind, seed, load factor), offsets as u64 LE [V+1], keys as u32 LE [N].  A
# table over 64-bit keys is written as b"HGR8": the same header and offsets,
# keys as u64 LE (the reference has no 64-bit tables).
SNAPSHOT_MAGIC = {32: b"HGR1", 64: b"HGR8"}
SNAPSHOT_HEADER = struct.Struct("<QQBId")


def save_table(table, path) -> None:
    """Write a table snapshot (core.py:212-225); the device CSR is widened on the GPU."""
    t = as_device_table(table)
    kind, seed = family_code(t.family)
    with open(path, "wb") as f:
        f.write(SNAPSHOT_MAGIC[t.key_bits])
        f.write(SNAPSHOT_HEADER.pack(t.hash_range, t.num_keys, kind, seed, t.load_factor))
        f.write(np.ascontiguousarray(t.offset, dtype="<u8").tobytes())
        f.write(np.ascontiguousarray(t.keys, dtype="<u4" if t.key_bits == 32 else "<u8").tobytes())


def read_snapshot(path):
    """Parse and validate a snapshot on the host (core.py:228-255).

    Returns (hash_range, family, load_factor, key_bits, offset int64[V+1], keys).
    Raises SnapshotFormatError for a bad magic, a truncated header, an unknown
    hash family, a body of the wrong length or a corrupt offset array."""
    with open(path, "rb") as f:
        blob = f.read()
    bits = {m: b for b, m in SNAPSHOT_MAGIC.items()}.get(blob[:4])
    if bits is None:
        raise SnapshotFormatError(f"{path}: bad magic {blob[:4]!r}")
    hdr = SNAPSHOT_HEADER.size
    if len(blob) - 4 < hdr:
        raise SnapshotFormatError(f"{path}: truncated header")
    v, n, kind, seed, load_factor = SNAPSHOT_HEADER.unpack_from(blob, 4)
    try:
        family = HashFamily(HashKind(kind), seed)
    except ValueError as e:
        raise SnapshotFormatError(f"{path}: unknown hash family {kind}") from e
    kb = bits // 8
    if len(blob) - 4 != hdr + 8 * (v + 1) + kb * n:
        raise SnapshotFormatError(f"{path}: body is {len(blob) - 4} bytes, expected "
                                  f"{hdr + 8 * (v + 1) + kb * n} for V={v} N={n}")
    offset = np.frombuffer(blob, dtype="<u8", count=v + 1, offset=4 + hdr).astype(np.int64)
    keys = np.frombuffer(blob, dtype="<u4" if bits == 32 else "<u8", count=n, offset=4 + hdr + 8 * (v + 1))
    keys = keys.astype(np.uint32 if bits == 32 else np.uint64)
    if offset[0] != 0 or offset[-1] != n or (v > 0 and bool(np.any(offset[1:] < offset[:-1]))):
        raise SnapshotFormatError(f"{path}: corrupt offset array")
    return v, family, float(load_factor), bits, offset, keys


def load_table(path) -> HashGraph:
    """Read a snapshot into a device table (core.py:228-255)."""
    v, family, load_factor, bits, offset, keys = read_snapshot(path)
    D.require_cuda()
    if len(keys) >= 1 << 32:
        raise ConfigError("device tables hold fewer than 2^32 keys")
    off_dev = D.torch().from_numpy(offset.astype(np.uint32).view(np.int32)).to(D.device())
    return HashGraph(off_dev, D.to_device_keys(keys, bits), v, family, load_factor, bits)
