"""numpy restatement of the reference HashGraph hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference `file:line` (relative to
/root/reference/pkg/src/hashgraph/) whose behaviour it restates.  The code is a
fresh transcription of the algorithm, written as free functions over plain
numpy arrays (no dataclasses), so tests can compare the CUDA product path
against it array by array.

Width extension: `key_bits=64` restates the same algorithm over uint64 keys
with the 64-bit Murmur3 finalizer (fmix64).  The reference truncates keys to
uint32 (`core.py:84-88`), so the 64-bit mode is *parity unpinned*: it is only
pinned through its structural properties and its agreement with the 32-bit
mode's algorithm.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "M32",
    "KIND_MURMUR",
    "KIND_IDENTITY",
    "fmix32_scalar",
    "fmix64_scalar",
    "hash_scalar",
    "hash_keys",
    "hash_range_for",
    "coerce_keys",
    "build_csr",
    "default_workers",
    "canonical",
    "intersect_csr",
    "query",
    "count_occurrences",
    "resolve_shards",
    "splits_from_bins",
    "bin_histogram",
    "plan_splits",
    "dest_of_hash",
    "reorganize",
    "exchange_rows",
    "build_sharded",
    "query_sharded",
    "splitmix64_at",
    "generate_keys",
]

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
KIND_MURMUR = 0  # hashing.py:31-35 (HashKind.MURMUR32 = 0)
KIND_IDENTITY = 1  # hashing.py:31-35 (HashKind.IDENTITY = 1)

_C1, _C2 = 0x85EBCA6B, 0xC2B2AE35  # hashing.py:27-28
_D1, _D2 = 0xFF51AFD7ED558CCD, 0xC4CEB9FE1A85EC53  # Murmur3 fmix64 (extension)


# --------------------------------------------------------------------------- hashing


def fmix32_scalar(x: int) -> int:
    """hashing.py:77-85 -- 32-bit avalanche cascade with wrapping multiplies."""
    x &= M32
    x = (x ^ (x >> 16)) & M32
    x = (x * _C1) & M32
    x ^= x >> 13
    x = (x * _C2) & M32
    return x ^ (x >> 16)


def fmix64_scalar(x: int) -> int:
    """64-bit extension of hashing.py:77-85 (Murmur3 fmix64)."""
    x &= M64
    x ^= x >> 33
    x = (x * _D1) & M64
    x ^= x >> 33
    x = (x * _D2) & M64
    return x ^ (x >> 33)


def hash_scalar(kind: int, seed: int, key: int, v: int, key_bits: int = 32) -> int:
    """hashing.py:88-95 -- one key into [0, v)."""
    if v < 1:
        raise ValueError("hash range must be >= 1")
    if key_bits == 32:
        key &= M32
        mixed = key if kind == KIND_IDENTITY else fmix32_scalar(key ^ seed)
    else:
        key &= M64
        mixed = key if kind == KIND_IDENTITY else fmix64_scalar(key ^ seed)
    return mixed % v


def hash_keys(kind: int, seed: int, keys: np.ndarray, v: int) -> np.ndarray:
    """hashing.py:98-114 -- vectorised hash; int64 values in [0, v).

    uint32 input follows the reference bit for bit; uint64 input uses fmix64.
    """
    if v < 1:
        raise ValueError("hash range must be >= 1")
    keys = np.asarray(keys)
    if keys.dtype == np.uint64:
        x = keys.copy()
        if kind != KIND_IDENTITY:
            x ^= np.uint64(seed)
            x ^= x >> np.uint64(33)
            x *= np.uint64(_D1)
            x ^= x >> np.uint64(33)
            x *= np.uint64(_D2)
            x ^= x >> np.uint64(33)
        return (x % np.uint64(v)).astype(np.int64) if v < (1 << 64) else x.astype(np.int64)
    x = keys.astype(np.uint32, copy=True)
    if kind != KIND_IDENTITY:
        x ^= np.uint32(seed)
        x ^= x >> np.uint32(16)
        x *= np.uint32(_C1)
        x ^= x >> np.uint32(13)
        x *= np.uint32(_C2)
        x ^= x >> np.uint32(16)
    return (x.astype(np.uint64) % np.uint64(min(v, 1 << 63))).astype(np.int64)


def hash_range_for(count: int, load_factor: float) -> int:
    """hashing.py:62-74 -- max(1, ceil(count / load_factor)) in float64."""
    if load_factor <= 0:
        raise ValueError("load factor must be positive")
    if count < 0:
        raise ValueError("key count must be non-negative")
    raw = count / load_factor
    if not math.isfinite(raw) or raw > 1 << 62:
        raise ValueError("hash range overflows")
    return max(1, math.ceil(raw))


def coerce_keys(keys, key_bits: int = 32) -> np.ndarray:
    """core.py:84-88 -- contiguous 1-D key array (uint32 truncation for 32-bit)."""
    arr = np.ascontiguousarray(np.asarray(keys, dtype=np.uint32 if key_bits == 32 else np.uint64))
    if arr.ndim != 1:
        raise ValueError("keys must be one-dimensional")
    return arr


# --------------------------------------------------------------------------- build


def _chunks(n: int, workers: int):
    """core.py:91-93 -- ceil(n / workers)-sized contiguous chunks."""
    step = -(-n // workers)
    return [(lo, min(lo + step, n)) for lo in range(0, n, step)] if n else []


def build_csr(keys: np.ndarray, v: int, kind: int = KIND_MURMUR, seed: int = 0, workers: int = 1):
    """core.py:148-155 (+ _place_serial 96-101, _place_parallel 104-145).

    Returns (offset int64[v+1], placed keys, positions int64[N]).  Placement is
    stable: inside a bucket keys keep input order, whichever branch runs (the
    reference's parallel branch reproduces the serial arrays exactly).
    """
    n = len(keys)
    h = hash_keys(kind, seed, keys, v) if n else np.empty(0, np.int64)
    offset = np.zeros(v + 1, dtype=np.int64)
    if workers <= 1 or n < (1 << 14):  # core.py:31, :150
        np.cumsum(np.bincount(h, minlength=v), out=offset[1:])
        order = np.argsort(h, kind="stable")
        return offset, keys[order], order.astype(np.int64)

    bounds = _chunks(n, workers)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        per_chunk = list(pool.map(lambda b: np.bincount(h[b[0]:b[1]], minlength=v), bounds))
        np.cumsum(np.sum(per_chunk, axis=0), out=offset[1:])
        placed = np.empty(n, dtype=keys.dtype)
        positions = np.empty(n, dtype=np.int64)
        bases, run = [], offset[:v].copy()
        for c in per_chunk:
            bases.append(run)
            run = run + c

        def place(job):
            (lo, hi), base = job
            hh = h[lo:hi]
            o = np.argsort(hh, kind="stable")
            sh = hh[o]
            rank = np.arange(hi - lo, dtype=np.int64) - np.searchsorted(sh, sh, side="left")
            slots = base[sh] + rank
            placed[slots] = keys[lo:hi][o]
            positions[slots] = o + lo

        list(pool.map(place, zip(bounds, bases)))
    return offset, placed, positions


def canonical(offset: np.ndarray, keys: np.ndarray):
    """test_acceptance.py:44-51 -- offsets plus bucket-sorted payload.

    Two tables are equal under the north-star rule iff both arrays are equal.
    Works for 32- and 64-bit keys (lexicographic (bucket, key) order).
    """
    offset = np.asarray(offset, dtype=np.int64)
    keys = np.asarray(keys)
    owner = np.repeat(np.arange(len(offset) - 1, dtype=np.int64), np.diff(offset))
    order = np.lexsort((keys, owner))
    return offset, keys[order]


# --------------------------------------------------------------------------- query


def intersect_csr(offset_a, keys_a, offset_b, keys_b, positions_b, workers: int = 1):
    """query.py:120-179 (+ _bucket_ids 98-99, _count_slice 102-117).

    For every query-table slot, the number of equal keys in the same bucket of
    the table, scattered back to query order through `positions_b`.  Returns
    (multiplicities int64[Q], matched_positions, total_matches, comparisons,
    hash_values).
    """
    v = len(offset_a) - 1
    if len(offset_b) - 1 != v:
        raise ValueError("hash ranges differ")
    deg_a, deg_b = np.diff(offset_a), np.diff(offset_b)
    owner_a = np.repeat(np.arange(v, dtype=np.int64), deg_a)
    owner_b = np.repeat(np.arange(v, dtype=np.int64), deg_b)
    keys_a = np.asarray(keys_a)
    keys_b = np.asarray(keys_b)
    if keys_a.dtype == np.uint64 or keys_b.dtype == np.uint64:
        # lexicographic (bucket, key) rank via a structured view
        ka = np.rec.fromarrays([owner_a, keys_a.astype(np.uint64)], names="b,k")
        kb = np.rec.fromarrays([owner_b, keys_b.astype(np.uint64)], names="b,k")
        ka = np.sort(ka, order=("b", "k"))
        counts = np.searchsorted(ka, kb, side="right") - np.searchsorted(ka, kb, side="left")
    else:
        comp_a = (owner_a.astype(np.uint64) << np.uint64(32)) | keys_a.astype(np.uint64)
        comp_a.sort()
        comp_b = (owner_b.astype(np.uint64) << np.uint64(32)) | keys_b.astype(np.uint64)

        def count(lo_hi):
            lo, hi = lo_hi
            a = comp_a[offset_a[lo]:offset_a[hi]]
            b = comp_b[offset_b[lo]:offset_b[hi]]
            return np.searchsorted(a, b, side="right") - np.searchsorted(a, b, side="left")

        w = max(1, min(workers, v))
        cuts = np.linspace(0, v, w + 1, dtype=np.int64)
        jobs = [(int(cuts[i]), int(cuts[i + 1])) for i in range(w) if cuts[i] < cuts[i + 1]]
        if len(jobs) > 1:
            with ThreadPoolExecutor(max_workers=len(jobs)) as pool:
                counts = np.concatenate(list(pool.map(count, jobs)))
        else:
            counts = count(jobs[0]) if jobs else np.zeros(0, np.int64)
    mult = np.zeros(len(keys_b), dtype=np.int64)
    mult[np.asarray(positions_b, dtype=np.int64)] = counts
    comparisons = int(np.dot(deg_a.astype(np.int64), deg_b.astype(np.int64)))
    return mult, int(np.count_nonzero(mult)), int(mult.sum()), comparisons, v


def query(offset_a, keys_a, queries, kind=KIND_MURMUR, seed=0, workers: int = 1):
    """query.py:84-95 + 182-202 -- build the query-side table with the table's
    hash range, then intersect bucket pairs."""
    v = len(offset_a) - 1
    off_b, keys_b, pos_b = build_csr(queries, v, kind, seed, workers=1)
    return intersect_csr(offset_a, keys_a, off_b, keys_b, pos_b, workers)


def count_occurrences(table_keys, queries) -> np.ndarray:
    """tests/oracles.py:25-29 -- occurrences of each query in the raw input,
    with no hashing at all (an independent oracle for multiplicities)."""
    inp = np.sort(np.asarray(table_keys))
    q = np.asarray(queries, dtype=inp.dtype)
    return (np.searchsorted(inp, q, side="right") - np.searchsorted(inp, q, side="left")).astype(np.int64)


# --------------------------------------------------------------------------- multishard


def resolve_shards(shards: int, total_keys: int, load_factor: float = 1.0, bins_g: int = 0, hash_range: int = 0):
    """multishard.py:73-80 -- (hash_range, bins_g, bin_size)."""
    hr = hash_range or hash_range_for(total_keys, load_factor)
    bins = bins_g or max(shards, round(math.sqrt(hr)))
    if bins < shards:
        raise ValueError("bins_g below shard count")
    return hr, bins, -(-hr // bins)


def splits_from_bins(bin_counts: np.ndarray, total_keys: int, shards: int) -> np.ndarray:
    """multishard.py:249-263 -- lower-bound search of r*floor(N/P) in the
    inclusive prefix, +1; first split 0, last split BINS_G."""
    cum = np.cumsum(np.asarray(bin_counts, dtype=np.int64))
    out = np.empty(shards + 1, dtype=np.int64)
    out[0] = 0
    out[shards] = len(cum)
    quota = total_keys // shards
    for r in range(1, shards):
        out[r] = int(np.searchsorted(cum, r * quota, side="left")) + 1
    return out


def bin_histogram(keys, hash_range: int, bins_g: int, kind=KIND_MURMUR, seed=0) -> np.ndarray:
    """multishard.py:371-377 / 286-289 -- bincount(hash(k, HR) // bin_size)."""
    bin_size = -(-hash_range // bins_g)
    keys = np.asarray(keys)
    if len(keys) == 0:
        return np.zeros(bins_g, dtype=np.int64)
    return np.bincount(hash_keys(kind, seed, keys, hash_range) // bin_size, minlength=bins_g).astype(np.int64)


def plan_splits(per_shard_keys, hash_range: int, bins_g: int, kind=KIND_MURMUR, seed=0) -> np.ndarray:
    """multishard.py:266-291 -- Phase 1 as a function of the input multiset."""
    total = sum(len(k) for k in per_shard_keys)
    counts = np.zeros(bins_g, dtype=np.int64)
    for k in per_shard_keys:
        counts += bin_histogram(k, hash_range, bins_g, kind, seed)
    return splits_from_bins(counts, total, len(per_shard_keys))


def dest_of_hash(hashes: np.ndarray, splits: np.ndarray, bin_size: int) -> np.ndarray:
    """multishard.py:107-113 -- searchsorted(boundaries, h, 'right') - 1.

    Equal boundaries (empty shards) route to the later shard."""
    bounds = np.asarray(splits, dtype=np.int64) * bin_size
    return np.searchsorted(bounds, np.asarray(hashes, dtype=np.int64), side="right") - 1


def reorganize(keys, splits, hash_range: int, bin_size: int, kind=KIND_MURMUR, seed=0):
    """multishard.py:294-318 -- per-destination CSR (rows in input order).

    Returns (row_offsets int64[P+1], grouped keys, search_steps)."""
    keys = np.asarray(keys)
    p = len(splits) - 1
    if len(keys) == 0:
        return np.zeros(p + 1, dtype=np.int64), keys, 0
    dest = dest_of_hash(hash_keys(kind, seed, keys, hash_range), splits, bin_size)
    offs = np.zeros(p + 1, dtype=np.int64)
    np.cumsum(np.bincount(dest, minlength=p), out=offs[1:])
    return offs, keys[np.argsort(dest, kind="stable")], int(dest.sum()) + len(dest)


def exchange_rows(sends):
    """multishard.py:137-166, 321-333 -- row d of every sender, ascending sender."""
    p = len(sends)
    out = []
    for d in range(p):
        rows = [keys[offs[d]:offs[d + 1]] for offs, keys in sends]
        out.append(np.concatenate(rows) if rows else np.empty(0, np.uint32))
    return out


def build_sharded(per_shard_keys, shards: int, load_factor=1.0, bins_g=0, hash_range=0, kind=KIND_MURMUR, seed=0):
    """multishard.py:336-471 -- the four phases, shards run one after another.

    Returns dict(hash_range, bins_g, bin_size, splits, received, tables=[(offset,
    keys)], search_steps)."""
    arrays = [np.asarray(a) for a in per_shard_keys]
    if len(arrays) != shards:
        raise ValueError("shard input count mismatch")
    total = sum(len(a) for a in arrays)
    hr, bins, bin_size = resolve_shards(shards, total, load_factor, bins_g, hash_range)
    splits = plan_splits(arrays, hr, bins, kind, seed)
    sends, steps = [], 0
    for a in arrays:
        offs, grouped, st = reorganize(a, splits, hr, bin_size, kind, seed)
        sends.append((offs, grouped))
        steps += st
    received = exchange_rows(sends)
    tables = []
    for r in received:
        v_d = hash_range_for(len(r), load_factor)  # multishard.py:403-409 (local V)
        off, placed, _ = build_csr(r, v_d, kind, seed)
        tables.append((off, placed))
    return dict(hash_range=hr, bins_g=bins, bin_size=bin_size, splits=splits,
                received=[len(r) for r in received], tables=tables, search_steps=steps)


def query_sharded(sharded: dict, queries, kind=KIND_MURMUR, seed=0):
    """multishard.py:485-542 -- route with the table's plan, per-shard query
    table + intersect, positional merge.  Returns (mult, matched, total,
    comparisons, hash_values)."""
    q = np.asarray(queries)
    p = len(sharded["splits"]) - 1
    mult = np.zeros(len(q), dtype=np.int64)
    comparisons = hash_values = 0
    if len(q):
        dest = dest_of_hash(hash_keys(kind, seed, q, sharded["hash_range"]), sharded["splits"], sharded["bin_size"])
        order = np.argsort(dest, kind="stable")
        offs = np.zeros(p + 1, dtype=np.int64)
        np.cumsum(np.bincount(dest, minlength=p), out=offs[1:])
    else:
        order = np.empty(0, np.int64)
        offs = np.zeros(p + 1, dtype=np.int64)
    for d, (off_a, keys_a) in enumerate(sharded["tables"]):
        sel = order[offs[d]:offs[d + 1]]
        m, _, _, comp, hv = query(off_a, keys_a, q[sel], kind, seed)
        mult[sel] = m
        comparisons += comp
        hash_values += hv
    return mult, int(np.count_nonzero(mult)), int(mult.sum()), comparisons, hash_values


# --------------------------------------------------------------------------- workload


_GOLDEN = 0x9E3779B97F4A7C15
_MIX1, _MIX2 = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def splitmix64_at(seed: int, indices) -> np.ndarray:
    """workload.py:63-68 -- SplitMix64 output at stream index i (0-based)."""
    i = np.asarray(indices, dtype=np.uint64)
    z = np.uint64(seed & M64) + (i + np.uint64(1)) * np.uint64(_GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
    return z ^ (z >> np.uint64(31))


def generate_keys(k: int, count: int, rng_seed: int = 0, start: int = 0, key_bits: int = 32) -> np.ndarray:
    """workload.py:71-85 -- uniform-with-replacement keys 1 + (z mod 2^k).

    `start` addresses a slice of the stream (np.array_split shards);
    key_bits=64 returns the full SplitMix64 words (extension, configs C4)."""
    z = splitmix64_at(rng_seed, np.arange(start, start + count, dtype=np.uint64))
    if key_bits == 64:
        return z
    return ((z & np.uint64((1 << k) - 1)) + np.uint64(1)).astype(np.uint32)


def default_workers() -> int:
    return max(1, os.cpu_count() or 1)
