"""Device plumbing: torch supplies CUDA memory and the current stream; every
computation is a libhashgraph_b200 kernel launched through _lib."""

from __future__ import annotations

import os
import threading
import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .errors import ConfigError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_2104_00792_b200 needs a CUDA device (sm_100a); no CPU fallback exists"
        )
    _lib.load()
    return t


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


def device():
    return torch().device("cuda", torch().cuda.current_device())


def on(where):
    """Context manager making `where` (a CUDA tensor, torch.device or index) the
    current device, so allocations, `device()` and `stream_ptr()` follow it."""
    t = torch()
    if is_tensor(where):
        where = where.device
    return t.cuda.device(where)


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def storage_dtype(key_bits: int):
    t = torch()
    return t.int32 if key_bits == 32 else t.int64


def np_key_dtype(key_bits: int):
    return np.uint32 if key_bits == 32 else np.uint64


def empty(n: int, key_bits: int = 32):
    return torch().empty(max(int(n), 0), dtype=storage_dtype(key_bits), device=device())


def zeros(n: int, key_bits: int = 32):
    return torch().zeros(max(int(n), 0), dtype=storage_dtype(key_bits), device=device())


def workspace(nbytes: int):
    return torch().empty(max(int(nbytes), 1), dtype=torch().uint8, device=device())


def is_cuda_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def is_tensor(x) -> bool:
    return isinstance(x, torch().Tensor)


def key_count(keys) -> int:
    return keys.numel() if is_tensor(keys) else len(keys)


def coerce_host_keys(keys, key_bits: int = 32) -> np.ndarray:
    """core.py:84-88 -- contiguous 1-D array; 32-bit mode truncates like the reference."""
    arr = np.asarray(keys, dtype=np_key_dtype(key_bits))
    if arr.ndim != 1:
        raise ConfigError(f"keys must be one-dimensional, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


def to_device_keys(keys, key_bits: int = 32):
    """Keys as a contiguous CUDA tensor (int32/int64 storage of uint32/uint64)."""
    t = require_cuda()
    if is_cuda_tensor(keys):
        if keys.dim() != 1:
            raise ConfigError(f"keys must be one-dimensional, got shape {tuple(keys.shape)}")
        want = storage_dtype(key_bits)
        if keys.dtype == want:
            return keys.contiguous()
        if keys.dtype in (t.uint32,) and key_bits == 32:
            return keys.view(t.int32).contiguous()
        if keys.dtype in (t.uint64,) and key_bits == 64:
            return keys.view(t.int64).contiguous()
        return keys.to(want).contiguous()
    if isinstance(keys, t.Tensor):  # host tensor (pinned memory copies asynchronously)
        if keys.dim() != 1:
            raise ConfigError(f"keys must be one-dimensional, got shape {tuple(keys.shape)}")
        want = storage_dtype(key_bits)
        if keys.dtype in (t.uint32, t.uint64) and keys.element_size() == (4 if key_bits == 32 else 8):
            keys = keys.view(want)
        elif keys.dtype != want:
            keys = keys.to(want)
        return keys.to(device(), non_blocking=keys.is_pinned())
    arr = coerce_host_keys(keys, key_bits)
    return h2d_numpy(arr.view(np.int32 if key_bits == 32 else np.int64))


# ---- host <-> device transfers for numpy callers (the reference API's arrays)
#
# A pageable copy runs at ~10 GB/s and a fresh pageable destination pays a
# page fault per 4 KB (a 2 GB int64 result took ~1 s).  Host -> device goes
# through two cached pinned chunks filled by a thread pool (several cores'
# memory bandwidth) while the other chunk's DMA runs; device -> host lands in
# pinned memory from torch's caching host allocator and is returned as a
# numpy view of it (no copy, no page faults once the allocator has the block).
_H2D_CHUNK = 64 << 20  # bytes per staging chunk
_state = threading.local()
_pool = None
_pool_lock = threading.Lock()


def _copy_pool():
    global _pool
    with _pool_lock:
        if _pool is None:
            _pool = ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1)))
    return _pool


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src with the copy split over the pool (numpy releases the GIL)."""
    n = len(src)
    parts = 8 if n * src.itemsize >= (8 << 20) else 1
    if parts == 1:
        np.copyto(dst, src)
        return
    step = -(-n // parts)
    futs = [_copy_pool().submit(np.copyto, dst[i:i + step], src[i:i + step]) for i in range(0, n, step)]
    for f in futs:
        f.result()


def _staging():
    t = torch()
    key = t.cuda.current_device()
    st = getattr(_state, "staging", None)
    if st is None or st[0] != key:
        bufs = [t.empty(_H2D_CHUNK, dtype=t.uint8, pin_memory=True) for _ in range(2)]
        evs = [t.cuda.Event() for _ in range(2)]
        st = (key, bufs, evs, [False, False])
        _state.staging = st
    return st


def h2d_numpy(arr: np.ndarray):
    """Contiguous numpy array -> CUDA tensor of the same dtype, enqueued on the
    current stream through the pinned staging chunks (returns after the last
    chunk is staged; the DMA itself is asynchronous)."""
    t = torch()
    arr = np.ascontiguousarray(arr)
    with warnings.catch_warnings():  # read-only arrays (e.g. a table's keys) are only read here
        warnings.simplefilter("ignore", UserWarning)
        src = t.from_numpy(arr)
    out = t.empty(arr.shape, dtype=src.dtype, device=device())
    nbytes = arr.nbytes
    if nbytes < (1 << 20):
        return src.to(device())
    _, bufs, evs, used = _staging()
    flat = arr.view(np.uint8).reshape(-1)
    out_b = out.view(t.uint8).reshape(-1)
    stream = t.cuda.current_stream()
    for i, off in enumerate(range(0, nbytes, _H2D_CHUNK)):
        k = i & 1
        m = min(_H2D_CHUNK, nbytes - off)
        if used[k]:
            evs[k].synchronize()  # the chunk's previous DMA has read it
        _par_copy(bufs[k].numpy()[:m], flat[off:off + m])
        out_b[off:off + m].copy_(bufs[k][:m], non_blocking=True)
        evs[k].record(stream)
        used[k] = True
    return out


def d2h_numpy(t_dev) -> np.ndarray:
    """CUDA tensor -> numpy array viewing pinned host memory (synchronises)."""
    t = torch()
    host = t.empty(t_dev.shape, dtype=t_dev.dtype, pin_memory=True)
    host.copy_(t_dev, non_blocking=True)
    t.cuda.current_stream().synchronize()
    return host.numpy()


def to_numpy_keys(t, key_bits: int = 32) -> np.ndarray:
    with on(t):
        a = d2h_numpy(t)
    return a.view(np_key_dtype(key_bits))


def widen_u32_to_numpy(t) -> np.ndarray:
    """uint32 device array -> int64 numpy (kernel widening, then one D2H)."""
    n = t.numel()
    with on(t):
        out = torch().empty(n, dtype=torch().int64, device=t.device)
        _lib.call("hg_widen_u32", ptr(t), n, ptr(out), stream_ptr())
        return d2h_numpy(out)


def frozen(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a
