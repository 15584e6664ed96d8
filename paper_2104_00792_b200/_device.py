"""Device plumbing: torch supplies CUDA memory and the current stream; every
computation is a libhashgraph_b200 kernel launched through _lib."""

from __future__ import annotations

import warnings

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
    with warnings.catch_warnings():  # read-only arrays (e.g. a table's keys) are only read here
        warnings.simplefilter("ignore", UserWarning)
        host = t.from_numpy(arr.view(np.int32 if key_bits == 32 else np.int64))
    return host.to(device(), non_blocking=False)


def to_numpy_keys(t, key_bits: int = 32) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view(np_key_dtype(key_bits))


def widen_u32_to_numpy(t) -> np.ndarray:
    """uint32 device array -> int64 numpy (kernel widening, then one D2H)."""
    n = t.numel()
    out = torch().empty(n, dtype=torch().int64, device=t.device)
    _lib.call("hg_widen_u32", ptr(t), n, ptr(out), stream_ptr())
    return out.cpu().numpy()


def frozen(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a
