"""ctypes binding of libhashgraph_b200.so (the C ABI in include/hashgraph_b200.h).

The library is the only compute path: if it is missing or no CUDA device is
visible, every operation raises instead of falling back to host code.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HG_LIB") or os.path.join(_HERE, "libhashgraph_b200.so")  # HG_LIB: experiment builds (tools/build_variant.py)

HG_ERR_CONFIG = -1
HG_ERR_CUDA = -2

_c_u64 = ctypes.c_uint64
_c_u32 = ctypes.c_uint32
_c_int = ctypes.c_int
_c_ptr = ctypes.c_void_p
_c_size = ctypes.c_size_t

# name -> (restype, argtypes); the declaration order of include/hashgraph_b200.h
SIGNATURES = {
    "hg_version": (ctypes.c_char_p, []),
    "hg_last_error": (ctypes.c_char_p, []),
    "hg_launch_count": (_c_u64, []),
    "hg_timing_enable": (None, [_c_int]),
    "hg_timing_collect": (_c_int, [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float), _c_int]),
    "hg_hash": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_ptr, _c_int, _c_ptr]),
    "hg_build_workspace_size": (_c_size, [_c_u64, _c_u64, _c_int]),
    "hg_build_traced_workspace_size": (_c_size, [_c_u64, _c_u64, _c_int]),
    "hg_build": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
                          _c_size, _c_ptr]),
    "hg_intersect": (_c_int, [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64,
                              _c_ptr, _c_ptr, _c_ptr]),
    "hg_intersect_tables_workspace_size": (_c_size, [_c_u64, _c_u64, _c_u64, _c_int]),
    "hg_intersect_tables": (_c_int, [_c_ptr, _c_ptr, _c_u64, _c_ptr, _c_ptr, _c_ptr, _c_u64, _c_int, _c_int, _c_u32,
                                     _c_u64, _c_ptr, _c_size, _c_ptr, _c_ptr, _c_ptr, _c_size, _c_ptr]),
    "hg_query_workspace_size": (_c_size, [_c_u64, _c_u64, _c_u64, _c_int]),
    "hg_query": (_c_int, [_c_ptr, _c_ptr, _c_u64, _c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_ptr, _c_ptr,
                          _c_ptr, _c_size, _c_ptr]),
    "hg_query_timed": (_c_int, [_c_ptr, _c_ptr, _c_u64, _c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_ptr, _c_ptr,
                                _c_ptr, _c_size, _c_ptr, _c_ptr]),
    "hg_bin_histogram": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_u64, _c_u64, _c_ptr, _c_ptr]),
    "hg_split_plan": (_c_int, [_c_ptr, _c_u64, _c_u64, _c_u32, _c_ptr, _c_ptr]),
    "hg_reorganize_workspace_size": (_c_size, [_c_u64, _c_u32]),
    "hg_reorganize": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_u64, _c_ptr, _c_u32, _c_ptr,
                               _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_size, _c_ptr]),
    "hg_reorganize_gather": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_u64, _c_ptr, _c_u32, _c_ptr,
                                      _c_ptr, _c_ptr, _c_ptr, _c_size, _c_ptr]),
    "hg_reorganize_count": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_u64, _c_ptr, _c_u32, _c_ptr,
                                     _c_ptr, _c_ptr, _c_size, _c_ptr]),
    "hg_reorganize_place_peers": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_u64, _c_ptr, _c_u32,
                                           _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_size, _c_ptr]),
    "hg_route": (_c_int, [_c_ptr, _c_u64, _c_int, _c_int, _c_u32, _c_u64, _c_u64, _c_ptr, _c_u32, _c_ptr, _c_ptr,
                          _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr]),
    "hg_return_peers": (_c_int, [_c_ptr, _c_u64, _c_ptr, _c_ptr, _c_ptr, _c_u32, _c_ptr]),
    "hg_scatter_u32": (_c_int, [_c_ptr, _c_ptr, _c_u64, _c_ptr, _c_ptr]),
    "hg_generate": (_c_int, [_c_u64, _c_u64, _c_u64, _c_int, _c_int, _c_ptr, _c_ptr]),
    "hg_widen_u32": (_c_int, [_c_ptr, _c_u64, _c_ptr, _c_ptr]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library handle.  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -m paper_2104_00792_b200._build` "
                "(or __graft_entry__.build()); there is no host fallback"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols(path: str = LIB_PATH) -> list[str]:
    lib = load(path)
    return [n for n in SIGNATURES if hasattr(lib, n)]


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load().hg_last_error() or b"").decode(errors="replace")
    if rc == HG_ERR_CONFIG:
        raise ConfigError(msg)
    raise RuntimeError(f"libhashgraph_b200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def launch_count() -> int:
    return int(load().hg_launch_count())


def timing_enable(on: bool) -> None:
    load().hg_timing_enable(1 if on else 0)


def timing_collect(cap: int = 4096) -> list[tuple[str, float]]:
    names = (ctypes.c_char_p * cap)()
    ms = (ctypes.c_float * cap)()
    n = load().hg_timing_collect(names, ms, cap)
    return [(names[i].decode(), float(ms[i])) for i in range(n)]
