"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/hashgraph_b200.h declares, the ctypes table matches the
header, host-side validation raises the reference's error types, and the
product path refuses to run without a GPU (no host fallback)."""

import os
import re
import sys

import numpy as np
import pytest

import paper_2104_00792_b200 as hg
from paper_2104_00792_b200 import _lib
from conftest import ROOT, has_cuda

HEADER = os.path.join(ROOT, "include", "hashgraph_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"HG_API\s+[\w\s\*]+?\b(hg_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.hg_version().startswith(b"hashgraph_b200")


def test_workspace_queries_are_host_only():
    lib = _lib.load()
    assert lib.hg_build_workspace_size(1 << 20, 1 << 20, 32) >= 4 * (1 << 20)
    assert lib.hg_query_workspace_size(1 << 20, 1 << 20, 1 << 20, 32) > lib.hg_build_workspace_size(1 << 20, 1 << 20, 32)
    assert lib.hg_reorganize_workspace_size(1 << 20, 8) > 0


def test_two_step_abi_host_checks():
    """hg_build_traced_workspace_size covers the trace on top of the build;
    hg_intersect_tables sizes its workspace and rejects a missing positions
    array before touching the device."""
    lib = _lib.load()
    n = 1 << 22
    # the trace: grouped keys, two u16 position maps and the carried input indices (12 B per key)
    assert lib.hg_build_traced_workspace_size(n, n, 32) > lib.hg_build_workspace_size(n, n, 32) + 12 * n
    assert lib.hg_build_traced_workspace_size(100, 100, 32) == lib.hg_build_workspace_size(100, 100, 32)  # direct path
    assert lib.hg_intersect_tables_workspace_size(n, n, n, 32) > 8 * n
    rc = lib.hg_intersect_tables(None, None, n, None, None, None, n, 32, 0, 0, n, None, 0, None, None, None, 0, None)
    assert rc == -1 and b"positions_b" in lib.hg_last_error()
    # layouts beyond 32768 fine bins (2^30 keys at C = 1) stay on the binned path's workspace
    big = 1 << 30
    assert lib.hg_build_workspace_size(big, big, 32) > 4 * big


def test_config_errors_match_reference_types():
    assert issubclass(hg.ConfigError, ValueError)
    assert issubclass(hg.SnapshotFormatError, RuntimeError)
    with pytest.raises(hg.ConfigError):
        hg.ShardConfig(shards=0)
    with pytest.raises(hg.ConfigError):
        hg.ShardConfig(shards=1, load_factor=0.0)
    with pytest.raises(hg.ConfigError):
        hg.HashFamily(hg.HashKind.MURMUR32, 1 << 32)
    with pytest.raises(hg.ConfigError):
        hg.hash_range_for(10, 0.0)
    with pytest.raises(hg.ConfigError):
        hg.ShardConfig(shards=2, bins_g=1).resolve(10)
    cfg = hg.ShardConfig(shards=4, load_factor=0.5)
    hr, bins, bs = cfg.resolve(1 << 20)
    assert hr == 1 << 21 and bins == round((1 << 21) ** 0.5) and bs == -(-hr // bins)
    assert hg.ShardConfig(shards=8).resolve(4)[:2] == (4, 8)


def test_scalar_hash_helpers():
    assert hg.fmix32(1) == 0x514E28B7
    assert hg.hash_key(hg.HashFamily.identity(), 7, 4) == 3
    assert hg.hash_key(hg.HashFamily.murmur32(0x9E3779B9), 12345, 1 << 32) == hg.fmix32(12345 ^ 0x9E3779B9)


def test_public_surface_covers_reference_hot_path():
    for name in ["build", "build_traced", "build_query_table", "intersect_tables", "intersect", "intersect_timed",
                 "plan_partition", "reorganize", "exchange", "build_sharded", "query_sharded", "query_sharded_timed",
                 "HashGraph", "QueryResult", "PhaseReport", "ShardConfig", "PartitionPlan", "SendBuffers",
                 "ExchangeFabric", "ShardedHashGraph", "work_audit", "hash_array", "generate"]:
        assert hasattr(hg, name), name


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU behaviour")
def test_no_host_fallback_without_gpu():
    with pytest.raises(RuntimeError, match="CUDA"):
        hg.build(np.arange(10, dtype=np.uint32))
    with pytest.raises(RuntimeError, match="CUDA"):
        hg.hash_array(hg.HashFamily(), np.arange(10, dtype=np.uint32), 7)


def test_conformance_shim_maps_the_reference_names():
    """tests/conformance/hashgraph binds every reference export and submodule
    to this package (the reference suite runs through it on the GPU)."""
    import importlib

    sys.path.insert(0, os.path.join(ROOT, "tests", "conformance"))
    try:
        shim = importlib.import_module("hashgraph")
        import paper_2104_00792_b200 as impl

        assert shim.__file__.startswith(os.path.join(ROOT, "tests", "conformance"))
        for name in impl.__all__:
            assert getattr(shim, name) is getattr(impl, name)
        for sub in ("cli", "core", "errors", "hashing", "multishard", "query", "workload"):
            assert importlib.import_module(f"hashgraph.{sub}") is importlib.import_module(f"paper_2104_00792_b200.{sub}")
    finally:
        sys.path.remove(os.path.join(ROOT, "tests", "conformance"))
        for k in [k for k in sys.modules if k == "hashgraph" or k.startswith("hashgraph.")]:
            del sys.modules[k]
