"""HGR1 / KEY1 formats and CLI argument handling, on CPU (no GPU needed).

The snapshots and key file under tests/golden/ were written by the reference
itself (tests/golden/make_snapshots.py); our host-side parser must read them
back exactly, and reject malformed files with the reference's errors
(core.py:228-255, workload.py:104-118, cli.py:365-386)."""

import json
import os
import struct

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN

from paper_2104_00792_b200 import SnapshotFormatError, load_keys, save_keys
from paper_2104_00792_b200.cli import SWEEP_COLUMNS, main
from paper_2104_00792_b200.core import SNAPSHOT_HEADER, read_snapshot

REF_KEYS = O.generate_keys(12, 3000, 7)  # the fixture's input (make_snapshots.py)


def test_read_reference_snapshot_murmur():
    v, fam, lf, bits, offset, keys = read_snapshot(os.path.join(GOLDEN, "ref_murmur.hgr"))
    assert (v, fam.kind.value, fam.seed, lf, bits) == (2000, 0, 5, 1.5, 32)
    off, placed, _ = O.build_csr(REF_KEYS, v, O.KIND_MURMUR, 5)
    assert np.array_equal(offset, off)
    assert np.array_equal(keys, placed)  # the reference places stably: byte-identical


def test_read_reference_snapshot_identity():
    v, fam, lf, bits, offset, keys = read_snapshot(os.path.join(GOLDEN, "ref_identity.hgr"))
    assert (v, fam.kind.value, fam.seed, lf, bits) == (1000, 1, 0, 1.0, 32)
    off, placed, _ = O.build_csr(REF_KEYS, v, O.KIND_IDENTITY, 0)
    assert np.array_equal(offset, off) and np.array_equal(keys, placed)


def test_reference_key_file_roundtrip(tmp_path):
    keys, k = load_keys(os.path.join(GOLDEN, "ref_keys.key"))
    assert k == 12 and keys.dtype == np.uint32 and np.array_equal(keys, REF_KEYS)
    p = tmp_path / "k.key"
    save_keys(keys, 12, p)
    assert p.read_bytes() == open(os.path.join(GOLDEN, "ref_keys.key"), "rb").read()


def test_key_file_64bit_roundtrip(tmp_path):
    keys = O.generate_keys(32, 100, 3, key_bits=64)
    p = tmp_path / "k8.key"
    save_keys(keys, 64, p, key_bits=64)
    got, k = load_keys(p)
    assert k == 64 and got.dtype == np.uint64 and np.array_equal(got, keys)


def _blob(path):
    return bytearray(open(os.path.join(GOLDEN, path), "rb").read())


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b[:0] + b"JUNK" + b[4:], "bad magic"),
    (lambda b: b[:10], "truncated header"),
    (lambda b: b[:20] + bytes([7]) + b[21:], "unknown hash family"),
    (lambda b: b[:-4], "expected"),
    (lambda b: b + b"\0\0\0\0", "expected"),
])
def test_snapshot_rejects_malformed(tmp_path, mutate, msg):
    p = tmp_path / "bad.hgr"
    p.write_bytes(bytes(mutate(_blob("ref_murmur.hgr"))))
    with pytest.raises(SnapshotFormatError, match=msg):
        read_snapshot(p)


def test_snapshot_rejects_corrupt_offsets(tmp_path):
    b = _blob("ref_murmur.hgr")
    at = 4 + SNAPSHOT_HEADER.size + 8 * 5  # offset[5] made huge: no longer monotone
    b[at:at + 8] = struct.pack("<Q", 1 << 40)
    p = tmp_path / "bad.hgr"
    p.write_bytes(bytes(b))
    with pytest.raises(SnapshotFormatError, match="corrupt offset"):
        read_snapshot(p)


def test_key_file_rejects_malformed(tmp_path):
    p = tmp_path / "k.key"
    p.write_bytes(b"KEY1")
    with pytest.raises(SnapshotFormatError, match="truncated"):
        load_keys(p)
    b = _blob("ref_keys.key")
    p.write_bytes(b"XXXX" + bytes(b[4:]))
    with pytest.raises(SnapshotFormatError, match="bad magic"):
        load_keys(p)
    p.write_bytes(bytes(b[:-1]))
    with pytest.raises(SnapshotFormatError, match="expected"):
        load_keys(p)


# ---- CLI: argument and config handling never reaches the GPU

def run(*args) -> int:
    return main([str(a) for a in args])


def test_cli_usage_errors(tmp_path):
    out = tmp_path / "x.json"
    assert run("build", "--shards", 0, "--out", out) == 2
    assert run("build", "--nope", "1", "--out", out) == 2
    assert run("build", "--count", 100, "--shards", 2, "--out", out, "--snapshot-out", tmp_path / "t.hgr") == 2
    assert run("query", "--count", 10, "--out", out) == 2
    assert run("query", "--table", "x.hgr", "--input-count", 10, "--out", out) == 2
    for vals in ("4,2", "2,2", "", "0,1"):
        assert run("sweep", "--axis", "shards", "--values", vals, "--out", tmp_path / "s.csv") == 2


def test_cli_config_file_errors(tmp_path):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"shard_count": 4}))
    assert run("build", "--config", cfg, "--out", tmp_path / "r.json") == 2
    cfg.write_text("{not json")
    assert run("build", "--config", cfg, "--out", tmp_path / "r.json") == 2
    cfg.write_text(json.dumps({"hash": "sha1"}))
    assert run("build", "--config", cfg, "--out", tmp_path / "r.json") == 2
    assert run("build", "--config", tmp_path / "missing.json", "--out", tmp_path / "r.json") == 3


def test_cli_bad_snapshot_is_runtime_error(tmp_path):
    bad = tmp_path / "bad.hgr"
    bad.write_bytes(b"JUNKJUNKJUNK" + b"\x00" * 64)
    assert run("query", "--table", bad, "--count", 1, "--out", tmp_path / "q.json") == 3


def test_sweep_columns_match_reference_order():
    assert SWEEP_COLUMNS[:3] == ["axis", "value", "shards"] and SWEEP_COLUMNS[-2:] == ["status", "error"]
    assert len(SWEEP_COLUMNS) == 19
