"""compute-sanitizer over the binned build and query (GPU).

The kernels use mbarriers, TMA bulk copies, `fence.proxy.async`, packed-u16
shared-memory atomics and a named barrier; memcheck, racecheck and synccheck
each run tests/sanitize_case.py (every binned kernel, answers checked against
the oracle) and must report zero errors."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    tail = "\n".join(out.splitlines()[-40:])
    if r.returncode != 0 and "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (it has left
        # GPUs needing a reset there); the clean runs of this round are
        # recorded in DESIGN.md
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + out.strip().splitlines()[-1][:200])
    assert r.returncode == 0, tail
    assert "sanitize_case ok" in out, tail
    assert "ERROR SUMMARY: 0 errors" in out or "SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, tail
