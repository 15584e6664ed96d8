"""The reference's own test suite, unmodified, against this package (GPU).

SURVEY §4 implication 2 / VERDICT r1 "Next round" item 8: the reference's
pkg/tests (193 tests: hashing, core, query, multishard, workload, CLI and the
c01-c10 acceptance criteria) run through a shim package named `hashgraph`
(tests/conformance/hashgraph) that re-exports paper_2104_00792_b200.  The
suite is packed from /root/reference by oracle/pack_reference_tests.py into the
git-ignored oracle/_ref/reference_tests.tar, which travels to the GPU box; the
test skips (with the reason) when that archive is absent.

Nothing is deselected: every reference test, timed acceptance cases included,
must pass on the drop-in.
"""

import os
import subprocess
import sys
import tarfile

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAR = os.path.join(ROOT, "oracle", "_ref", "reference_tests.tar")
SHIM = os.path.join(ROOT, "tests", "conformance")

# reference tests that cannot be expressed on this backend, with the reason
# (empty: the whole suite runs)
DESELECT: dict[str, str] = {}


def run_suite(tmp_path, shim_root, extra_env=None):
    with tarfile.open(TAR) as tar:
        tar.extractall(tmp_path, filter="data")
    tests = os.path.join(tmp_path, "tests")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([shim_root, ROOT, env.get("PYTHONPATH", "")])
    env.update(extra_env or {})
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=", "--rootdir", tests, tests]
    for nodeid in DESELECT:
        cmd += ["--deselect", os.path.join(tests, nodeid)]
    return subprocess.run(cmd, cwd=tests, env=env, capture_output=True, text=True, timeout=1800)


@pytest.mark.skipif(not os.path.exists(TAR), reason="oracle/_ref/reference_tests.tar not packed (needs /root/reference at build time)")
def test_reference_suite_on_the_drop_in(tmp_path):
    import torch

    assert torch.cuda.is_available()
    r = run_suite(tmp_path, SHIM)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-60:])
    assert r.returncode == 0, f"reference suite failed on the drop-in:\n{tail}"
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
    # the shim really served the drop-in (the extension was loaded by the child)
    assert "error" not in r.stdout.splitlines()[-1].lower(), tail
