"""`hashgraph` shim: the reference package's import name bound to this repo's
B200 implementation, so the reference's own test suite (pkg/tests, run
unmodified by tests/test_reference_suite_gpu.py) exercises the drop-in.

Every public name and every submodule the reference exposes
(`/root/reference/pkg/src/hashgraph/__init__.py:10-113`) resolves to
`paper_2104_00792_b200`; nothing here computes anything.
"""

import sys as _sys

import paper_2104_00792_b200 as _impl
from paper_2104_00792_b200 import *  # noqa: F401,F403
from paper_2104_00792_b200 import __all__, __version__  # noqa: F401

for _name in ("cli", "core", "errors", "hashing", "multishard", "query", "workload"):
    _mod = __import__(f"paper_2104_00792_b200.{_name}", fromlist=[_name])
    _sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod
