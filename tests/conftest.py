import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name: str):
    """Golden cases recorded from the reference (tests/golden/make_golden.py)."""
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    n = int(z["ncases"])
    cases = [dict() for _ in range(n)]
    shared = {}
    for key in z.files:
        if key.startswith("c") and "." in key:
            idx, field = key[1:].split(".", 1)
            cases[int(idx)][field] = z[key]
        elif key != "ncases":
            shared[key] = z[key]
    return cases, shared


@pytest.fixture(scope="session")
def golden():
    return load_golden


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
