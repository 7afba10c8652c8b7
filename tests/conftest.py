import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


@pytest.fixture(scope="session")
def golden():
    return load_golden


def _ensure_library():
    """Build the in-tree libnncp_b200.so when it is missing (fresh checkout: it is git-ignored)."""
    lib = os.path.join(ROOT, "paper_1909_01149_b200", "libnncp_b200.so")
    if os.path.exists(lib):
        return
    import shutil

    if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
        return  # nothing to build with; tests that need the library will fail loudly
    from paper_1909_01149_b200 import build_ext

    build_ext.build()


_ensure_library()
