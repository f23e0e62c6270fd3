import os
import sys

# one BLAS thread per process: the oracle forks worker pools (like the reference's
# multiprocessing sweep), and forking after OpenBLAS has started threads can deadlock
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

# numpy may already be imported (pytest plugins) with a multi-threaded BLAS: pin it to one
# thread so the fork pools of the oracle neither deadlock nor oversubscribe
threadpool_limits(1)
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def g_domain():
    return golden("domain.npz")


@pytest.fixture(scope="session")
def g_desk():
    return golden("desk.npz")


@pytest.fixture(scope="session")
def g_c0():
    return golden("c0.npz")


def frob_rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def gap_rel(a, b):
    """relative_gap of the reference tests (test_engine3d.py:7-9)."""
    scale = max(np.max(np.abs(a)), np.max(np.abs(b)))
    return float(np.max(np.abs(a - b)) / scale)
