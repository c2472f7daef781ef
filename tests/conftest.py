"""Shared test setup.  `-m gpu` tests need a CUDA device (the B200 box); the
rest run on CPU.  oracle/ is test infrastructure: the checker, never the
thing under test."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_PY = os.path.join(ROOT, "oracle", "_ref", "py")
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def tib():
    import paper_2504_19171_b200 as m

    return m


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o

    return o


@pytest.fixture(scope="session")
def ref():
    """The reference's own pybind module, built by oracle/Makefile from
    /root/reference (oracle/_ref/py/tileinv)."""
    if not os.path.isdir(os.path.join(REF_PY, "tileinv")):
        pytest.skip("oracle/_ref not built (run __graft_entry__.build() where /root/reference exists)")
    if REF_PY not in sys.path:
        sys.path.insert(0, REF_PY)
    import tileinv

    return tileinv


def normwise(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def elementwise(a, b, floor=1e-30):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))
