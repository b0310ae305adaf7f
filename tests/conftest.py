import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# the reference's own tests (tests/ref_suite/_fetched) run in a subprocess of
# their own (tests/test_*ref_suite.py), never collected into this session
collect_ignore = ["ref_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running (full-size) cases")
    # a fresh checkout has no in-tree libqsb200.so yet (it is git-ignored):
    # compile it once with nvcc (sm_100a) before any test imports the package
    from paper_2001_10554_b200 import build as _build

    if not os.path.exists(_build.LIB):
        _build.build()


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    return a.shape == b.shape and bool(np.array_equal(a.view(np.uint64), b.view(np.uint64)))


def max_dev(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) if np.size(a) else 0.0


@pytest.fixture
def rng():
    return np.random.default_rng(20260809)
