import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    """(meta dict, npz arrays) of a reference-generated fixture."""
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    path = os.path.join(GOLDEN, f"{name}.npz")
    arrays = np.load(path) if os.path.exists(path) else None
    return meta, arrays


def relative_diff(a, b):
    """max-abs difference / max-abs scale (reference tests/conftest.py:21-23)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(np.abs(a).max(), np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / scale)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
