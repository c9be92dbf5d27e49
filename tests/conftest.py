"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as f:
        return {k: f[k] for k in f.files}


@pytest.fixture
def runtime():
    """A live device runtime (reference conftest.py:19-25 `pool` analogue)."""
    import paper_2505_00136_b200 as gpb

    rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
    yield rt
    if gpb.current_runtime() is rt:
        rt.stop()


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
