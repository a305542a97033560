"""Shared test setup.

* ``gpu`` marker: tests that need a B200 (run with ``-m gpu`` on the GPU box).
* ``oracle`` on sys.path: the float64 CPU oracle (test infrastructure only).
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")


@pytest.fixture
def rng():
    return np.random.default_rng(42)


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def max_grad_error(analytic, numeric, abs_floor=1e-8):
    """T/conftest.py:41-48: largest relative error over entries above the floor."""
    analytic = np.asarray(analytic, dtype=np.float64).ravel()
    numeric = np.asarray(numeric, dtype=np.float64).ravel()
    diff = np.abs(analytic - numeric)
    scale = np.maximum(np.abs(analytic), np.abs(numeric))
    rel = np.where(diff <= abs_floor, 0.0, diff / np.maximum(scale, 1e-300))
    return float(rel.max()) if rel.size else 0.0
