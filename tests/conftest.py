"""Shared fixtures.  ``-m gpu`` tests need a B200 and the built CUDA library;
``-m "not gpu"`` tests run on any CPU host (oracle vs golden, host logic,
C-ABI symbol exports, gloo multi-process logic)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(20240811)


def _load(name):
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_small():
    return _load("golden_small.npz")


@pytest.fixture(scope="session")
def golden_sweep():
    return _load("golden_sweep.npz")


@pytest.fixture(scope="session")
def golden_c0():
    return _load("golden_c0.npz")


def random_field(rng, n, r=None):
    shape = (n,) if r is None else (n, r)
    return rng.normal(size=shape) + 1j * rng.normal(size=shape)


def relerr(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
