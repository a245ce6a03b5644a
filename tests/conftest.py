"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
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
    config.addinivalue_line("markers", "slow: large sizes (minutes)")


def random_f32(n, seed):
    """reference pkg/tests/conftest.py:7-9"""
    rng = np.random.default_rng(seed)
    return rng.random(n, dtype=np.float32) - np.float32(0.5)


def random_c(n, seed, dtype=np.complex128):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
