"""Shared pytest setup: the `gpu` marker and fixture loading helpers."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def g_rng():
    return golden("rng.npz")


@pytest.fixture(scope="session")
def g_collision():
    return golden("collision.npz")


@pytest.fixture(scope="session")
def g_serial():
    return golden("serial_small.npz")


@pytest.fixture(scope="session")
def g_config1():
    return golden("config1_L16.npz")
