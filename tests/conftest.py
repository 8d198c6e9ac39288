"""Shared pytest configuration.

Markers:
  gpu — needs a CUDA device (B200) and the built libfif_b200.so; parity tests proper.
Tests without the marker run on CPU: oracle vs golden fixtures, host logic,
C-ABI exports, multi-process (gloo) sharding logic.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU and the built CUDA extension")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def g_small():
    return golden("small_field.npz")


@pytest.fixture(scope="session")
def g_models():
    return golden("models.npz")


@pytest.fixture(scope="session")
def g_cfg1():
    return golden("config1_rows.npz")


@pytest.fixture(scope="session")
def g_pc():
    return golden("pc.npz")


@pytest.fixture(scope="session")
def g_kats():
    return golden("kats.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def g_match():
    return golden("match.npz")
