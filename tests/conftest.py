"""Shared fixtures.  Markers: ``gpu`` = needs a CUDA device (run on the B200
box with ``-m gpu``); everything else runs on CPU (``-m "not gpu"``)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

GOLDEN = os.path.join(HERE, "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")


def int_clmul(a: int, b: int) -> int:
    """Independent bitwise shift-and-XOR oracle (cf. reference conftest.py:15-23)."""
    acc = 0
    while b:
        if b & 1:
            acc ^= a
        a <<= 1
        b >>= 1
    return acc


@pytest.fixture
def rng():
    return np.random.default_rng(0xF2F2)  # reference conftest.py:46


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_10473_b200 import _lib

    _lib.load()  # fail loudly if the extension is missing
    return torch.device("cuda", 0)
