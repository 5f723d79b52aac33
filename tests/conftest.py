"""Shared fixtures.  GPU tests are marked ``gpu``; the CPU suite runs with
``-m "not gpu"``.  GPU tests never skip silently: without a CUDA device they
fail, so a GPU box without a working device cannot pass them."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "reference_small.npz")


@pytest.fixture(scope="session")
def oracle():
    import irk_oracle

    return irk_oracle


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    from paper_2403_08084_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
