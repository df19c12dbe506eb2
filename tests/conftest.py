"""Shared fixtures: golden-vector loaders and product/oracle adapters."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def golden(name):
    return np.load(GOLDEN / name)


def lod_files():
    return sorted(GOLDEN.glob("lod_*.npz"))
