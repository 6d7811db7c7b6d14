"""Test configuration: the `gpu` marker and golden-fixture helpers.

CPU suite:  python -m pytest tests -x -q -m "not gpu"   (oracle vs reference
            goldens/KATs, host logic, C-ABI exports, gloo multi-process)
GPU suite:  python -m pytest tests -x -q -m gpu         (parity of the CUDA
            path through the C ABI against the oracle and the goldens)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the libtmb CUDA path")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name: str):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
        return cache[name]

    return load


def principal_angle(u: np.ndarray, v: np.ndarray) -> float:
    """Largest principal angle between span(u) and span(v)."""
    d = u - v @ (v.T @ u)
    return float(np.arcsin(min(1.0, np.linalg.norm(d, 2))))
