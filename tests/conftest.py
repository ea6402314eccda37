"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else
runs on a CPU-only machine."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "codec_cases.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_a2a():
    with np.load(GOLDEN / "a2a_frames.npz") as z:
        return {k: z[k] for k in z.files}


def gaussian_words(n: int, sigma: float = 1.0, seed: int = 0) -> np.ndarray:
    """Same generator as the reference tests/conftest.py:10-12."""
    from oracle import zc_oracle as zo
    return zo.gaussian(n, sigma, seed)


def rank_words(rank: int, n: int, seed: int = 0, sigma: float = 1.0) -> np.ndarray:
    """Same generator as the reference tests/conftest.py:15-17."""
    from oracle import zc_oracle as zo
    return zo.rank_gaussian(rank, n, seed, sigma)
