"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def canon(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128) + np.complex128(0)


def digest(a) -> str:
    """Same canonical digest as tests/golden/make_golden.py."""
    return hashlib.sha256(canon(a).tobytes()).hexdigest()


def rel_l2(got, want) -> float:
    got = np.asarray(got)
    want = np.asarray(want)
    den = float(np.linalg.norm(want))
    return float(np.linalg.norm(got - want)) / (den if den > 0 else 1.0)


def pairs_to_complex(p) -> np.ndarray:
    return np.array([complex(a, b) for a, b in p], dtype=np.complex128)


def dense_from_pairs(rows) -> np.ndarray:
    return np.array([[complex(a, b) for a, b in row] for row in rows], dtype=np.complex128)


@pytest.fixture(scope="session")
def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def configs():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def random_cases():
    return dict(np.load(os.path.join(GOLDEN, "random_cases.npz")))


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
