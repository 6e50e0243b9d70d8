import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libisq.so")


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def random_unitary(dim: int, rng: np.random.Generator) -> np.ndarray:
    """QR-Haar, as the reference's conftest (pkg/tests/conftest.py:10-14)."""
    z = rng.normal(size=(dim, dim)) + 1j * rng.normal(size=(dim, dim))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def fit_close(a, b, rel=1e-9, abs_=1e-12):
    """The north-star fp64 fitness tolerance: |d| <= 1e-9 |ref| + 1e-12."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) <= rel * np.abs(b) + abs_
