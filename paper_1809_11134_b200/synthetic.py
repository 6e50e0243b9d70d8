"""Synthetic workloads of BASELINE.json's configurations (inputs only).

`haar_target(n)` is the C5 target: the QR-Haar unitary of the reference's
test fixture (pkg/tests/conftest.py:10-14) drawn from default_rng(12345), so
every host builds identical bits.  `qeqea_like_circuits` draws explicit
circuits with the QEQEA gate mix (slot kind uniform over the n + C(n, 2)
kinds, engine.py:180; measured axis uniform; angle uniform) for the
explicit-gate fitness API.
"""
from __future__ import annotations

import math

import numpy as np


def haar_target(n: int) -> np.ndarray:
    rng = np.random.default_rng(12345)
    d = 2 ** n
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def qeqea_like_circuits(n: int, L: int, count: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    K = n + n * (n - 1) // 2
    kinds = rng.integers(0, K, size=(count, L))
    axes = rng.integers(0, 3, size=(count, L))
    codes = np.where(kinds < n, 3 * kinds + axes, 3 * n + (kinds - n)).astype(np.uint8)
    thetas = rng.uniform(0.0, 2 * math.pi, size=(count, L))
    return codes, thetas
