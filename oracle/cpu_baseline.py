"""CPU baseline timing of the reference's fitness path (TEST / BENCH INFRASTRUCTURE ONLY).

Times the oracle's restatement of evaluate_circuit (engine.py:187-199): dense
Kronecker-expanded rotation matmuls + row-scaled interactions with the same
lru-cached expansions (gates.py:101-116,154-184) and fitness_value
(fitness.py:36-49), one circuit at a time, over a process pool on all host
cores with OPENBLAS_NUM_THREADS=1.  bench.py is the only
product-side caller, for its `cpu_baseline` leg and the `--impl reference` arm.
"""
from __future__ import annotations

import math
import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def qeqea_like_circuits(n: int, L: int, count: int, seed: int = 0):
    """Random circuits with the QEQEA gate mix: slot kind uniform over the
    n + C(n,2) kinds (engine.py:180), measured axis uniform, theta uniform."""
    rng = np.random.default_rng(seed)
    K = n + n * (n - 1) // 2
    kinds = rng.integers(0, K, size=(count, L))
    axes = rng.integers(0, 3, size=(count, L))
    codes = np.where(kinds < n, 3 * kinds + axes, 3 * n + (kinds - n)).astype(np.uint8)
    thetas = rng.uniform(0.0, 2 * math.pi, size=(count, L))
    return codes, thetas


def haar_target(n: int) -> np.ndarray:
    """The C5 synthetic target: QR-Haar unitary from default_rng(12345)
    (pkg/tests/conftest.py:10-14), identical bits on every host."""
    rng = np.random.default_rng(12345)
    d = 2 ** n
    z = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def _worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle.qeqea import circuit_fitness

    n, codes, thetas, target = args
    t0 = time.perf_counter()
    fits = np.array([circuit_fitness(codes[i], thetas[i], target, n) for i in range(codes.shape[0])])
    return fits, time.perf_counter() - t0


class CpuPool:
    def __init__(self, workers: int | None = None):
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        import multiprocessing as mp

        self.workers = workers or os.cpu_count() or 1
        self.pool = ProcessPoolExecutor(max_workers=self.workers, mp_context=mp.get_context("spawn"))

    def evaluate(self, n: int, codes: np.ndarray, thetas: np.ndarray, target: np.ndarray):
        """Returns (fitness array, wall seconds) for all circuits, split evenly over the pool."""
        parts = np.array_split(np.arange(codes.shape[0]), self.workers)
        t0 = time.perf_counter()
        res = list(self.pool.map(_worker, [(n, codes[p], thetas[p], target) for p in parts]))
        wall = time.perf_counter() - t0
        return np.concatenate([r[0] for r in res]), wall

    def close(self):
        self.pool.shutdown()
