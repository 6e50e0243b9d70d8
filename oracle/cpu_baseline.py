"""CPU baseline timing of the reference's fitness path (TEST / BENCH INFRASTRUCTURE ONLY).

Times the oracle's restatement of evaluate_circuit (engine.py:187-199): dense
Kronecker-expanded rotation matmuls + row-scaled interactions with the same
lru-cached expansions (gates.py:101-116,154-184) and fitness_value
(fitness.py:36-49), one circuit at a time, over a process pool on all host
cores with OPENBLAS_NUM_THREADS=1.  bench.py is the only
product-side caller, for its `cpu_baseline` leg and the `--impl reference` arm.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np


# the synthetic workload generators live with the product (inputs, not the
# computation); re-exported here for the CPU baseline's callers
from paper_1809_11134_b200.synthetic import haar_target, qeqea_like_circuits  # noqa: E402,F401


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

    def warm(self, n: int, L: int):
        """Spawn every worker and run a few circuits on each (imports, lru
        caches) so that the timed calls measure evaluation only."""
        codes, thetas = qeqea_like_circuits(n, L, 4 * self.workers, seed=99)
        self.evaluate(n, codes, thetas, np.eye(2 ** n, dtype=np.complex128))

    def evaluate(self, n: int, codes: np.ndarray, thetas: np.ndarray, target: np.ndarray):
        """Returns (fitness array, wall seconds) for all circuits, split evenly over the pool."""
        parts = np.array_split(np.arange(codes.shape[0]), self.workers)
        t0 = time.perf_counter()
        res = list(self.pool.map(_worker, [(n, codes[p], thetas[p], target) for p in parts]))
        wall = time.perf_counter() - t0
        return np.concatenate([r[0] for r in res]), wall

    def close(self):
        self.pool.shutdown()
