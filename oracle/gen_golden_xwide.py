"""Goldens for numberOfWires 9..13 from the REFERENCE itself (TEST
INFRASTRUCTURE ONLY; build container).  13 is the reference's default cap
(4^n <= 2^26, engine.py:43,60-63); the device runs these on the
block-per-circuit kernel (kernels_fitness.cu fitness_generic_kernel).  The
targets are oracle/targets.product_target(n, seed) (not stored: 1 GB at n = 13).

  fitness_xwide.npz         fitness_value(compose_gates(...)) per (n, L)
  traj_qeqea_n11.npz        PhiloxQeqeaEngine trajectory, n = 11, L = 4, P = 2
  traj_ga_n11.npz           PhiloxGaEngine trajectory, n = 11, L = 4, P = 3

Usage:  python oracle/gen_golden_xwide.py      (a few minutes, ~8 GB RAM)
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import gen_golden as G  # noqa: E402  (imports the reference)
from targets import product_target  # noqa: E402
from isingsynth import gates as R_gates  # noqa: E402


def _strip_target(path: Path, seed: int) -> None:
    d = dict(np.load(path))
    del d["target"]
    np.savez_compressed(path, target_seed=seed, **d)


def main():
    rng = np.random.default_rng(909)
    out = {}
    for n, L, count in ((9, 12, 3), (10, 8, 2), (11, 6, 2), (12, 3, 1), (13, 3, 1)):
        t0 = time.time()
        T = product_target(n, 100 + n)
        nc = 3 * n + n * (n - 1) // 2
        codes = rng.integers(0, nc, size=(count, L)).astype(np.uint8)
        codes[:, :2] = rng.integers(0, 3 * n, size=(count, 2))  # at least two rotations (dense in the reference)
        thetas = rng.uniform(-0.5, 0.5, size=(count, L)) + rng.choice([0.0, 2 * np.pi, -2 * np.pi], size=(count, L))
        fits = np.array([G.fitness_value(G.compose_gates([G.gate_of(k, t, n) for k, t in zip(codes[c], thetas[c])], n), T)
                         for c in range(count)])
        key = f"n{n}_L{L}"
        out[key + "_codes"], out[key + "_thetas"], out[key + "_fit"] = codes, thetas, fits
        out[key + "_target_seed"] = np.int64(100 + n)
        R_gates._expanded_rotation_cached.cache_clear()  # 1 GB per cached n = 13 gate
        print(f"n={n}: {codes.tolist()} {fits} ({time.time() - t0:.1f} s)", flush=True)
    np.savez_compressed(G.OUT / "fitness_xwide.npz", **out)
    G.gen_qeqea_traj("n11", 11, 4, 2, product_target(11, 111), 2, 71)
    _strip_target(G.OUT / "traj_qeqea_n11.npz", 111)
    G.gen_ga_traj("n11", 11, 4, 3, product_target(11, 112), 2, 72)
    _strip_target(G.OUT / "traj_ga_n11.npz", 112)
    print("wrote fitness_xwide.npz, traj_qeqea_n11.npz, traj_ga_n11.npz")


if __name__ == "__main__":
    main()
