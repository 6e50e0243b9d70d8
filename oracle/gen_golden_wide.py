"""Goldens for numberOfWires 6..8 from the REFERENCE itself (TEST INFRASTRUCTURE
ONLY; build container).  n > 5 runs on the block-per-circuit kernel
(kernels_fitness.cu fitness_generic_kernel), not the register-resident ones:

  fitness_wide.npz        fitness_value(compose_gates(...)) (+ unitaries at n = 6)
  traj_qeqea_n6.npz       PhiloxQeqeaEngine trajectory, n = 6, L = 8, P = 4
  traj_ga_n6.npz          PhiloxGaEngine trajectory, n = 6, L = 8, P = 12

Usage:  python oracle/gen_golden_wide.py
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import gen_golden as G  # noqa: E402  (imports the reference)


def main():
    rng = np.random.default_rng(606)
    out = {}
    for n, tname, Ls in ((6, "haar", (0, 5, 20)), (6, "identity", (9,)), (7, "haar", (12,)), (8, "identity", (6,))):
        T = G.target_for(n, tname)
        nc = 3 * n + n * (n - 1) // 2
        for L in Ls:
            count = 6 if L else 2
            codes = rng.integers(0, nc, size=(count, L)).astype(np.uint8)
            thetas = rng.uniform(0.0, 2 * math.pi, size=(count, L))
            fits = np.empty(count)
            unis = np.empty((count, 2 ** n, 2 ** n), dtype=np.complex128)
            for c in range(count):
                u = G.compose_gates([G.gate_of(k, t, n) for k, t in zip(codes[c], thetas[c])], n)
                unis[c] = u
                fits[c] = G.fitness_value(u, T)
            key = f"n{n}_{tname}_L{L}"
            out[key + "_codes"], out[key + "_thetas"], out[key + "_fit"], out[key + "_target"] = codes, thetas, fits, T
            if n == 6:
                out[key + "_unitary"] = unis
    np.savez_compressed(G.OUT / "fitness_wide.npz", **out)
    G.gen_qeqea_traj("n6", 6, 8, 4, G.target_for(6, "haar"), 6, 61)
    G.gen_ga_traj("n6", 6, 8, 12, G.target_for(6, "haar"), 5, 62)
    print("wrote fitness_wide.npz, traj_qeqea_n6.npz, traj_ga_n6.npz")


if __name__ == "__main__":
    main()
