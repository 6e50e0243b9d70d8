"""Run a few QEQEA generations at a given shape (profiling helper)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np

from paper_1809_11134_b200.synthetic import haar_target
from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
from paper_1809_11134_b200.fitness import TargetSpec, target_matrix

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=5)
ap.add_argument("--L", type=int, default=64)
ap.add_argument("--P", type=int, default=1 << 16)
ap.add_argument("--gens", type=int, default=4)
a = ap.parse_args()
T = haar_target(a.n)
cfg = PopulationConfig(number_of_wires=a.n, size_of_individual=a.L, size_of_population=a.P,
                       target_fitness=1.0)
eng = QeqeaEngine(cfg, TargetSpec("haar", a.n, T), seed=1)
eng.steps(2)
t0 = time.perf_counter()
r = eng.steps(a.gens)
dt = time.perf_counter() - t0
print(f"n={a.n} L={a.L} P={a.P}: {a.gens / dt:.2f} gen/s, {a.P * a.gens / dt:.4g} evals/s, best {r['best_fitness'][-1]:.4f}")
