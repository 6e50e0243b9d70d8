"""Generations/s of one QEQEA shape under each launch mode (kernels / graph)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1809_11134_b200 import PopulationConfig, QeqeaEngine, target_matrix

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--L", type=int, default=32)
ap.add_argument("--P", type=int, default=65536)
ap.add_argument("--gens", type=int, default=200)
ap.add_argument("--modes", default="kernels,graph")
a = ap.parse_args()
T = target_matrix({3: "Toffoli", 4: "CCCNOT"}.get(a.n, "Toffoli")) if a.n in (3, 4) else None
for mode in a.modes.split(","):
    eng = QeqeaEngine(PopulationConfig(a.n, a.L, a.P, max_generations=10**7, target_fitness=1.0), T, 1)
    eng.set_launch_mode(mode)
    eng.steps(20)
    t0 = time.perf_counter()
    r = eng.steps(a.gens)
    dt = time.perf_counter() - t0
    print(f"n={a.n} L={a.L} P={a.P} {mode}: {len(r) / dt:.1f} gen/s, best {r['best_fitness'][-1]:.4f}")
    eng.close()
