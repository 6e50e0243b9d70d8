"""One C1-shaped QEQEA run (Toffoli, P=5, L=16): generations/s of the fused
single-block launch (profiling helper)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1809_11134_b200 import PopulationConfig, QeqeaEngine, target_matrix

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
eng = QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=10**7, target_fitness=1.0), target_matrix("Toffoli"), 1)
eng.steps(50)
t0 = time.perf_counter()
r = eng.steps(n)
print(f"C1 QEQEA: {len(r) / (time.perf_counter() - t0):.1f} gen/s")
