"""One C2-shaped GA run (GPUGA on Toffoli, P=50, L=16): generations/s of the
fused cooperative launch (profiling helper)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1809_11134_b200 import GaConfig, GaEngine, target_matrix

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
eng = GaEngine(GaConfig(3, 16, 50, max_generations=10**7, target_fitness=1.0), target_matrix("Toffoli"), 1)
eng.steps(50)
t0 = time.perf_counter()
r = eng.steps(n)
print(f"C2 GA: {len(r) / (time.perf_counter() - t0):.1f} gen/s")
