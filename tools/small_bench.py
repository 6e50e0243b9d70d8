"""Generations/s at the tiny configs C1-C3 (latency bound)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

def run(eng, n):
    eng.steps(50)
    t0 = time.perf_counter()
    r = eng.steps(n)
    return len(r) / (time.perf_counter() - t0)

t = target_matrix("Toffoli")
f = target_matrix("Fredkin")
out = {}
out["C1 qeqea toffoli P=5 L=16"] = run(QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=10**7, target_fitness=1.0), t, 1), 4000)
out["C3 qeqea fredkin P=5 L=16"] = run(QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=10**7, target_fitness=1.0), f, 1), 4000)
out["C2 ga toffoli P=50 L=16"] = run(GaEngine(GaConfig(3, 16, 50, max_generations=10**7, target_fitness=1.0), t, 1), 4000)
out["C4 qeqea cccnot P=65536 L=32"] = run(QeqeaEngine(PopulationConfig(4, 32, 65536, max_generations=10**7, target_fitness=1.0), target_matrix("CCCNOT"), 1), 50)
for k, v in out.items():
    print(f"{k}: {v:.1f} gen/s")
