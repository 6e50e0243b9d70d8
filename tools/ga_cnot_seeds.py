"""Criterion 2 (GA synthesizes CNOT) over seeds 1..40 on the device GA: the
success count beside the reference's 34/40 (tests/golden/ga_cnot_outcomes_reference.json)."""
import math, sys, json
sys.path.insert(0, '.')
from paper_1809_11134_b200 import GaConfig, GaEngine, target_matrix
res = []
for s in range(1, 41):
    e = GaEngine(GaConfig(2, 6, 50, mutation_rate=0.2, mutation_range=math.pi / 8, structural_rate=0.2,
                          max_generations=10_000, target_fitness=0.999), target_matrix("CNOT"), s)
    while not e.done:
        e.steps(4096)
    res.append((s, round(e.best_fitness, 5), e.generation))
ok = sum(1 for _, b, g in res if b >= 0.999)
print(json.dumps({"ok": ok, "n": len(res), "runs": res}))
