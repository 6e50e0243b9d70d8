"""Outcome distribution of the REFERENCE GA on criterion 2 (TEST INFRASTRUCTURE ONLY).

Runs the reference's own GaEngine (pkg/src/isingsynth/ga.py:141-214) with the
configuration of pkg/tests/test_acceptance.py:65-79 (CNOT, n = 2, L = 6,
P = 50, 10,000 generations, target 0.999) for seeds 1..N and writes
tests/golden/ga_cnot_outcomes_reference.json: per seed (seed, best fitness,
generations).  The reference's criterion asserts 5/5 successes on seeds 1..5;
with independent streams per seed that is one draw of a ~85 % per-seed
success rate, so tests/test_acceptance_gpu.py compares success RATES over 40
seeds against this file.

Usage:  python oracle/gen_ga_cnot_outcomes.py [N=40] [workers=os.cpu_count()]
"""
import json
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "ga_cnot_outcomes_reference.json"


def run(seed: int):
    sys.path.insert(0, REF)
    from isingsynth import GaConfig, GaEngine, target_matrix

    e = GaEngine(GaConfig(number_of_wires=2, size_of_individual=6, population=50, mutation_rate=0.2,
                          mutation_range=math.pi / 8, structural_rate=0.2, max_generations=10_000,
                          target_fitness=0.999), target_matrix("CNOT"), seed)
    while not e.done:
        e.step()
    return [seed, round(float(e.best_fitness), 5), int(e.generation)]


if __name__ == "__main__":
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
    with ProcessPoolExecutor(workers) as ex:
        runs = list(ex.map(run, range(1, n + 1)))
    ok = sum(1 for _, b, _ in runs if b >= 0.999)
    OUT.write_text(json.dumps({"source": "reference isingsynth GaEngine, pkg/tests/test_acceptance.py:65-79",
                               "successes": ok, "seeds": n, "runs": runs}) + "\n")
    print(f"{ok}/{n} -> {OUT}")
