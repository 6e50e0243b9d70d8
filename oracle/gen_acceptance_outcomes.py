"""Outcome distributions of the REFERENCE on acceptance criteria 3 and 12
over many seeds (TEST INFRASTRUCTURE ONLY; build container).

The reference's criteria are stated on seeds 1..5 (criterion 3,
pkg/tests/test_acceptance.py:82-105, 249-255) or one seed (criterion 12,
smoke_run, :140-164); with per-seed outcomes being draws of each run's random
streams, the device engines (counter-based Philox streams) are compared with
the reference as distributions over seeds 1..N.  This script runs the
reference's own engines with exactly those configurations and writes
tests/golden/acceptance_outcomes_reference.json: per seed, the best fitness.

Usage:  python oracle/gen_acceptance_outcomes.py [N=40] [workers=os.cpu_count()]
"""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "acceptance_outcomes_reference.json"


def run(job):
    sys.path.insert(0, REF)
    from isingsynth import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

    kind, seed = job
    if kind == "c3_ga_toffoli":  # test_acceptance.py:82-91
        e = GaEngine(GaConfig(number_of_wires=3, size_of_individual=16, population=50, max_generations=20_000),
                     target_matrix("Toffoli"), seed)
    elif kind == "c3_qeqea_toffoli":  # :94-104
        e = QeqeaEngine(PopulationConfig(number_of_wires=3, size_of_individual=16, size_of_population=5,
                                         max_generations=20_000), target_matrix("Toffoli"), seed)
    else:  # c12 smoke_run (:140-164) at this seed
        _, algo, name, gens = kind.split("_")
        spec = target_matrix(name)
        if algo == "qeqea":
            e = QeqeaEngine(PopulationConfig(number_of_wires=spec.number_of_wires, size_of_individual=16,
                                             size_of_population=5, max_generations=int(gens)), spec, seed)
        else:
            e = GaEngine(GaConfig(number_of_wires=spec.number_of_wires, size_of_individual=16, population=20,
                                  max_generations=int(gens)), spec, seed)
    while not e.done:
        e.step()
    return kind, seed, round(float(e.best_fitness), 6)


KINDS = ("c3_ga_toffoli", "c3_qeqea_toffoli", "c12_qeqea_CCCNOT_2000", "c12_qeqea_Peres_2000", "c12_ga_Peres_1000")

if __name__ == "__main__":
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
    jobs = [(k, s) for k in KINDS for s in range(1, n + 1)]
    jobs.sort(key=lambda j: j[0] != "c3_ga_toffoli")  # longest first
    with ProcessPoolExecutor(workers) as ex:
        res = list(ex.map(run, jobs))
    out = {"source": "reference isingsynth engines, pkg/tests/test_acceptance.py criteria 3 and 12", "seeds": n}
    for k in KINDS:
        out[k] = {str(s): b for kk, s, b in res if kk == k}
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", OUT)
