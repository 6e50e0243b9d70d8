"""Cost of the CPU baseline's oracle port against the reference's own
evaluate_circuit, same circuits, one core (build container: imports the
reference from /root/reference/pkg/src).  bench.py's `--impl reference` arm
and `cpu_baseline` leg time the port (it travels to the GPU box; the
reference cannot), so this records how faithful the port is in cost.

    OPENBLAS_NUM_THREADS=1 python tools/port_vs_reference.py > profiles/r02_port_vs_reference.json
"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
from isingsynth import engine as R_eng  # noqa: E402
from isingsynth.gates import enumerate_templates  # noqa: E402

from oracle.qeqea import circuit_fitness  # noqa: E402
from paper_1809_11134_b200.synthetic import haar_target  # noqa: E402


def main():
    out = {"cores": 1, "cpu": [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                               if ln.startswith("model name")][0]}
    for n, L, count in [(3, 16, 2000), (4, 32, 600), (5, 64, 300)]:
        cfg = R_eng.PopulationConfig(number_of_wires=n, size_of_individual=L, size_of_population=4096)
        rng = np.random.default_rng(n)
        pop = R_eng.init_population(cfg, rng)
        bank = R_eng.construct_segments(pop, cfg, enumerate_templates(n), rng)
        bps = [R_eng.sample_circuit(cfg, rng) for _ in range(count)]
        T = haar_target(n)
        # the same circuits as explicit (code, theta) rows for the port
        codes = np.empty((count, L), dtype=np.uint8)
        thetas = np.empty((count, L))
        for c, bp in enumerate(bps):
            for p, f in enumerate(bp):
                g = bank.descriptor(int(f))
                if g.kind == "rotation":
                    codes[c, p] = 3 * (g.wire - 1) + int(g.axis)
                else:
                    pairs = [t.pair for t in enumerate_templates(n)]
                    codes[c, p] = 3 * n + pairs.index(g.pair)
                thetas[c, p] = g.theta
        t0 = time.perf_counter()
        ref = [R_eng.evaluate_circuit(bp, bank, T) for bp in bps]
        t_ref = time.perf_counter() - t0
        t0 = time.perf_counter()
        port = [circuit_fitness(codes[c], thetas[c], T, n) for c in range(count)]
        t_port = time.perf_counter() - t0
        err = float(np.max(np.abs(np.array(ref) - np.array(port)) / np.maximum(np.abs(ref), 1e-300)))
        out[f"n{n}_L{L}"] = {"circuits": count, "reference_evals_per_s": count / t_ref,
                             "port_evals_per_s": count / t_port, "port_over_reference": t_ref / t_port,
                             "max_rel_diff": err}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
