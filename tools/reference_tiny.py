"""the reference's own step() rate at the latency-bound
configurations C1-C3 (build container: imports the reference from
/root/reference/pkg/src; it does not exist on the GPU box, so the numbers are
recorded here, beside the device's `tiny` bench side measurement).  One
process per seed; "box" runs os.cpu_count() seeds in a process pool.

    OPENBLAS_NUM_THREADS=1 python tools/reference_tiny.py > profiles/r02_reference_tiny.json
"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

from isingsynth.engine import PopulationConfig, QeqeaEngine  # noqa: E402
from isingsynth.fitness import TargetSpec, target_matrix  # noqa: E402
from isingsynth.ga import GaConfig, GaEngine  # noqa: E402

BIG = dict(max_generations=10 ** 7, target_fitness=1.0)


def _fredkin():
    import numpy as np

    m = np.eye(8, dtype=np.complex128)
    m[[5, 6], [5, 6]] = 0.0
    m[5, 6] = m[6, 5] = 1.0
    return TargetSpec("Fredkin", 3, m)


def _engine(kind, seed):
    if kind == "C1":
        return QeqeaEngine(PopulationConfig(3, 16, 5, **BIG), target_matrix("Toffoli"), seed)
    if kind == "C2":
        return GaEngine(GaConfig(3, 16, 50, **BIG), target_matrix("Toffoli"), seed)
    return QeqeaEngine(PopulationConfig(3, 16, 5, n_meas=3, **BIG), _fredkin(), seed)


def gens_per_s(kind, seed=1, seconds=10.0):
    eng = _engine(kind, seed)
    for _ in range(20):
        eng.step()
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        eng.step()
        n += 1
    return n / (time.perf_counter() - t0)


def main():
    cores = os.cpu_count()
    out = {"unit": "generations/s", "cpu": [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                                            if ln.startswith("model name")][0], "cores": cores,
           "configs": {"C1": "QEQEA Toffoli P=5 L=16", "C2": "GA Toffoli P=50 L=16",
                       "C3": "QEQEA Fredkin P=5 L=16 nMeas=3"}}
    for kind in ("C1", "C2", "C3"):
        one = gens_per_s(kind)
        with ProcessPoolExecutor(cores) as ex:
            box = sum(ex.map(gens_per_s, [kind] * cores, range(1, cores + 1)))
        out[kind] = {"one_process": round(one, 1), "box_independent_seeds": round(box, 1)}
        print(kind, out[kind], file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
