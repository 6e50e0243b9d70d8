"""GA generation time at large populations (phase split with a plain-kernel
engine): where a P = 2^16 .. 2^20 GaEngine generation spends its time."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1809_11134_b200 import GaConfig, GaEngine  # noqa: E402
from paper_1809_11134_b200.fitness import TargetSpec  # noqa: E402
from paper_1809_11134_b200.synthetic import haar_target  # noqa: E402


def main():
    out = {}
    for n, L, P in [(4, 32, 1 << 16), (5, 64, 1 << 18), (5, 64, 1 << 20)]:
        eng = GaEngine(GaConfig(n, L, P, max_generations=10 ** 6, target_fitness=1.0),
                       TargetSpec("haar", n, haar_target(n)), 1)
        eng.steps(3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k = 5
        eng.steps(k)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / k * 1e3
        out[f"n{n} L{L} P{P}"] = {"ms_per_gen": round(ms, 3), "evals_per_s": round(P / ms * 1e3)}
        print(n, L, P, out[f"n{n} L{L} P{P}"], flush=True)
        eng.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
