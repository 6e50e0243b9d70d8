"""Kernel micro-benchmarks (device-resident inputs, CUDA events)."""
import ctypes
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_1809_11134_b200 import _lib


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-peak", action="store_true")
    ap.add_argument("--mix", default="", help="ga | qeqea (default both)")
    ap.add_argument("--prec", default="", help="fp64 | fp32 (default both)")
    args_ = ap.parse_args()
    lib = _lib.load()
    res = {"fp64_peak_tflops": 36.5}
    for fp64 in (() if args_.no_peak else (1, 0)):
        v = ctypes.c_double()
        _lib.check(lib.isq_fma_peak(fp64, 0, ctypes.cast(ctypes.pointer(v), ctypes.c_void_p)))
        res["fp64_peak_tflops" if fp64 else "fp32_peak_tflops"] = v.value / 1e12
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream()
    for prec_name, prec in (("fp64", 0), ("fp32", 1)):
        if args_.prec and prec_name != args_.prec:
            continue
        for mix in ("ga", "qeqea"):
            if args_.mix and mix != args_.mix:
                continue
            for n, L, count in [(3, 16, 1 << 20), (4, 32, 1 << 18), (5, 64, 1 << 18)]:
                if args_.only and f"n{n}" != args_.only:
                    continue
                nc = 3 * n + n * (n - 1) // 2
                K = n + n * (n - 1) // 2
                g = torch.Generator(device=dev).manual_seed(1)
                if mix == "ga":  # uniform over the gate choices (ga.py:47-59)
                    codes = torch.randint(0, nc, (count, L), device=dev, dtype=torch.uint8, generator=g)
                else:  # QEQEA: slot kind uniform over K, measured axis uniform
                    kinds = torch.randint(0, K, (count, L), device=dev, generator=g)
                    axes = torch.randint(0, 3, (count, L), device=dev, generator=g)
                    codes = torch.where(kinds < n, 3 * kinds + axes, 3 * n + (kinds - n)).to(torch.uint8)
                thetas = torch.rand((count, L), device=dev, dtype=torch.float64, generator=g) * 2 * math.pi
                T = torch.eye(2 ** n, dtype=torch.complex128, device=dev)
                out = torch.empty(count, dtype=torch.float64, device=dev)
                args = (n, L, count, codes.data_ptr(), thetas.data_ptr(), T.data_ptr(), out.data_ptr(), prec,
                        stream.cuda_stream)
                for _ in range(3):
                    _lib.check(lib.isq_fitness_batch_device_ex(*args))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = args_.reps
                trials = []
                for _ in range(3):  # best of 3 trials (the first can run before the clocks settle)
                    e0.record()
                    for _ in range(reps):
                        lib.isq_fitness_batch_device_ex(*args)
                    e1.record()
                    torch.cuda.synchronize()
                    trials.append(e0.elapsed_time(e1) / reps)
                ms = min(trials)
                evals = count / (ms * 1e-3)
                flop = (6 * L + 8) * 4 ** n
                res[f"{prec_name}_{mix}_n{n}_L{L}_P{count}"] = {
                    "ms": ms, "evals_per_s": evals, "canon_tflops": evals * flop / 1e12,
                    "frac_fp64_peak": evals * flop / 1e12 / res["fp64_peak_tflops"],
                    "trials_ms": trials}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
