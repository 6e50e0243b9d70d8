"""Fitness throughput of the block-per-circuit kernel (n = 6 .. 10) on
device-resident circuits (QEQEA-like gate mix, identity target), CUDA events."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1809_11134_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream()
    out = {}
    for n, L, count in [(6, 32, 1 << 14), (7, 32, 1 << 12), (8, 32, 1 << 11), (10, 16, 1 << 8)]:
        nc, K = 3 * n + n * (n - 1) // 2, n + n * (n - 1) // 2
        g = torch.Generator(device=dev).manual_seed(n)
        kinds = torch.randint(0, K, (count, L), device=dev, generator=g)
        axes = torch.randint(0, 3, (count, L), device=dev, generator=g)
        codes = torch.where(kinds < n, 3 * kinds + axes, 3 * n + (kinds - n)).to(torch.uint8)
        thetas = torch.rand((count, L), device=dev, dtype=torch.float64, generator=g) * 2 * math.pi
        T = torch.eye(2 ** n, dtype=torch.complex128, device=dev)
        fit = torch.empty(count, dtype=torch.float64, device=dev)
        a = (n, L, count, codes.data_ptr(), thetas.data_ptr(), T.data_ptr(), fit.data_ptr(), 0, s.cuda_stream)
        with torch.cuda.stream(s):
            _lib.check(lib.isq_fitness_batch_device_ex(*a))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(3):
                lib.isq_fitness_batch_device_ex(*a)
            e1.record(s)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out[f"n{n}_L{L}"] = {"circuits": count, "ms": round(ms, 3), "evals_per_s": round(count / ms * 1e3)}
        print(n, out[f"n{n}_L{L}"], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
