"""H2D bandwidth from pinned memory and the isq_fitness_batch pipeline at C5 shape."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_1809_11134_b200 import _lib
from paper_1809_11134_b200.synthetic import haar_target, qeqea_like_circuits

for mb in (75, 603):
    h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"H2D {mb} MB: {mb / 1024 / dt:.1f} GB/s ({dt*1e3:.2f} ms)")
P, L, N = 1 << 20, 64, 5
codes, thetas = qeqea_like_circuits(N, L, P, seed=1)
hc = torch.empty((P, L), dtype=torch.uint8, pin_memory=True).numpy(); hc[:] = codes
ht = torch.empty((P, L), dtype=torch.float64, pin_memory=True).numpy(); ht[:] = thetas
hf = torch.empty(P, dtype=torch.float64, pin_memory=True).numpy()
T = np.ascontiguousarray(haar_target(5))
lib = _lib.load()
for _ in range(2):
    _lib.check(lib.isq_fitness_batch(N, L, P, _lib.ptr(hc), _lib.ptr(ht), _lib.ptr(T), _lib.ptr(hf), None, 0))
t0 = time.perf_counter()
for _ in range(5):
    _lib.check(lib.isq_fitness_batch(N, L, P, _lib.ptr(hc), _lib.ptr(ht), _lib.ptr(T), _lib.ptr(hf), None, 0))
dt = (time.perf_counter() - t0) / 5
print(f"isq_fitness_batch 2^20 x 64: {dt*1e3:.2f} ms, {P/dt/1e6:.1f}M evals/s")
