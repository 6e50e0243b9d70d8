"""Benchmark of the QEQEA generation loop (BASELINE.json metric: circuit
fitness evals/sec, whole box; generations/sec).

Workload (config C5 of BASELINE.json, the largest single-GPU configuration):
one step = one full QEQEA generation (sample + measure + lazy mutation +
compose + score 2^20 circuits of 64 gates on 5 qubits, reductions, commit,
table update) over a device-resident bank of 1.0e9 slots (36 GB, far above the
126 MB L2), Haar-random target.  At N > 1 (torchrun) the 2^20 circuits are
sharded over the ranks and the bank by slot position: per
generation the touches go to their owners, gate codes / live angles come back
and fitness / shard elites go to every rank — stored by the producing kernels
straight into the peers' buffers over NVLink (`--transport p2p`, default,
ordered by one-element all-reduces) or as NCCL all-to-alls / all-gathers
(`--transport nccl`); no O(P*L) pass is replicated.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` (N > 1) outside torchrun re-launches this script as N ranks
through `torch.distributed.run` on 127.0.0.1 (one process per GPU, NCCL
communicator init logged with NCCL_DEBUG=INFO / SUBSYS=INIT); under torchrun
WORLD_SIZE must equal N.

`--impl reference` times the reference algorithm's CPU path (the oracle port
of evaluate_circuit, dense kron-matmul per gate) on all host cores for a
bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "circuit fitness evals/sec (whole box) at 3–5 qubits; generations/sec"
# BASELINE.json configs: C5 (the headline, default) and C4
CONFIGS = {
    "c5": dict(n=5, L=64, P=1 << 20, target="haar",
               workload="C5: QEQEA generation, n=5 qubits, depth L=64, population 2^20, "
                        "Haar-random 32x32 target; bank 1.0e9 slots (36 GB) resident in HBM",
               l2="inputs larger than L2 (36 GB bank vs 126 MB)"),
    "c4": dict(n=4, L=32, P=1 << 16, target="CCCNOT",
               workload="C4: QEQEA generation on C^3NOT, n=4 qubits, depth L=32, population 2^16; "
                        "bank 2.1e7 slots (738 MB) resident in HBM",
               l2="bank larger than L2 (738 MB vs 126 MB)"),
}
N, L, P = 5, 64, 1 << 20
CONFIG = "c5"


def target_of(name: str, n: int):
    if name == "haar":
        from paper_1809_11134_b200.synthetic import haar_target

        return haar_target(n)
    from paper_1809_11134_b200.fitness import target_matrix

    return target_matrix(name, n).matrix


def kernel_name(n: int, precision: str = "fp64") -> str:
    from paper_1809_11134_b200 import _lib  # noqa: F401  (instantiation names of include/isq.h kernels)

    return f"fitness_fast_kernel<{n}, *, {'double' if precision == 'fp64' else 'float'}>"


def canonical_flops(n: int, L: int) -> int:
    """F(n, L) = (6L + 8) 4^n real flops per fitness eval."""
    return (6 * L + 8) * 4 ** n


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clock and clock-event reasons sampled during the timed region: NVML
    polled every 10 ms from a thread (the device found by its PCI bus id), or
    `nvidia-smi -lms 100` when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.sm, self.mx, self.reasons = [], [], set()
        self._halt = threading.Event()

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        pr = torch.cuda.get_device_properties(self.index)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except pynvml.NVMLError:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        nv, h = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self._halt.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.reasons.update(k for k, b in bits.items() if r & b)
            except nv.NVMLError:
                pass
            self._halt.wait(0.01)

    def start(self):
        try:
            self.nvml = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.nvml is not None:
            self._halt.set()
            self.thread.join(timeout=2)
            src = "nvml (10 ms)"
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            src = "nvidia-smi (100 ms)"
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(self.NAMES, parts[4:8]):
                    if v.lower() == "active":
                        self.reasons.add(nm)
        sm = sorted(self.sm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": src}


# --------------------------------------------------------------- helpers --
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def emit(obj):
    print(json.dumps(obj), flush=True)


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_sample(steps: int, warmup: int, per_worker: int):
    """The reference algorithm's CPU path on all host cores (oracle port).
    The worker pool is spawned and warmed (imports, lru caches) before any
    timed step."""
    from oracle.cpu_baseline import CpuPool
    from paper_1809_11134_b200.synthetic import qeqea_like_circuits

    pool = CpuPool()
    pool.warm(N, L)
    T = target_of(CONFIGS[CONFIG]["target"], N)
    count = per_worker * pool.workers
    times, evals = [], 0
    for i in range(warmup + steps):
        codes, thetas = qeqea_like_circuits(N, L, count, seed=1000 + i)
        _, wall = pool.evaluate(N, codes, thetas, T)
        if i >= warmup:
            times.append(wall)
            evals += count
    pool.close()
    total = sum(times)
    return {
        "value": evals / total,
        "unit": "evals/s",
        "cores": pool.workers,
        "cpu_model": cpu_model(),
        "kind": "port",
        "sample": (f"{count} {CONFIG.upper()}-shaped circuits (n={N}, L={L}, QEQEA gate mix, "
                   f"{CONFIGS[CONFIG]['target']} target) per step, oracle restatement of evaluate_circuit "
                   f"(dense kron matmul per gate), warmed ProcessPool x{pool.workers}, OPENBLAS_NUM_THREADS=1"),
        "ms_per_step": 1000.0 * total / max(1, len(times)),
    }


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cb = cpu_reference_sample(args.steps, args.warmup, per_worker=args.cpu_per_worker)
    emit({
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{CONFIG.upper()} fitness evals (bounded sample per step)", "n": N, "L": L,
                   "P": P},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "cpu_model", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


def _ncu_value(text: str) -> float:
    """'0.605691 Gbyte' / '48.2 %' -> float in base units (bytes, percent)."""
    num, _, unit = str(text).partition(" ")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit.strip(), 1)
    return float(num.replace(",", "")) * scale


def profile_evidence(kernel_prefix: str):
    """(DRAM bytes per launch, FP64 pipe fraction, source) of `kernel_prefix`
    from the committed `ncu --set full` captures (profiles/r*_ncu_full.json,
    newest round first); Nones when no capture of this kernel instantiation
    exists.  Not measured by this run."""
    for f in sorted((ROOT / "profiles").glob("r*_ncu_full.json"), reverse=True):
        try:
            rows = json.loads(f.read_text())
        except (OSError, ValueError):
            continue
        for r in rows:
            if r.get("kernel", "").startswith(kernel_prefix) and "dram__bytes_read.sum" in r:
                traffic = _ncu_value(r["dram__bytes_read.sum"]) + _ncu_value(r.get("dram__bytes_write.sum", "0"))
                pipe = r.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
                return (traffic, _ncu_value(pipe) / 100 if pipe else None,
                        f"{f.relative_to(ROOT)}: {r['kernel'].split('(')[0]}")
    return None, None, None


def time_generations(ops, comm, steps: int, warmup: int, stream, dist=None, clocks=None):
    """Warm-up, then `steps` generations bracketed by CUDA events on the
    handle's stream (barrier + synchronize on both sides); per-generation
    phase events (before prepare, before / after score, after finish)."""
    import torch

    ops.begin_batch()
    for _ in range(warmup):
        ops.generation(comm)
    stream.synchronize()
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks is not None:
        clocks.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    start.record(stream)
    for i in range(steps):
        ops.generation(comm, marks=ev[i])
    end.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    if clocks is not None:
        clocks.clk = clocks.stop()
    ms = start.elapsed_time(end)
    phases = [[e[k].elapsed_time(e[k + 1]) for e in ev] for k in range(3)]
    return ms, [sum(p) / len(p) for p in phases]


def time_engine_steps(cfg, spec, local: int, stream, steps: int, warmup: int):
    """`steps` generations through QeqeaEngine.steps() in its automatic launch
    mode on `stream` (a fresh engine, seed 2024, after `warmup` + `steps`
    untimed generations, so the graphs are captured), CUDA events,
    synchronize on both sides, clocks sampled in between."""
    import torch

    from paper_1809_11134_b200 import _lib
    from paper_1809_11134_b200.engine import QeqeaEngine

    eng = QeqeaEngine(cfg, spec, seed=2024, device=local, max_batch=steps + warmup + 1)
    _lib.check(eng._lib.isq_qeqea_set_stream(eng._handle(), ctypes.c_void_p(stream.cuda_stream)))
    eng.steps(warmup)
    eng.steps(steps)  # also warm: captures the CUDA graphs of this batch's shape
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    rec = eng.steps(steps)
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    assert rec.size == steps
    eng.close()
    return start.elapsed_time(end), clk


def fitness_peak(lib, _lib, local: int, fp64: bool = True) -> float:
    v = ctypes.c_double()
    _lib.check(lib.isq_fma_peak(1 if fp64 else 0, local, ctypes.cast(ctypes.pointer(v), ctypes.c_void_p)))
    return v.value / 1e12


def side_c4(args, local: int, fp64_peak: float, stream):
    """BASELINE config 4 (n=4, L=32, P=2^16, C^3NOT): full generations through
    the engine's own steps() in its automatic launch mode for this size (16-
    generation CUDA graphs), CUDA events on the handle's stream; the phase
    split and the fitness roofline from a plain-kernel pass of the same
    generations (DeviceQeqeaOps)."""
    import torch

    from paper_1809_11134_b200.distributed import DeviceQeqeaOps
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import target_matrix

    c = CONFIGS["c4"]
    steps, warmup = max(args.steps, 48), max(args.warmup, 16)
    cfg = PopulationConfig(number_of_wires=c["n"], size_of_individual=c["L"], size_of_population=c["P"],
                           max_generations=10_000_000, target_fitness=1.0)
    eng = QeqeaEngine(cfg, target_matrix("CCCNOT"), seed=2024, device=local, max_batch=steps + warmup + 1)
    from paper_1809_11134_b200 import _lib

    _lib.check(eng._lib.isq_qeqea_set_stream(eng._handle(), ctypes.c_void_p(stream.cuda_stream)))
    eng.steps(warmup)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    rec = eng.steps(steps)  # enqueues the generations, then reads their records back
    end.record(stream)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    assert rec.size == steps
    eng.close()
    eng = QeqeaEngine(cfg, target_matrix("CCCNOT"), seed=2024, device=local, max_batch=steps + warmup + 1)
    with torch.cuda.stream(stream):
        ops = DeviceQeqeaOps(eng)
        kms, (prep, fit, fin) = time_generations(ops, None, steps, warmup, stream)
    eng.close()
    achieved = canonical_flops(c["n"], c["L"]) * c["P"] / (fit * 1e-3) / 1e12
    return {"workload": c["workload"], "steps": steps, "warmup": warmup,
            "value": c["P"] * steps / (ms * 1e-3), "unit": "evals/s", "gens_per_s": steps / (ms * 1e-3),
            "ms_per_step": ms / steps, "launch": "engine steps(), automatic mode (16-generation CUDA graphs)",
            "plain_kernels_ms_per_step": kms / steps,
            "phase_ms (plain kernels)": {"prepare": prep, "score (fitness kernel)": fit, "finish": fin},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": achieved / fp64_peak, "kernel": kernel_name(c["n"]),
                         "work": "canonical F(4,32) = 51,200 flop/eval x 65,536 circuits per launch"},
            "baseline_md_target": "BASELINE.md section 2: >= 3.6e8 evals/s (fitness at 50% of FP64 peak)"}


def side_fitness_sweep(lib, _lib, fp64_peak: float, stream):
    """The metric's "3-5 qubits": explicit-gate fitness (isq_fitness_batch_device_ex)
    on device-resident QEQEA- and GA-mix circuits, best of 3 trials of 10
    launches each, canonical roofline fraction."""
    import torch

    out = {}
    dev = torch.device("cuda", torch.cuda.current_device())
    for n, L, count in [(3, 16, 1 << 20), (4, 32, 1 << 18), (5, 64, 1 << 18)]:
        nc, K = 3 * n + n * (n - 1) // 2, n + n * (n - 1) // 2
        g = torch.Generator(device=dev).manual_seed(n)
        for mix in ("qeqea", "ga"):
            if mix == "ga":  # uniform over the gate choices (ga.py:47-59)
                codes = torch.randint(0, nc, (count, L), device=dev, dtype=torch.uint8, generator=g)
            else:  # slot kind uniform over K (engine.py:180), measured axis uniform
                kinds = torch.randint(0, K, (count, L), device=dev, generator=g)
                axes = torch.randint(0, 3, (count, L), device=dev, generator=g)
                codes = torch.where(kinds < n, 3 * kinds + axes, 3 * n + (kinds - n)).to(torch.uint8)
            thetas = torch.rand((count, L), device=dev, dtype=torch.float64, generator=g) * 2 * math.pi
            T = torch.eye(2 ** n, dtype=torch.complex128, device=dev)
            outv = torch.empty(count, dtype=torch.float64, device=dev)
            a = (n, L, count, codes.data_ptr(), thetas.data_ptr(), T.data_ptr(), outv.data_ptr(), 0,
                 stream.cuda_stream)
            with torch.cuda.stream(stream):
                for _ in range(3):
                    _lib.check(lib.isq_fitness_batch_device_ex(*a))
                best = None
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(10):
                        lib.isq_fitness_batch_device_ex(*a)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    t = e0.elapsed_time(e1) / 10
                    best = t if best is None else min(best, t)
            ev = count / (best * 1e-3)
            tf = ev * canonical_flops(n, L) / 1e12
            out[f"n{n}_L{L}_{mix}"] = {"circuits": count, "ms": best, "evals_per_s": ev, "canonical_tflops": tf,
                                       "frac_fp64_peak": tf / fp64_peak}
    return out


def side_tiny(local: int):
    """C1-C3 are latency bound (5 / 50 candidates): generations/s through the
    engines' steps() (host wall clock, records read back per call)."""
    from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

    def gps(eng, n):
        eng.steps(100)
        t0 = time.perf_counter()
        r = eng.steps(n)
        return len(r) / (time.perf_counter() - t0)

    t, f = target_matrix("Toffoli"), target_matrix("Fredkin")
    big = dict(max_generations=10 ** 7, target_fitness=1.0)
    return {"unit": "generations/s",
            "C1 QEQEA Toffoli P=5 L=16": gps(QeqeaEngine(PopulationConfig(3, 16, 5, **big), t, 1, device=local), 4000),
            "C2 GA Toffoli P=50 L=16": gps(GaEngine(GaConfig(3, 16, 50, **big), t, 1, device=local), 4000),
            "C3 QEQEA Fredkin P=5 L=16 nMeas=3": gps(QeqeaEngine(PopulationConfig(3, 16, 5, n_meas=3, **big), f, 1,
                                                                 device=local), 4000)}


def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_env()
    # ISQ_BENCH_SHARE_GPU=1: functional check of the N > 1 code path with every
    # rank on GPU 0 (gloo, host barriers); its timings mean nothing
    share = world > 1 and os.environ.get("ISQ_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    if world > 1 and not share and torch.cuda.device_count() < world:
        print(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPUs", file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    red_dev = "cpu" if share else f"cuda:{local}"
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1809_11134_b200 import _lib
    from paper_1809_11134_b200.distributed import Comm, DeviceQeqeaOps
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    lib = _lib.load()
    fp64_peak = fitness_peak(lib, _lib, local)
    conf = CONFIGS[CONFIG]
    T = target_of(conf["target"], N)
    cfg = PopulationConfig(number_of_wires=N, size_of_individual=L, size_of_population=P,
                           max_generations=10_000_000, target_fitness=1.0)
    eng = QeqeaEngine(cfg, TargetSpec(conf["target"], N, T), seed=2024, device=local, rank=rank, world=world,
                      max_batch=max(args.steps + args.warmup, 1) + 1)
    stream = torch.cuda.Stream(device=local)
    with torch.cuda.stream(stream):
        ops = DeviceQeqeaOps(eng, args.transport)  # binds the handle to `stream`
        comm = Comm() if world > 1 else None
        shard = ops.S
        transport = args.transport if world > 1 else None
        if world > 1 and args.transport == "p2p":
            # map every rank's exchange buffers (CUDA IPC over NVLink); if any
            # rank cannot, every rank falls back to the NCCL collectives
            err = ""
            try:
                comm.connect_peers(ops)
            except Exception as exc:  # noqa: BLE001 - reported in the JSON line
                err = str(exc).splitlines()[0][:200]
            ok = torch.tensor([0 if err else 1], device=red_dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                _lib.check(lib.isq_qeqea_set_peers(eng._handle(), None))
                ops.transport = "nccl"
                transport = f"nccl (p2p unavailable: {err or 'on another rank'})"
        clocks = ClockSampler(local)
        ms, (prep_ms, eval_ms, fin_ms) = time_generations(ops, comm, args.steps, args.warmup, stream, dist, clocks)
        clk = clocks.clk
    launch = "plain kernel launches (DeviceQeqeaOps)"
    plain_ms = None
    if CONFIG == "c4" and world == 1:
        # C4 generations are short enough for the engine's automatic mode to
        # batch them into CUDA graphs: the timed line is the engine's own
        # steps() in that mode (same seed, same generations), the phase split
        # above the plain-kernel pass
        plain_ms = ms
        ms, clk = time_engine_steps(cfg, TargetSpec(conf["target"], N, T), local, stream, args.steps, args.warmup)
        launch = "engine steps(), automatic mode (16-generation CUDA graphs); phase_ms from plain kernels"
    if world > 1:
        t = torch.tensor([ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    rec, _ = ops.read_batch()
    assert rec.size == args.steps + args.warmup, rec.size
    ranks_agree = None
    if world > 1:
        # the reductions are replicated: every rank must hold the same records
        mine = torch.tensor([float(rec["gen_best"].sum()), float(rec["gen_mean"].sum()),
                             float(rec["best_fitness"][-1])], device=red_dev, dtype=torch.float64)
        lo, hi = mine.clone(), mine.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        ranks_agree = bool(torch.equal(lo, hi))

    evals_per_s = P * args.steps / (ms * 1e-3)
    shard_circuits = min(shard, P - rank * shard)
    achieved = canonical_flops(N, L) * shard_circuits / (eval_ms * 1e-3) / 1e12
    kname = kernel_name(N)
    kprefix = f"fitness_fast_kernel<{N},"
    traffic, pipe, prof_src = profile_evidence(f"void {kprefix}")

    out = {
        "metric": METRIC, "value": evals_per_s, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": conf["workload"], "n": N, "L": L, "P": P, "global_batch": P,
                   "parallelism": f"dp{world} (circuit shards x position-owned bank shards)"
                                  + (f", {transport} transport" if world > 1 else ""),
                   "l2": conf["l2"]},
        "gens_per_s": args.steps / (ms * 1e-3),
        "launch": launch,
        **({"plain_kernels_ms_per_step": plain_ms / args.steps} if plain_ms is not None else {}),
        "phase_ms": {"prepare (sample + route + lazy mutation + measure; world > 1: + 2 all-to-alls)": prep_ms,
                     "score (fitness kernel)": eval_ms,
                     "finish (world > 1: all-gathers; reduce + commit + table)": fin_ms},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic, "fp64_pipe_active_ncu": pipe,
                     "profile_source": prof_src,
                     "kernel": f"{kname} (score phase, one launch per generation)",
                     "peak_source": "FP64 CUDA-core FMA peak measured live by isq_fma_peak "
                                    "(MEASURED_PEAKS.json carries no FP64 figure)",
                     "work": f"canonical F(n,L) = (6L+8) 4^n = {canonical_flops(N, L)} flop/eval (SURVEY.md §8d) "
                             f"x {shard_circuits} circuits per launch",
                     "note": ("frac > 1 is possible: diagonal gates (Rz, ZZ) cost O(2^n) phase updates here, not "
                              "the canonical 6*4^n; fp64_pipe_active_ncu is the executed FP64 pipe utilisation "
                              "and traffic the DRAM bytes per launch of the same kernel instantiation from the "
                              "committed ncu capture named in profile_source (not measured by this run; "
                              "DESIGN.md §6)")},
        "clocks": clk,
        **({"shared_gpu_functional_check": True} if share else {}),
        # per generation: sample, values, fitness, 2 reductions, commit, advance;
        # world > 1 adds route, unroute, elite (+ the fitness broadcast with p2p)
        "gpu_launches": (7 if world == 1 else (11 if ops.transport == "p2p" else 10)) * args.steps,
        "best_fitness": float(rec["best_fitness"][-1]),
        **({"ranks_agree": ranks_agree} if world > 1 else {}),
    }

    # e2e: the same metric through the C-ABI with host buffers (isq_fitness_batch:
    # pinned host codes/angles -> device, fitness -> host inside the timed
    # region), every rank on its shard of the circuits, max over ranks
    hc = ht = hf = Tc = None
    n_mine = shard_circuits
    if not args.skip_e2e:
        if world == 1:
            _, codes, thetas = eng.sample(0, P)  # this generation's circuits
            src = f"this generation's {CONFIG.upper()} circuits"
        else:
            from paper_1809_11134_b200.synthetic import qeqea_like_circuits

            codes, thetas = qeqea_like_circuits(N, L, n_mine, seed=77 + rank)
            src = f"QEQEA-mix {CONFIG.upper()}-shaped circuits, P/N per rank"
        hc = torch.empty((n_mine, L), dtype=torch.uint8, pin_memory=True).numpy()
        ht = torch.empty((n_mine, L), dtype=torch.float64, pin_memory=True).numpy()
        hf = torch.empty(n_mine, dtype=torch.float64, pin_memory=True).numpy()
        hc[:] = codes
        ht[:] = thetas
        Tc = np.ascontiguousarray(T, dtype=np.complex128)

        def batch():
            _lib.check(lib.isq_fitness_batch(N, L, n_mine, _lib.ptr(hc), _lib.ptr(ht), _lib.ptr(Tc),
                                             _lib.ptr(hf), None, local))

        for _ in range(max(1, args.warmup)):
            batch()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            batch()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device=red_dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        out["e2e"] = {"value": P * args.steps / dt, "unit": "evals/s",
                      "h2d_bytes_per_step": int(world * (hc.nbytes + ht.nbytes + Tc.nbytes)),
                      "d2h_bytes_per_step": int(world * hf.nbytes),
                      "path": f"isq_fitness_batch (C ABI, pinned host buffers) on {src}"}
        # CPU baseline on the first circuits of rank 0's batch, which is also a
        # parity spot-check of the GPU result
        if rank == 0 and not args.skip_cpu:
            from oracle.cpu_baseline import CpuPool

            pool = CpuPool()
            pool.warm(N, L)
            m = min(n_mine, args.cpu_per_worker * pool.workers)
            cpu_fit, wall = pool.evaluate(N, codes[:m], thetas[:m], T)
            pool.close()
            rel = np.abs(cpu_fit - hf[:m]) / np.maximum(np.abs(cpu_fit), 1e-300)
            out["cpu_baseline"] = {
                "value": m / wall, "unit": "evals/s", "cores": pool.workers, "cpu_model": cpu_model(),
                "kind": "port",
                "sample": (f"first {m} circuits of the e2e batch ({src}), oracle restatement of "
                           f"evaluate_circuit (dense kron matmul per gate), warmed ProcessPool x{pool.workers}, "
                           f"OPENBLAS_NUM_THREADS=1"),
                "parity_max_rel_err_vs_gpu": float(rel.max()),
            }
    # the reference's own call: QeqeaEngine.step() (engine.py:318-361), one
    # generation per call with its (max, mean) read back to the host, wall
    # clock around K calls (ctypes + launch + the synchronising record read)
    if world == 1 and not args.skip_e2e:
        eng.step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            eng.step()
        dt = time.perf_counter() - t0
        out["api_step"] = {"value": P * args.steps / dt, "unit": "evals/s", "ms_per_step": dt * 1e3 / args.steps,
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(_lib.GEN_RECORD.itemsize),
                           "path": "QeqeaEngine.step() through the C ABI (isq_qeqea_step), host wall clock"}
    if world > 1:
        dist.barrier()  # no rank unmaps / frees exchange buffers a peer may still store into
    eng.close()
    # the fp32 variant of the fitness kernel (include/isq.h ISQ_PRECISION_FP32):
    # a full generation with fp32 fitness, and its error on the e2e circuits
    if world == 1 and not args.skip_fp32:
        fe = QeqeaEngine(cfg, TargetSpec(conf["target"], N, T), seed=2024, device=local, precision="fp32",
                         max_batch=max(args.steps + args.warmup, 1) + 1)
        with torch.cuda.stream(stream):
            fops = DeviceQeqeaOps(fe)
            fms, (_, fit_ms, _) = time_generations(fops, None, args.steps, args.warmup, stream)
        p32 = fitness_peak(lib, _lib, local, fp64=False)
        a32 = canonical_flops(N, L) * P / (fit_ms * 1e-3) / 1e12
        var = {"value": P * args.steps / (fms * 1e-3), "unit": "evals/s", "ms_per_step": fms / args.steps,
               "fitness_kernel_ms": fit_ms,
               "roofline": {"bound": "fp32", "achieved": a32, "peak": p32, "unit": "TFLOP/s", "frac": a32 / p32,
                            "peak_source": "FP32 CUDA-core FMA peak measured live by isq_fma_peak"},
               "bound": "|fit32 - fit64| <= 1e-4 |fit64| + 1e-6 (tests/test_fitness_gpu.py)"}
        fe.close()
        if hf is not None:
            h32 = np.empty_like(hf)
            _lib.check(lib.isq_fitness_batch_ex(N, L, n_mine, _lib.ptr(hc), _lib.ptr(ht), _lib.ptr(Tc),
                                                _lib.ptr(h32), local, _lib.PRECISIONS["fp32"]))
            var["max_abs_err_vs_fp64"] = float(np.abs(h32 - hf).max())
            var["max_rel_err_vs_fp64"] = float((np.abs(h32 - hf) / np.maximum(np.abs(hf), 1e-300)).max())
        out["fp32_variant"] = var
    # side measurements (N = 1, headline config): BASELINE config 4, the
    # explicit-gate fitness kernels at n = 3/4/5, and the latency-bound C1-C3
    if world == 1 and CONFIG == "c5" and not args.skip_extras:
        out["c4"] = side_c4(args, local, fp64_peak, stream)
        out["fitness_sweep"] = side_fitness_sweep(lib, _lib, fp64_peak, stream)
        out["tiny"] = side_tiny(local)
    if rank == 0:
        emit(out)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> None:
    """--gpus N: become one rank of N.  Under torchrun WORLD_SIZE must be N;
    otherwise (N > 1) re-exec through torch.distributed.run and exit with
    its status."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}", file=sys.stderr)
            sys.exit(2)
        return
    if args.gpus <= 1 or (args.impl == "reference" and not args.launch_check):
        return  # the reference arm runs on rank 0 only
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"), *sys.argv[1:]]
    print("bench.py: launching " + " ".join(cmd[1:]), file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd, env=env))


def launch_check(args) -> None:
    """--launch-check: the rank plumbing alone (gloo, no GPU work): every rank
    joins the process group, rank 0 prints the world it saw."""
    import torch
    import torch.distributed as dist

    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([rank + 1])
        dist.all_reduce(t)
        ranks_sum = int(t.item())
        dist.destroy_process_group()
    else:
        ranks_sum = 1
    if rank == 0:
        emit({"launch_check": True, "n_gpus": world, "ranks_sum": ranks_sum, "impl": args.impl})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-fp32", action="store_true")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1: kernels store into peers over NVLink (p2p) or NCCL collectives between phases")
    ap.add_argument("--cpu-per-worker", type=int, default=400)
    ap.add_argument("--launch-check", action="store_true", help="test the rank launcher only (gloo, no GPU)")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5",
                    help="BASELINE.json configuration of the timed generation (c5: the headline)")
    ap.add_argument("--skip-extras", action="store_true",
                    help="c5 at N=1: skip the C4 / fitness-sweep / tiny-config side measurements")
    args = ap.parse_args()
    global N, L, P, CONFIG
    c = CONFIGS[args.config]
    N, L, P, CONFIG = c["n"], c["L"], c["P"], args.config
    launch_ranks(args)
    if args.launch_check:
        launch_check(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
