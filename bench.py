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
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "circuit fitness evals/sec (whole box) at 3–5 qubits; generations/sec"
N, L, P = 5, 64, 1 << 20


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


def cpu_reference_sample(steps: int, warmup: int, per_worker: int):
    """The reference algorithm's CPU path on all host cores (oracle port)."""
    from oracle.cpu_baseline import CpuPool
    from paper_1809_11134_b200.synthetic import haar_target, qeqea_like_circuits

    pool = CpuPool()
    T = haar_target(N)
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
        "kind": "port",
        "sample": (f"{count} C5-shaped circuits (n=5, L=64, QEQEA gate mix, Haar target) per step, "
                   f"oracle restatement of evaluate_circuit (dense kron matmul per gate), "
                   f"ProcessPool x{pool.workers}, OPENBLAS_NUM_THREADS=1"),
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
        "config": {"workload": "C5 fitness evals (bounded sample per step)", "n": N, "L": L, "P": P},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


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
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1809_11134_b200.synthetic import haar_target
    from paper_1809_11134_b200 import _lib
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    lib = _lib.load()
    peak = ctypes.c_double()
    _lib.check(lib.isq_fma_peak(1, local, ctypes.cast(ctypes.pointer(peak), ctypes.c_void_p)))
    fp64_peak = peak.value / 1e12

    T = haar_target(N)
    cfg = PopulationConfig(number_of_wires=N, size_of_individual=L, size_of_population=P,
                           max_generations=10_000_000, target_fitness=1.0)
    eng = QeqeaEngine(cfg, TargetSpec("haar32", N, T), seed=2024, device=local, rank=rank, world=world,
                      max_batch=max(args.steps + args.warmup, 1) + 1)
    from paper_1809_11134_b200.distributed import Comm, DeviceQeqeaOps

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
        ops.begin_batch()
        for _ in range(args.warmup):
            ops.generation(comm)
        stream.synchronize()
        ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(args.steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(local)
        clocks.start()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            ops.generation(comm, marks=ev[i])
        end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk = clocks.stop()
    ms = start.elapsed_time(end)
    prep_ms = [e[0].elapsed_time(e[1]) for e in ev]
    eval_ms = [e[1].elapsed_time(e[2]) for e in ev]
    fin_ms = [e[2].elapsed_time(e[3]) for e in ev]
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
    avg_eval_s = sum(eval_ms) / len(eval_ms) * 1e-3
    shard_circuits = min(shard, P - rank * shard)
    achieved = canonical_flops(N, L) * shard_circuits / avg_eval_s / 1e12
    traffic = None
    tf = ROOT / "profiles" / "traffic_eval_c5.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
    # executed FP64 pipe utilisation of the same kernel from the committed
    # `ncu --set full` capture (profiles/, not measured by this run)
    pipe_ncu = None
    nf = ROOT / "profiles" / "r01_c5_ncu_full.json"
    if nf.exists():
        for k in json.loads(nf.read_text()):
            if "fitness_fast_kernel<5" in k.get("kernel", ""):
                v = k.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "")
                pipe_ncu = float(v.split()[0]) / 100 if v else None

    out = {
        "metric": METRIC, "value": evals_per_s, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "C5: QEQEA generation, n=5 qubits, depth L=64, population 2^20, "
                               "Haar-random 32x32 target; bank 1.0e9 slots (36 GB) resident in HBM",
                   "n": N, "L": L, "P": P, "global_batch": P,
                   "parallelism": f"dp{world} (circuit shards x position-owned bank shards)"
                                  + (f", {transport} transport" if world > 1 else ""),
                   "l2": "inputs larger than L2 (36 GB bank vs 126 MB)"},
        "gens_per_s": args.steps / (ms * 1e-3),
        "phase_ms": {"prepare (sample + route + lazy mutation + measure; world > 1: + 2 all-to-alls)":
                         sum(prep_ms) / len(prep_ms),
                     "score (fitness kernel)": sum(eval_ms) / len(eval_ms),
                     "finish (world > 1: all-gathers; reduce + commit + table)": sum(fin_ms) / len(fin_ms)},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic,
                     "fp64_pipe_active_ncu": pipe_ncu,
                     "kernel": "fitness_fast_kernel<5> (score phase, one launch per generation)",
                     "peak_source": "FP64 CUDA-core FMA peak measured live by isq_fma_peak "
                                    "(MEASURED_PEAKS.json carries no FP64 figure)",
                     "work": "canonical F(n,L) = (6L+8) 4^n flop/eval (SURVEY.md §8d) x circuits per launch",
                     "note": ("frac > 1 is possible: diagonal gates (Rz, ZZ; 78% of QEQEA gates) cost O(2^n) "
                              "phase updates here, not the canonical 6*4^n; the executed FP64 pipe "
                              "utilisation is fp64_pipe_active_ncu (ncu sm__pipe_fp64_cycles_active of the "
                              "committed capture, profiles/r01_c5_ncu_full.json; DESIGN.md §6)")},
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
    if not args.skip_e2e:
        n_mine = shard_circuits
        if world == 1:
            _, codes, thetas = eng.sample(0, P)  # this generation's C5 circuits
            src = "this generation's C5 circuits"
        else:
            from paper_1809_11134_b200.synthetic import qeqea_like_circuits

            codes, thetas = qeqea_like_circuits(N, L, n_mine, seed=77 + rank)
            src = "QEQEA-mix C5-shaped circuits, P/N per rank"
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
            m = min(n_mine, args.cpu_per_worker * pool.workers)
            cpu_fit, wall = pool.evaluate(N, codes[:m], thetas[:m], T)
            pool.close()
            rel = np.abs(cpu_fit - hf[:m]) / np.maximum(np.abs(cpu_fit), 1e-300)
            out["cpu_baseline"] = {
                "value": m / wall, "unit": "evals/s", "cores": pool.workers, "kind": "port",
                "sample": (f"first {m} circuits of the e2e batch ({src}), oracle restatement of "
                           f"evaluate_circuit (dense kron matmul per gate), ProcessPool x{pool.workers}, "
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
    eng.close()
    # the fp32 variant of the fitness kernel (include/isq.h ISQ_PRECISION_FP32):
    # a full C5 generation with fp32 fitness, and its error on the e2e circuits
    if world == 1 and not args.skip_fp32:
        fe = QeqeaEngine(cfg, TargetSpec("haar32", N, T), seed=2024, device=local, precision="fp32",
                         max_batch=max(args.steps + args.warmup, 1) + 1)
        with torch.cuda.stream(stream):
            fops = DeviceQeqeaOps(fe)
            fops.begin_batch()
            for _ in range(args.warmup):
                fops.generation(None)
            fev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(args.steps)]
            torch.cuda.synchronize()
            start.record(stream)
            for i in range(args.steps):
                fops.generation(None, marks=fev[i])
            end.record(stream)
            torch.cuda.synchronize()
        fms = start.elapsed_time(end)
        fit_ms = sum(e[1].elapsed_time(e[2]) for e in fev) / args.steps
        p32 = ctypes.c_double()
        _lib.check(lib.isq_fma_peak(0, local, ctypes.cast(ctypes.pointer(p32), ctypes.c_void_p)))
        a32 = canonical_flops(N, L) * P / (fit_ms * 1e-3) / 1e12
        var = {"value": P * args.steps / (fms * 1e-3), "unit": "evals/s", "ms_per_step": fms / args.steps,
               "fitness_kernel_ms": fit_ms,
               "roofline": {"bound": "fp32", "achieved": a32, "peak": p32.value / 1e12, "unit": "TFLOP/s",
                            "frac": a32 / (p32.value / 1e12),
                            "peak_source": "FP32 CUDA-core FMA peak measured live by isq_fma_peak"},
               "bound": "|fit32 - fit64| <= 1e-4 |fit64| + 1e-6 (tests/test_fitness_gpu.py)"}
        fe.close()
        if not args.skip_e2e:
            h32 = np.empty_like(hf)
            _lib.check(lib.isq_fitness_batch_ex(N, L, n_mine, _lib.ptr(hc), _lib.ptr(ht), _lib.ptr(Tc),
                                                _lib.ptr(h32), local, _lib.PRECISIONS["fp32"]))
            var["max_abs_err_vs_fp64"] = float(np.abs(h32 - hf).max())
            var["max_rel_err_vs_fp64"] = float((np.abs(h32 - hf) / np.maximum(np.abs(hf), 1e-300)).max())
        out["fp32_variant"] = var
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
    args = ap.parse_args()
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
