"""Population sharding across the GPUs of one box.

One process per GPU (torchrun).  Every rank holds an identical replica of the
bank (QEQEA) or of the genomes (GA) and evaluates only its shard of the P
candidates: rank r scores circuits [r*S, (r+1)*S), S = ceil(P / world).  The
only per-generation exchange is an all-gather of the fitness shards (P fp64,
1 MiB per rank at C5) over NCCL / NVLink; every rank then replays the
O(P*L) reductions, commit and table update (QEQEA) or SUS + breeding (GA)
identically from counter-based RNG streams, so the replicas never diverge
and no genome or bank traffic crosses the links.

`ShardedRunner` is transport-agnostic: it drives an `ops` object

    ops.begin_batch()            mark the record window
    ops.eval()                   score this rank's shard into ops.fitness_full
    ops.finish()                 replay the generation's tail on the gathered vector
    ops.read_batch() -> (records, stop_reason_code)
    ops.fitness_full / ops.shard_len   the full (padded) fitness tensor, shard size

and a torch.distributed process group; the device ops bind libisq handles
(`DeviceQeqeaOps`, `DeviceGaOps`), the CPU tests bind the oracle.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from .engine import STOP_REASONS


class _CAI:
    """__cuda_array_interface__ view of a libisq-owned fp64 device buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class ShardedRunner:
    def __init__(self, ops, group=None):
        import torch.distributed as dist

        self.ops = ops
        self.group = group
        self.dist = dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.generation = 0
        self.best_fitness = 0.0
        self.stop_reason: Optional[str] = None

    @property
    def done(self) -> bool:
        return self.stop_reason is not None

    def _exchange(self):
        full, S = self.ops.fitness_full, self.ops.shard_len
        mine = full[self.rank * S:(self.rank + 1) * S].clone()
        self.dist.all_gather_into_tensor(full, mine, group=self.group)

    def steps(self, n: int) -> np.ndarray:
        """Up to n generations; stops where the single-device engine would."""
        out = []
        remaining = int(n)
        while remaining > 0 and not self.done:
            k = min(remaining, getattr(self.ops, "max_batch", remaining))
            self.ops.begin_batch()
            for _ in range(k):
                self.ops.eval()
                self._exchange()
                self.ops.finish()
            rec, stop = self.ops.read_batch()
            if rec.size:
                self.generation += int(rec.size)
                self.best_fitness = float(rec["best_fitness"][-1])
            self.stop_reason = STOP_REASONS[int(stop)]
            out.append(rec)
            remaining -= k
        return np.concatenate(out) if out else np.zeros(0, dtype=_lib.GEN_RECORD)


class _DeviceOps:
    _prefix = ""

    def __init__(self, engine):
        import torch

        self.engine = engine
        self.lib = engine._lib
        self.h = engine._handle()
        self.max_batch = engine.max_batch
        self.stream = torch.cuda.current_stream(engine.device)
        f = getattr(self.lib, f"isq_{self._prefix}_set_stream")
        _lib.check(f(self.h, ctypes.c_void_p(self.stream.cuda_stream)))
        ptr, shard = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(getattr(self.lib, f"isq_{self._prefix}_buffers")(self.h, ctypes.byref(ptr),
                                                                     ctypes.byref(shard), None))
        self.shard_len = int(shard.value)
        self.fitness_full = torch.as_tensor(_CAI(ptr.value, self.shard_len * engine.world),
                                            device=f"cuda:{engine.device}")

    def _call(self, name, *args):
        _lib.check(getattr(self.lib, f"isq_{self._prefix}_{name}")(self.h, *args))

    def begin_batch(self):
        self._call("begin_batch")

    def eval(self):
        self._call("eval")

    def finish(self):
        self._call("finish")

    def read_batch(self):
        rec = np.zeros(self.max_batch, dtype=_lib.GEN_RECORD)
        nd, stop = ctypes.c_int32(), ctypes.c_int32()
        self._call("read_batch", _lib.ptr(rec), ctypes.byref(nd), ctypes.byref(stop), None, None)
        return rec[: nd.value], int(stop.value)


class DeviceQeqeaOps(_DeviceOps):
    _prefix = "qeqea"


class DeviceGaOps(_DeviceOps):
    _prefix = "ga"


def sharded_qeqea(cfg, target, seed: int, group=None, **kw) -> ShardedRunner:
    """A QEQEA run sharded over the process group (one GPU per rank)."""
    import torch
    import torch.distributed as dist

    from .engine import QeqeaEngine

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device()
    eng = QeqeaEngine(cfg, target, seed, device=dev, rank=rank, world=world, **kw)
    runner = ShardedRunner(DeviceQeqeaOps(eng), group)
    runner.engine = eng
    return runner


def sharded_ga(cfg, target, seed: int, group=None, **kw) -> ShardedRunner:
    """A GA run sharded over the process group (one GPU per rank)."""
    import torch
    import torch.distributed as dist

    from .ga import GaEngine

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device()
    eng = GaEngine(cfg, target, seed, device=dev, rank=rank, world=world, **kw)
    runner = ShardedRunner(DeviceGaOps(eng), group)
    runner.engine = eng
    return runner
