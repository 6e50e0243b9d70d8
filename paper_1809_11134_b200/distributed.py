"""Population sharding across the GPUs of one box.

One process per GPU (torchrun).  Rank r of `world`:

* scores circuits [r*S, (r+1)*S) (S = ceil(P / world));
* owns the bank slots of positions [b[r], b[r+1]) of every slot kind and
  individual (b = `position_bounds(L, world)`).  A slot's position is fixed by
  Eq. 9 (engine.py:82-87), so every touch of position p goes to the same owner
  and the owners' bank shards never overlap.

Per QEQEA generation (include/isq.h split-phase protocol):

    prepare   sample this rank's circuits, group their touches by owner
    a2a       flat slots -> owners                      (S*L*4 B per rank)
    values    owners: live slot (lazy mutation) + measured gate code
    a2a       gate codes + live angles -> circuit ranks (S*L*9 B per rank)
    score     compose + score this rank's circuits, shard elite record
    gather    fitness (P fp64) + elite records          (all-gather)
    finish    reductions (replicated on the gathered vector), best gates from
              the elite of the rank holding them, commit + table update of
              the owned touches only

Two transports move the data, with identical results:

* "p2p" (default of sharded_qeqea / bench.py): every rank's exchange buffers
  are mapped into every process (CUDA IPC); route, values, the fitness
  broadcast and elite kernels store straight into the consuming ranks'
  buffers over NVLink while they compute, and four stream-ordered
  one-element all-reduces order the phases;
* "nccl": the a2a / gather steps are NCCL collectives between the phases.

So every O(P*L) pass (sampling, bank gathers, commit) and the O(P*L*4^n)
fitness are divided by `world`; only the O(P) reduction is replicated.
GA (`ga.py`): genomes are replicated, rank r scores its genome shard, the
fitness vector is all-gathered and every rank breeds identically from the
counter streams.

`ShardedRunner` drives an `ops` object through `ops.generation(comm)`; the
device ops bind libisq handles (`DeviceQeqeaOps`, `DeviceGaOps`), the CPU tests
bind oracle replicas, and `Comm` is the only code that calls torch.distributed.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional

import numpy as np

from . import _lib
from .engine import STOP_REASONS, position_bounds


class Routing:
    """Split sizes of the two all-to-alls (shared by the device and test ops).

    Exchange layout: the touches a circuit rank sends to owner o form a
    block of S x Lr(o) entries (row = circuit, column = owned position) at
    offset S * b[o]; an owner receives world blocks of S x Lr(r), i.e. one row
    per global (padded) circuit."""

    def __init__(self, length: int, shard: int, world: int, rank: int):
        self.L, self.S, self.world, self.rank = int(length), int(shard), int(world), int(rank)
        self.bounds = position_bounds(self.L, self.world)
        self.widths = [self.bounds[o + 1] - self.bounds[o] for o in range(self.world)]
        self.Lr = self.widths[self.rank]

    @property
    def to_owners(self) -> List[int]:
        """Send splits of the flats (and receive splits of the codes / angles)."""
        return [self.S * w for w in self.widths]

    @property
    def from_circuits(self) -> List[int]:
        """Receive splits of the flats (and send splits of the codes / angles)."""
        return [self.S * self.Lr] * self.world

    def route(self, circuit_major: np.ndarray) -> np.ndarray:
        """(S, L) -> owner-grouped flat layout (host restatement of qeqea_route_kernel)."""
        return np.concatenate([circuit_major[:, self.bounds[o]:self.bounds[o + 1]].reshape(-1)
                               for o in range(self.world)])

    def unroute(self, grouped: np.ndarray) -> np.ndarray:
        """Owner-grouped flat layout -> (S, L) (host restatement of qeqea_unroute_kernel)."""
        out = np.empty((self.S, self.L), dtype=grouped.dtype)
        for o in range(self.world):
            off = self.S * self.bounds[o]
            out[:, self.bounds[o]:self.bounds[o + 1]] = grouped[off:off + self.S * self.widths[o]].reshape(
                self.S, self.widths[o])
        return out


class Comm:
    """The collectives of one generation over a torch.distributed group."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._token = None

    def barrier(self):
        """Stream-ordered barrier of the peer transport: a one-element
        all-reduce (NCCL: on the current stream, no host synchronisation)."""
        import torch

        if self.dist.get_backend(self.group) == "gloo":
            # host barrier: this rank's kernels must have completed first
            torch.cuda.current_stream().synchronize()
            self.dist.barrier(group=self.group)
            return
        if self._token is None:
            self._token = torch.zeros(1, dtype=torch.int32, device=torch.cuda.current_device())
        self.dist.all_reduce(self._token, group=self.group)

    def connect_peers(self, ops):
        """Exchange the exchange-buffer IPC handles and map every rank's into
        this process (isq_qeqea_ipc_export / _ipc_open)."""
        mine = ops.ipc_handles()
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        ops.open_peers_ipc(allh)

    def all_to_all(self, out, inp, out_splits: List[int], in_splits: List[int]):
        self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def all_gather(self, full, chunk: int):
        """In-place all-gather: rank r contributes full[r*chunk:(r+1)*chunk]."""
        mine = full[self.rank * chunk:(self.rank + 1) * chunk].clone()
        self.dist.all_gather_into_tensor(full, mine, group=self.group)


class ShardedRunner:
    """Generation loop of one rank.  `comm` defaults to torch.distributed over
    `group`; anything with the same three methods works (the single-GPU
    emulation in tests/test_sharded_gpu.py passes an in-process one)."""

    def __init__(self, ops, group=None, comm=None):
        self.ops = ops
        self.comm = comm if comm is not None else Comm(group)
        self.world, self.rank = self.comm.world, self.comm.rank
        self.generation = 0
        self.best_fitness = 0.0
        self.stop_reason: Optional[str] = None

    @property
    def done(self) -> bool:
        return self.stop_reason is not None

    def steps(self, n: int) -> np.ndarray:
        """Up to n generations; stops where the single-device engine would."""
        out = []
        remaining = int(n)
        while remaining > 0 and not self.done:
            k = min(remaining, getattr(self.ops, "max_batch", remaining))
            self.ops.begin_batch()
            for _ in range(k):
                self.ops.generation(self.comm)
            rec, stop = self.ops.read_batch()
            if rec.size:
                self.generation += int(rec.size)
                self.best_fitness = float(rec["best_fitness"][-1])
            self.stop_reason = STOP_REASONS[int(stop)]
            out.append(rec)
            remaining -= k
        return np.concatenate(out) if out else np.zeros(0, dtype=_lib.GEN_RECORD)


def _device_view(ptr: int, n: int, typestr: str, device: int):
    """torch view of a libisq-owned device buffer (__cuda_array_interface__)."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_CAI(), device=f"cuda:{device}")


class _DeviceOps:
    _prefix = ""

    def __init__(self, engine):
        import torch

        self.engine = engine
        self.lib = engine._lib
        self.h = engine._handle()
        self.max_batch = engine.max_batch
        self.stream = torch.cuda.current_stream(engine.device)
        self._call("set_stream", ctypes.c_void_p(self.stream.cuda_stream))

    def _call(self, name, *args):
        _lib.check(getattr(self.lib, f"isq_{self._prefix}_{name}")(self.h, *args))

    def begin_batch(self):
        self._call("begin_batch")

    def read_batch(self):
        rec = np.zeros(self.max_batch, dtype=_lib.GEN_RECORD)
        nd, stop = ctypes.c_int32(), ctypes.c_int32()
        self._call("read_batch", _lib.ptr(rec), ctypes.byref(nd), ctypes.byref(stop), None, None)
        rec = rec[: nd.value]
        self.engine._absorb(rec, int(stop.value))  # keep the engine's host mirror (generation, best) current
        return rec, int(stop.value)


class DeviceQeqeaOps(_DeviceOps):
    """One rank's generation.  transport="nccl": the two all-to-alls and two
    all-gathers are collectives between the phases; transport="p2p": the
    producing kernels store straight into the other ranks' buffers over
    NVLink (include/isq.h peer transport) and the phases are only ordered by
    stream barriers.  Both give identical results."""

    _prefix = "qeqea"

    def __init__(self, engine, transport: str = "nccl"):
        if transport not in ("nccl", "p2p"):
            raise ValueError("transport must be 'nccl' or 'p2p'")
        super().__init__(engine)
        self.transport = transport
        self.connected = False
        x = _lib.QeqeaExchange()
        self._call("exchange", ctypes.byref(x))
        self.world, self.rank, self.S = x.world, x.rank, x.shard
        self.routing = Routing(engine.cfg.size_of_individual, self.S, self.world, self.rank)
        L, dev, no = engine.cfg.size_of_individual, engine.device, self.world * self.S * self.routing.Lr
        self.fitness = _device_view(x.fitness, self.world * self.S, "<f8", dev)
        self._x = x
        if self.world > 1:
            self.elite_len = x.elite_len
            self.elite = _device_view(x.elite, self.world * x.elite_len, "<f8", dev)
            # uint32 slot indices travel as int32 (same bytes)
            self.send_flats = _device_view(x.send_flats, self.S * L, "<i4", dev)
            self.recv_flats = _device_view(x.recv_flats, no, "<i4", dev)
            self.send_codes = _device_view(x.send_codes, no, "|u1", dev)
            self.recv_codes = _device_view(x.recv_codes, self.S * L, "|u1", dev)
            self.send_thetas = _device_view(x.send_thetas, no, "<f8", dev)
            self.recv_thetas = _device_view(x.recv_thetas, self.S * L, "<f8", dev)

    # -- peer transport ---------------------------------------------------
    def peer_buffers(self):
        """This rank's exchange buffers (device pointers, include/isq.h order)."""
        x = self._x
        return (x.recv_flats, x.recv_codes, x.recv_thetas, x.fitness, x.elite)

    def ipc_handles(self) -> bytes:
        buf = (ctypes.c_char * (_lib.PEER_BUFFERS * _lib.IPC_HANDLE_BYTES))()
        self._call("ipc_export", buf)
        return bytes(buf)

    def open_peers_ipc(self, all_handles):
        raw = b"".join(all_handles)
        buf = (ctypes.c_char * len(raw)).from_buffer_copy(raw)
        self._call("ipc_open", buf)
        self.connected = True

    def set_peer_pointers(self, all_buffers):
        """Peers already addressable in this process (several ranks' handles
        on one device, tests/test_sharded_gpu.py)."""
        arr = (_lib.PeerBuffers * self.world)(*[_lib.PeerBuffers(*b) for b in all_buffers])
        self._call("set_peers", arr)
        self.connected = True

    def generation(self, comm: Optional[Comm], marks=None):
        """One generation; `marks` (4 torch.cuda.Events, optional) are recorded
        on the handle's stream before prepare, before score, after score and
        after finish (bench.py phase timing)."""
        if self.transport == "p2p" and self.world > 1:
            return self._generation_p2p(comm, marks)
        r = self.routing
        if marks:
            marks[0].record(self.stream)
        self._call("prepare")
        if self.world > 1:
            comm.all_to_all(self.recv_flats, self.send_flats, r.from_circuits, r.to_owners)
        self._call("values")
        if self.world > 1:
            comm.all_to_all(self.recv_codes, self.send_codes, r.to_owners, r.from_circuits)
            comm.all_to_all(self.recv_thetas, self.send_thetas, r.to_owners, r.from_circuits)
        if marks:
            marks[1].record(self.stream)
        self._call("score")
        if marks:
            marks[2].record(self.stream)
        if self.world > 1:
            comm.all_gather(self.fitness, self.S)
            comm.all_gather(self.elite, self.elite_len)
        self._call("finish")
        if marks:
            marks[3].record(self.stream)

    def _generation_p2p(self, comm, marks):
        if not self.connected:
            comm.connect_peers(self)
        if marks:
            marks[0].record(self.stream)
        comm.barrier()           # every rank is done reading last generation's buffers
        self._call("prepare")    # touches -> owners' recv_flats
        comm.barrier()
        self._call("values")     # codes / angles -> circuit ranks' recv buffers
        comm.barrier()
        if marks:
            marks[1].record(self.stream)
        self._call("score")      # fitness + elite -> every rank
        if marks:
            marks[2].record(self.stream)
        comm.barrier()
        self._call("finish")
        if marks:
            marks[3].record(self.stream)


class DeviceGaOps(_DeviceOps):
    _prefix = "ga"

    def __init__(self, engine):
        super().__init__(engine)
        ptr, shard = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(self.lib.isq_ga_buffers(self.h, ctypes.byref(ptr), ctypes.byref(shard), None))
        self.S = int(shard.value)
        self.fitness = _device_view(ptr.value, self.S * engine.world, "<f8", engine.device)

    def generation(self, comm: Optional[Comm]):
        self._call("eval")
        if comm is not None and comm.world > 1:
            comm.all_gather(self.fitness, self.S)
        self._call("finish")


def sharded_qeqea(cfg, target, seed: int, group=None, transport: str = "p2p", **kw) -> ShardedRunner:
    """A QEQEA run sharded over the process group (one GPU per rank)."""
    import torch
    import torch.distributed as dist

    from .engine import QeqeaEngine

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device()
    eng = QeqeaEngine(cfg, target, seed, device=dev, rank=rank, world=world, **kw)
    runner = ShardedRunner(DeviceQeqeaOps(eng, transport), group)
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
