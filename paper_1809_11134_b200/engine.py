"""Quantum-encoded evolutionary engine (QEQEA) on the GPU.

Drop-in for isingsynth.engine (engine.py:1-393): `PopulationConfig`,
`PopulationState`, `QeqeaEngine` (step / done / best_fitness / best_gates /
generation / stop_reason / config_echo / close / pickling) and `run_qeqea`.
The generation loop runs in libisq (csrc/kernels_qeqea.cu); this module only
validates, marshals and mirrors the reference's attributes.

Differences from the reference, by design:
  * random draws come from counter-based Philox streams per (generation,
    circuit | slot) instead of one sequential numpy Generator, so trajectories
    equal the Philox restatement of the reference (oracle/), not a PCG64 run;
  * the initial bank is drawn on the device from per-slot streams (θ uniform,
    Box-Muller qutrits) unless `population=` injects one (e.g. the reference's
    own init_population output);
  * numberOfWires is limited to 2..13, the reference's default
    4^n <= 2^26 cap (a raised memory_cap_entries beyond it is a
    ConfigurationError here); any nMeas >= 1
    (numpy's inversion and BTPE binomial branches are both reproduced).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _lib
from .errors import ConfigurationError
from .fitness import TargetSpec
from .gates import Axis, GateOp, enumerate_templates, gate_from_code

DEFAULT_MAX_GENERATIONS = 10_000_000
STOP_REASONS = {0: None, 1: "target-reached", 2: "generation-limit"}
_STOP_CODES = {v: k for k, v in STOP_REASONS.items()}


@dataclass(frozen=True)
class PopulationConfig:
    """engine.py:33-94 (fields, defaults, validation, slot accounting)."""

    number_of_wires: int
    size_of_individual: int
    size_of_population: int
    probability_of_mutation: float = 0.3
    mutation_range: float = math.pi / 4
    n_meas: int = 1
    max_generations: int = DEFAULT_MAX_GENERATIONS
    target_fitness: float = 0.999
    memory_cap_entries: int = 2 ** 26

    def __post_init__(self):
        if self.number_of_wires < 2:
            raise ConfigurationError("numberOfWires must be ≥ 2")
        if self.size_of_individual < 1 or self.size_of_population < 1:
            raise ConfigurationError("sizeOfIndividual and sizeOfPopulation must be ≥ 1")
        if not 0.0 <= self.probability_of_mutation <= 1.0:
            raise ConfigurationError("probabilityOfMutation must be in [0, 1]")
        if self.mutation_range <= 0.0:
            raise ConfigurationError("mutationRange must be > 0")
        if self.n_meas < 1:
            raise ConfigurationError("nMeas must be ≥ 1")
        if self.max_generations < 1:
            raise ConfigurationError("maxGenerations must be ≥ 1")
        if not 0.0 < self.target_fitness <= 1.0:
            raise ConfigurationError("targetFitness must be in (0, 1]")
        if (2 ** self.number_of_wires) ** 2 > self.memory_cap_entries:
            raise ConfigurationError(
                f"numberOfWires={self.number_of_wires} exceeds the dense-matrix memory cap"
            )

    @property
    def template_count(self) -> int:
        n = self.number_of_wires
        return n * (n - 1) // 2

    @property
    def slot_kind_count(self) -> int:
        return self.number_of_wires + self.template_count

    @property
    def qubit_count(self) -> int:
        return self.slot_kind_count * self.size_of_population * self.size_of_individual

    @property
    def qutrit_count(self) -> int:
        return self.number_of_wires * self.size_of_population * self.size_of_individual

    def flat_index(self, slot_kind: int, individual: int, position: int) -> int:
        return (
            slot_kind * self.size_of_individual * self.size_of_population
            + individual * self.size_of_individual
            + position
        )

    def decode_flat(self, flat: int) -> Tuple[int, int, int]:
        per_kind = self.size_of_individual * self.size_of_population
        slot_kind, rest = divmod(flat, per_kind)
        individual, position = divmod(rest, self.size_of_individual)
        return slot_kind, individual, position


@dataclass
class PopulationState:
    """The flat bank (engine.py:97-102): thetas (Q,), qutrits (Qt, 3) complex."""

    thetas: np.ndarray
    qutrits: np.ndarray


class SegmentTableView:
    """Read-only view of SegmentFitnessTable.slot_max (engine.py:202-209)."""

    def __init__(self, engine: "QeqeaEngine"):
        self._engine = engine

    @property
    def slot_max(self) -> np.ndarray:
        return self._engine._get_state()[2]


def position_bounds(length: int, world: int) -> List[int]:
    """Rank o of a sharded run owns the bank slots of positions [b[o], b[o+1])
    (csrc/api_qeqea.cu isq_qeqea_create)."""
    return [o * length // world for o in range(world + 1)]


def owned_slots(cfg: PopulationConfig, rank: int, world: int) -> np.ndarray:
    """Flat slot indices (Eq. 9, engine.py:82-87) owned by `rank`, in the
    device's local order (slot kind, individual, owned position)."""
    b = position_bounds(cfg.size_of_individual, world)
    ki = np.arange(cfg.slot_kind_count * cfg.size_of_population, dtype=np.int64)[:, None]
    pos = np.arange(b[rank], b[rank + 1], dtype=np.int64)[None, :]
    return (ki * cfg.size_of_individual + pos).reshape(-1)


def _target_array(target: TargetSpec | np.ndarray, n: int, name: str = "target") -> np.ndarray:
    m = target.matrix if isinstance(target, TargetSpec) else np.asarray(target)
    if m.shape[0] != 2 ** n:
        raise ConfigurationError(f"target {name} dimension {m.shape[0]} != 2^{n}")
    return np.ascontiguousarray(m, dtype=np.complex128)


class _DeviceLimits:
    """`cfg` and `stop_reason` mirrored onto the device handle.

    The reference's resume flow (harness.py:95-110) replaces `engine.cfg`
    with a larger max_generations and clears `stop_reason`; the device stop
    rule (engine.py:354-358, ga.py:189-192) reads both from the handle, so
    assigning either attribute pushes them with isq_*_set_limits.
    """

    _limits_fn = ""
    _structural: Tuple[str, ...] = ()

    @property
    def cfg(self):
        return self.__dict__["_cfg"]

    @cfg.setter
    def cfg(self, cfg):
        old = self.__dict__.get("_cfg")
        if old is not None:
            changed = [f for f in self._structural if getattr(old, f) != getattr(cfg, f)]
            if changed:
                raise ConfigurationError(
                    f"cannot change {', '.join(changed)} of a live engine (only the stop rule)")
        self.__dict__["_cfg"] = cfg
        self._push_limits()

    @property
    def stop_reason(self) -> Optional[str]:
        return self.__dict__.get("_stop_reason")

    @stop_reason.setter
    def stop_reason(self, reason: Optional[str]):
        if reason not in _STOP_CODES:
            raise ConfigurationError(f"stop_reason must be one of {sorted(map(str, _STOP_CODES))}")
        self.__dict__["_stop_reason"] = reason
        self._push_limits()

    def _push_limits(self):
        h = self.__dict__.get("_h")
        if h is None or h.value is None:
            return
        c = self.cfg
        _lib.check(getattr(self._lib, self._limits_fn)(h, int(c.max_generations), float(c.target_fitness),
                                                       _STOP_CODES[self.stop_reason]))

    def _step_once(self):
        """One generation even after a stop, as the reference's step() runs
        one whenever it is called (engine.py:318-361, ga.py:165-194); the
        stop reason is then re-derived by the device and, as in the
        reference, never cleared by the step itself."""
        prev = self.stop_reason
        if prev is not None:
            self.stop_reason = None
        rec = self.steps(1)
        if prev is not None and self.stop_reason is None:
            self.stop_reason = prev
        return float(rec["gen_best"][0]), float(rec["gen_mean"][0])


class QeqeaEngine(_DeviceLimits):
    """Stepwise generation loop on one device (or one rank of a sharded run)."""

    algorithm = "qeqea"
    _limits_fn = "isq_qeqea_set_limits"
    _structural = ("number_of_wires", "size_of_individual", "size_of_population",
                   "probability_of_mutation", "mutation_range", "n_meas", "memory_cap_entries")

    def __init__(
        self,
        cfg: PopulationConfig,
        target: TargetSpec,
        seed: int,
        workers: int = 1,
        *,
        device: int = 0,
        population: Optional[PopulationState] = None,
        rank: int = 0,
        world: int = 1,
        max_batch: int = 4096,
        precision: str = "fp64",
    ):
        name = target.name if isinstance(target, TargetSpec) else "target"
        if precision not in _lib.PRECISIONS:
            raise ConfigurationError(f"precision must be one of {sorted(_lib.PRECISIONS)}")
        self.precision = precision
        self._tmat = _target_array(target, cfg.number_of_wires, name)
        if seed < 0:
            raise ConfigurationError("seed must be non-negative")
        self.cfg = cfg
        self.target = target if isinstance(target, TargetSpec) else TargetSpec(
            "custom", cfg.number_of_wires, self._tmat)
        self.seed = int(seed)
        self.workers = max(1, int(workers))
        self.device = int(device)
        self.rank, self.world = int(rank), int(world)
        self.max_batch = int(max_batch)
        self.templates = enumerate_templates(cfg.number_of_wires)
        self._h = None
        self._open()
        self.generation = 0
        self.best_fitness = 0.0
        self.__dict__["_stop_reason"] = None
        self._best_gates: List[GateOp] = []
        self._best_dirty = False
        if population is not None:
            self._set_population(population)

    # ------------------------------------------------------------ handle --
    def _open(self):
        lib = _lib.load()
        c = self.cfg
        conf = _lib.QeqeaConfig(
            number_of_wires=c.number_of_wires,
            size_of_individual=c.size_of_individual,
            size_of_population=c.size_of_population,
            probability_of_mutation=c.probability_of_mutation,
            mutation_range=c.mutation_range,
            n_meas=c.n_meas,
            rank=self.rank,
            max_generations=c.max_generations,
            target_fitness=c.target_fitness,
            seed=self.seed,
            world=self.world,
            precision=_lib.PRECISIONS[self.precision],
        )
        h = ctypes.c_void_p()
        _lib.check(lib.isq_qeqea_create(ctypes.byref(conf), _lib.ptr(self._tmat), self.device,
                                        self.max_batch, ctypes.byref(h)))
        self._h = h
        self._lib = lib

    def close(self) -> None:
        """Releases the device bank (the reference's close() shuts its thread
        pool); best_fitness / best_gates / generation stay readable."""
        if getattr(self, "_h", None) is not None and self._h.value is not None:
            _ = self.best_gates
            self._lib.isq_qeqea_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _handle(self):
        if self._h is None:
            raise RuntimeError("engine is closed (its device bank was released)")
        return self._h

    # ------------------------------------------------------------- state --
    def _local_counts(self):
        """(owned slots, owned rotation-region slots): Q and Qt at world 1."""
        c = self.cfg
        b = position_bounds(c.size_of_individual, self.world)
        lr = b[self.rank + 1] - b[self.rank]
        return (c.slot_kind_count * c.size_of_population * lr,
                c.number_of_wires * c.size_of_population * lr)

    def _get_state(self):
        ql, qtl = self._local_counts()
        th = np.empty(ql)
        qa = np.empty((3, qtl), dtype=np.complex128)
        sm = np.empty(ql)
        gen = ctypes.c_uint64()
        best = ctypes.c_double()
        stop = ctypes.c_int32()
        _lib.check(self._lib.isq_qeqea_get_state(self._handle(), _lib.ptr(th), _lib.ptr(qa), _lib.ptr(sm),
                                                 ctypes.byref(gen), ctypes.byref(best), ctypes.byref(stop)))
        return th, qa, sm, int(gen.value), float(best.value), int(stop.value)

    def _set_population(self, pop: PopulationState):
        """Injects the reference's full arrays (init_population); a sharded
        rank keeps the slots it owns."""
        c = self.cfg
        th = np.asarray(pop.thetas, dtype=np.float64)
        q = np.asarray(pop.qutrits, dtype=np.complex128)
        if th.shape != (c.qubit_count,) or q.shape != (c.qutrit_count, 3):
            raise ConfigurationError("population shape does not match the configuration")
        if self.world > 1:
            own = owned_slots(c, self.rank, self.world)
            th = th[own]
            q = q[own[own < c.qutrit_count]]
        th = np.ascontiguousarray(th)
        qa = np.ascontiguousarray(q.T)
        _lib.check(self._lib.isq_qeqea_set_state(self._handle(), _lib.ptr(th), _lib.ptr(qa), None,
                                                 self.generation, self.best_fitness,
                                                 _STOP_CODES[self.stop_reason], None, None))

    def owned_population(self):
        """(flat slots, PopulationState) of the live bank slots this rank
        owns; at world 1 the whole bank in flat order (== pop)."""
        ql, qtl = self._local_counts()
        th = np.empty(ql)
        q = np.empty((qtl, 3), dtype=np.complex128)
        _lib.check(self._lib.isq_qeqea_live_population(self._handle(), _lib.ptr(th), _lib.ptr(q)))
        return owned_slots(self.cfg, self.rank, self.world), PopulationState(thetas=th, qutrits=q)

    @property
    def pop(self) -> PopulationState:
        """The live bank (engine.pop after the last step)."""
        if self.world > 1:
            raise ConfigurationError("the bank is sharded over the ranks; use owned_population()")
        return self.owned_population()[1]

    @property
    def table(self) -> SegmentTableView:
        return SegmentTableView(self)

    # -------------------------------------------------------------- step --
    @property
    def done(self) -> bool:
        return self.stop_reason is not None

    def steps(self, n: int) -> np.ndarray:
        """Run up to n generations on the device (stops exactly where step()
        would); returns the structured records of the generations run."""
        if self.world != 1:
            raise ConfigurationError("use paper_1809_11134_b200.distributed for world > 1")
        out = []
        remaining = int(n)
        while remaining > 0 and not self.done:
            k = min(remaining, self.max_batch)
            rec = np.zeros(k, dtype=_lib.GEN_RECORD)
            nd = ctypes.c_int32()
            stop = ctypes.c_int32()
            _lib.check(self._lib.isq_qeqea_step(self._handle(), k, _lib.ptr(rec), ctypes.byref(nd),
                                                ctypes.byref(stop)))
            rec = rec[: nd.value]
            self._absorb(rec, stop.value)
            out.append(rec)
            remaining -= k
        return np.concatenate(out) if out else np.zeros(0, dtype=_lib.GEN_RECORD)

    def set_launch_mode(self, mode: str) -> None:
        """How steps() launches generations: "auto" (default), "kernels",
        "graph" (16-generation CUDA graphs) or "fused" (one single-block
        launch); every mode gives identical results (include/isq.h)."""
        if mode not in _lib.LAUNCH_MODES:
            raise ConfigurationError(f"launch mode must be one of {sorted(_lib.LAUNCH_MODES)}")
        _lib.check(self._lib.isq_qeqea_set_launch_mode(self._handle(), _lib.LAUNCH_MODES[mode]))

    def _absorb(self, rec: np.ndarray, stop: int):
        if rec.size:
            self.generation += int(rec.size)
            if rec["best_fitness"][-1] > self.best_fitness:
                self._best_dirty = True
            self.best_fitness = float(rec["best_fitness"][-1])
        self.__dict__["_stop_reason"] = STOP_REASONS[int(stop)]  # already the device's

    def step(self) -> Tuple[float, float]:
        """One generation; returns (generation best, generation mean) (engine.py:318-361).
        Like the reference, a step after a stop still runs a generation."""
        return self._step_once()

    @property
    def best_gates(self) -> List[GateOp]:
        if self._best_dirty:
            L = self.cfg.size_of_individual
            codes = np.empty(L, dtype=np.uint8)
            th = np.empty(L)
            fit = ctypes.c_double()
            _lib.check(self._lib.isq_qeqea_best(self._handle(), _lib.ptr(codes), _lib.ptr(th), ctypes.byref(fit)))
            self._best_gates = [gate_from_code(k, t, self.cfg.number_of_wires) for k, t in zip(codes, th)]
            self._best_dirty = False
        return list(self._best_gates)

    @best_gates.setter
    def best_gates(self, gates: List[GateOp]):
        self._best_gates = list(gates)
        self._best_dirty = False

    # --------------------------------------------------------- functional --
    def sample(self, c0: int = 0, c1: Optional[int] = None):
        """(blueprints, gate codes, live angles) of circuits [c0, c1) for the
        current generation — sample_circuit + construct_segments on device."""
        c1 = self.cfg.size_of_population if c1 is None else c1
        L = self.cfg.size_of_individual
        n = (c1 - c0) * L
        f = np.empty(n, dtype=np.int64)
        k = np.empty(n, dtype=np.uint8)
        t = np.empty(n)
        _lib.check(self._lib.isq_qeqea_sample(self._handle(), c0, c1, _lib.ptr(f), _lib.ptr(k), _lib.ptr(t)))
        return f.reshape(-1, L), k.reshape(-1, L), t.reshape(-1, L)

    def last_fitness(self) -> np.ndarray:
        out = np.empty(self.cfg.size_of_population)
        _lib.check(self._lib.isq_qeqea_fitness(self._handle(), _lib.ptr(out)))
        return out

    # ---------------------------------------------------------- pickling --
    def __getstate__(self):
        th, qa, sm, gen, best, stop = self._get_state()
        d = {k: v for k, v in self.__dict__.items() if k not in ("_h", "_lib")}
        d["_best_gates"] = self.best_gates
        d["_best_dirty"] = False
        d["_pending_state"] = (th, qa, sm, gen, best, stop)
        return d

    def __setstate__(self, d):
        self.__dict__.update(d)
        self._h = None
        self._open()
        self._restore(d["_pending_state"])
        del self._pending_state

    def _restore(self, state):
        th, qa, sm, gen, best, stop = state
        codes, thetas = None, None
        if self._best_gates:
            from .gates import encode_gates

            codes, thetas = encode_gates(self._best_gates, self.cfg.number_of_wires)
        _lib.check(self._lib.isq_qeqea_set_state(self._h, _lib.ptr(th), _lib.ptr(np.ascontiguousarray(qa)),
                                                 _lib.ptr(sm), gen, best, stop, _lib.ptr(codes),
                                                 _lib.ptr(thetas)))

    def config_echo(self) -> dict:
        cfg = self.cfg
        return {
            "numberOfWires": cfg.number_of_wires,
            "sizeOfIndividual": cfg.size_of_individual,
            "sizeOfPopulation": cfg.size_of_population,
            "probabilityOfMutation": cfg.probability_of_mutation,
            "mutationRange": cfg.mutation_range,
            "nMeas": cfg.n_meas,
            "maxGenerations": cfg.max_generations,
            "targetFitness": cfg.target_fitness,
            "workers": self.workers,
        }


def run_qeqea(cfg: PopulationConfig, target: TargetSpec, seed: int, workers: int = 1):
    """Full evolution run returning a RunReport (engine.py:387-393)."""
    from .report import run_engine

    return run_engine(QeqeaEngine(cfg, target, seed, workers=workers))


_FUNCTIONAL = {"init_population", "SegmentBank", "construct_segments", "sample_circuit", "evaluate_circuit",
               "SegmentFitnessTable", "mutate_population", "Snapshot", "CounterStreams"}


def __getattr__(name):
    """The reference's module-level operators (engine.py:105-263) live in
    .functional (device-backed, counter streams); re-exported here so
    `from paper_1809_11134_b200.engine import SegmentFitnessTable` works as
    `from isingsynth.engine import SegmentFitnessTable` does."""
    if name in _FUNCTIONAL:
        from . import functional

        return getattr(functional, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
