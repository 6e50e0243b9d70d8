"""Classical genetic-algorithm baseline ("GPUGA") on the GPU.

Drop-in for isingsynth.ga (ga.py:1-220): `GaConfig` (gate_choices),
`GaEngine` (step / done / best_fitness / best_gates / generation /
stop_reason / genomes / config_echo / close / pickling) and `run_ga`.
Genomes are device-resident gate codes + angles (csrc/kernels_ga.cu); SUS,
two-point crossover and per-gene mutation run on the device with the
per-unit Philox streams of the oracle (pair / (child, gene) / generation).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from itertools import combinations
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from .engine import STOP_REASONS, _STOP_CODES, _DeviceLimits, _target_array
from .errors import ConfigurationError
from .fitness import TargetSpec
from .gates import Axis, GateOp, encode_gates, gate_from_code

CircuitGenome = Tuple[GateOp, ...]


@dataclass(frozen=True)
class GaConfig:
    """ga.py:22-59."""

    number_of_wires: int
    size_of_individual: int
    population: int = 50
    mutation_rate: float = 0.1
    mutation_range: float = math.pi / 8
    structural_rate: float = 0.1
    max_generations: int = 10_000_000
    target_fitness: float = 0.999

    def __post_init__(self):
        if self.number_of_wires < 2:
            raise ConfigurationError("numberOfWires must be ≥ 2")
        if self.size_of_individual < 1:
            raise ConfigurationError("sizeOfIndividual must be ≥ 1")
        if self.population < 2:
            raise ConfigurationError("GA population must be ≥ 2")
        if not 0.0 <= self.mutation_rate <= 1.0:
            raise ConfigurationError("mutation rate must be in [0, 1]")
        if not 0.0 <= self.structural_rate <= 1.0:
            raise ConfigurationError("structural rate must be in [0, 1]")
        if not 0.0 < self.target_fitness <= 1.0:
            raise ConfigurationError("targetFitness must be in (0, 1]")

    @property
    def gate_choices(self) -> List[GateOp]:
        protos = [GateOp(kind="rotation", theta=0.0, wire=w, axis=Axis(a))
                  for w in range(1, self.number_of_wires + 1) for a in range(3)]
        protos += [GateOp(kind="interaction", theta=0.0, pair=p)
                   for p in combinations(range(1, self.number_of_wires + 1), 2)]
        return protos


class GaEngine(_DeviceLimits):
    """Generational GA loop with the same step interface as QeqeaEngine."""

    algorithm = "ga"
    _limits_fn = "isq_ga_set_limits"
    _structural = ("number_of_wires", "size_of_individual", "population", "mutation_rate",
                   "mutation_range", "structural_rate")

    def __init__(self, cfg: GaConfig, target: TargetSpec, seed: int, workers: int = 1, *,
                 device: int = 0, genomes: Optional[List[CircuitGenome]] = None,
                 rank: int = 0, world: int = 1, max_batch: int = 4096, precision: str = "fp64"):
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
        self._h = None
        self._open()
        self.generation = 0
        self.best_fitness = 0.0
        self.__dict__["_stop_reason"] = None
        self._best_gates: List[GateOp] = []
        self._best_dirty = False
        if genomes is not None:
            codes = np.stack([encode_gates(g, cfg.number_of_wires)[0] for g in genomes])
            thetas = np.stack([encode_gates(g, cfg.number_of_wires)[1] for g in genomes])
            self.set_genome_arrays(codes, thetas)

    def _open(self):
        lib = _lib.load()
        c = self.cfg
        conf = _lib.GaConfigC(
            number_of_wires=c.number_of_wires, size_of_individual=c.size_of_individual,
            population=c.population, mutation_rate=c.mutation_rate, mutation_range=c.mutation_range,
            structural_rate=c.structural_rate, max_generations=c.max_generations,
            target_fitness=c.target_fitness, seed=self.seed, rank=self.rank, world=self.world,
            precision=_lib.PRECISIONS[self.precision], reserved=0)
        h = ctypes.c_void_p()
        _lib.check(lib.isq_ga_create(ctypes.byref(conf), _lib.ptr(self._tmat), self.device,
                                     self.max_batch, ctypes.byref(h)))
        self._h, self._lib = h, lib

    def _handle(self):
        if self._h is None:
            raise RuntimeError("engine is closed (its device state was released)")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value is not None:
            _ = self.best_gates
            self._lib.isq_ga_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ genomes --
    def genome_arrays(self) -> Tuple[np.ndarray, np.ndarray]:
        c = self.cfg
        codes = np.empty((c.population, c.size_of_individual), dtype=np.uint8)
        thetas = np.empty((c.population, c.size_of_individual))
        _lib.check(self._lib.isq_ga_get_state(self._handle(), _lib.ptr(codes), _lib.ptr(thetas),
                                              None, None, None))
        return codes, thetas

    def set_genome_arrays(self, codes: np.ndarray, thetas: np.ndarray) -> None:
        c = self.cfg
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        thetas = np.ascontiguousarray(thetas, dtype=np.float64)
        if codes.shape != (c.population, c.size_of_individual) or thetas.shape != codes.shape:
            raise ConfigurationError("genome arrays do not match the configuration")
        bc, bt = (encode_gates(self._best_gates, c.number_of_wires) if self._best_gates else (None, None))
        _lib.check(self._lib.isq_ga_set_state(self._handle(), _lib.ptr(codes), _lib.ptr(thetas),
                                              self.generation, self.best_fitness,
                                              _STOP_CODES[self.stop_reason], _lib.ptr(bc), _lib.ptr(bt)))

    @property
    def genomes(self) -> List[CircuitGenome]:
        codes, thetas = self.genome_arrays()
        n = self.cfg.number_of_wires
        return [tuple(gate_from_code(k, t, n) for k, t in zip(cr, tr)) for cr, tr in zip(codes, thetas)]

    # --------------------------------------------------------------- step --
    @property
    def done(self) -> bool:
        return self.stop_reason is not None

    def steps(self, n: int) -> np.ndarray:
        if self.world != 1:
            raise ConfigurationError("use paper_1809_11134_b200.distributed for world > 1")
        out = []
        remaining = int(n)
        while remaining > 0 and not self.done:
            k = min(remaining, self.max_batch)
            rec = np.zeros(k, dtype=_lib.GEN_RECORD)
            nd, stop = ctypes.c_int32(), ctypes.c_int32()
            _lib.check(self._lib.isq_ga_step(self._handle(), k, _lib.ptr(rec), ctypes.byref(nd),
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
        _lib.check(self._lib.isq_ga_set_launch_mode(self._handle(), _lib.LAUNCH_MODES[mode]))

    def _absorb(self, rec: np.ndarray, stop: int):
        if rec.size:
            self.generation += int(rec.size)
            if rec["best_fitness"][-1] > self.best_fitness:
                self._best_dirty = True
            self.best_fitness = float(rec["best_fitness"][-1])
        self.__dict__["_stop_reason"] = STOP_REASONS[int(stop)]  # already the device's

    def step(self) -> Tuple[float, float]:
        """One generation (ga.py:165-194); returns (generation best, mean).
        Like the reference, a step after a stop still runs a generation."""
        return self._step_once()

    @property
    def best_gates(self) -> List[GateOp]:
        if self._best_dirty:
            L = self.cfg.size_of_individual
            codes = np.empty(L, dtype=np.uint8)
            th = np.empty(L)
            fit = ctypes.c_double()
            _lib.check(self._lib.isq_ga_best(self._handle(), _lib.ptr(codes), _lib.ptr(th), ctypes.byref(fit)))
            self._best_gates = [gate_from_code(k, t, self.cfg.number_of_wires) for k, t in zip(codes, th)]
            self._best_dirty = False
        return list(self._best_gates)

    def last_fitness(self) -> np.ndarray:
        out = np.empty(self.cfg.population)
        _lib.check(self._lib.isq_ga_fitness(self._handle(), _lib.ptr(out)))
        return out

    def last_parents(self) -> np.ndarray:
        out = np.empty(self.cfg.population, dtype=np.int32)
        _lib.check(self._lib.isq_ga_parents(self._handle(), _lib.ptr(out)))
        return out

    # ----------------------------------------------------------- pickling --
    def __getstate__(self):
        codes, thetas = self.genome_arrays()
        d = {k: v for k, v in self.__dict__.items() if k not in ("_h", "_lib")}
        d["_best_gates"] = self.best_gates
        d["_best_dirty"] = False
        d["_pending"] = (codes, thetas)
        return d

    def __setstate__(self, d):
        codes, thetas = d.pop("_pending")
        self.__dict__.update(d)
        self._h = None
        self._open()
        self.set_genome_arrays(codes, thetas)

    def config_echo(self) -> dict:
        cfg = self.cfg
        return {
            "numberOfWires": cfg.number_of_wires,
            "sizeOfIndividual": cfg.size_of_individual,
            "gaPopulation": cfg.population,
            "gaMutationRate": cfg.mutation_rate,
            "gaMutationRange": cfg.mutation_range,
            "gaStructuralRate": cfg.structural_rate,
            "maxGenerations": cfg.max_generations,
            "targetFitness": cfg.target_fitness,
        }


def run_ga(cfg: GaConfig, target: TargetSpec, seed: int, workers: int = 1):
    """ga.py:217-220."""
    from .report import run_engine

    return run_engine(GaEngine(cfg, target, seed, workers=workers))


_FUNCTIONAL = {"random_genome", "decode_genome", "two_point_crossover", "sus_select", "ga_mutate"}


def __getattr__(name):
    """The reference's GA operators (ga.py:62-138) live in .functional
    (device-backed, counter streams); re-exported as isingsynth.ga exports them."""
    if name in _FUNCTIONAL:
        from . import functional

        return getattr(functional, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
