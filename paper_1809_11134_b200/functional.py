"""The reference's functional API on the device (engine.py:105-263,
ga.py:62-138; the names its tests import, pkg/tests/test_engine.py:8-17,
test_ga.py:7-15).

Same names, argument order, return types and exceptions as the reference,
with one documented difference: where the reference takes a sequential
`numpy.random.Generator` (`rng`), these take a `CounterStreams` position —
the counter-based Philox streams the device engines draw from (DESIGN.md
§5.1; csrc/np_random.cuh).  A call then computes exactly what the engine
computes for that unit of work:

    init_population(cfg, CounterStreams(seed))                       per slot
    construct_segments(pop, cfg, templates, CounterStreams(seed, g)) per slot
    sample_circuit(cfg, CounterStreams(seed, g, c))                  circuit c of generation g
    mutate_population(pop, table, cfg, CounterStreams(seed, g))      per slot
    random_genome(cfg, CounterStreams(seed, index=i))                genome i
    two_point_crossover(a, b, CounterStreams(seed, g, k))            pair k of generation g
    sus_select(fitnesses, count, CounterStreams(seed, g))
    ga_mutate(genome, cfg, CounterStreams(seed, g, i))               child i of generation g

A Generator cannot be honoured: its draws are a single sequence whose
position depends on every earlier call (the reference's init_population,
construct_segments and mutate_population all advance the same engine
Generator, engine.py:283), while every device operator is a pure function
of (seed, generation, unit).  Passing one raises TypeError.  Integer seeds
are accepted as CounterStreams(seed).

Generator-independent calls keep the reference's signatures exactly:
SegmentBank, evaluate_circuit, SegmentFitnessTable, decode_genome.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Set, Tuple

import numpy as np

from . import _lib
from .engine import PopulationConfig, PopulationState
from .errors import ConfigurationError
from .fitness import fitness_batch
from .ga import CircuitGenome, GaConfig
from .gates import Axis, GateOp, compose_gates, encode_gates, enumerate_templates, gate_from_code

Snapshot = Tuple[float, Optional[np.ndarray]]


@dataclass(frozen=True)
class CounterStreams:
    """Position in the engines' counter streams: (seed, generation, index)."""

    seed: int
    generation: int = 0
    index: int = 0

    def __post_init__(self):
        if min(self.seed, self.generation, self.index) < 0:
            raise ConfigurationError("seed, generation and index must be non-negative")


def _streams(rng) -> CounterStreams:
    if isinstance(rng, CounterStreams):
        return rng
    if isinstance(rng, (int, np.integer)):
        return CounterStreams(int(rng))
    if isinstance(rng, np.random.Generator):
        raise TypeError(
            "the device operators draw from counter-based streams (seed, generation, index), not from a "
            "sequential numpy Generator; pass CounterStreams(seed, generation, index) (see "
            "paper_1809_11134_b200.functional)")
    raise TypeError(f"expected CounterStreams or an integer seed, got {type(rng).__name__}")


def _device(device: int) -> int:
    return int(device)


# ------------------------------------------------------------------ QEQEA --

def init_population(cfg: PopulationConfig, rng, device: int = 0) -> PopulationState:
    """engine.py:105-112: thetas uniform on [0, 2pi), qutrits normalised complex
    Gaussians (Box-Muller), from the per-slot init streams of `rng.seed`."""
    st = _streams(rng)
    lib = _lib.load()
    th = np.empty(cfg.qubit_count)
    q = np.empty((cfg.qutrit_count, 3), dtype=np.complex128)
    _lib.check(lib.isq_init_population(cfg.number_of_wires, cfg.size_of_individual, cfg.size_of_population,
                                       st.seed, _lib.ptr(th), _lib.ptr(q), _device(device)))
    return PopulationState(thetas=th, qutrits=q)


class SegmentBank:
    """engine.py:115-153: measured axes plus the angle snapshot; descriptor()
    decodes a flat slot, unitary() composes its gate on the device."""

    def __init__(self, cfg: PopulationConfig, templates, thetas: np.ndarray, axes: np.ndarray):
        self.cfg = cfg
        self.templates = templates
        self.thetas = thetas
        self.axes = axes

    def descriptor(self, flat: int) -> GateOp:
        cfg = self.cfg
        kind, _, _ = cfg.decode_flat(int(flat))
        theta = float(self.thetas[flat])
        if kind < cfg.number_of_wires:
            return GateOp(kind="rotation", theta=theta, wire=kind + 1, axis=Axis(int(self.axes[flat])))
        return GateOp(kind="interaction", theta=theta, pair=self.templates[kind - cfg.number_of_wires].pair)

    def unitary(self, flat: int) -> np.ndarray:
        return compose_gates([self.descriptor(flat)], self.cfg.number_of_wires)

    def gate_arrays(self, blueprints: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        """Gate codes (include/isq.h) and angles of (count, L) blueprints."""
        cfg = self.cfg
        bp = np.asarray(blueprints, dtype=np.int64)
        if bp.size and (bp.min() < 0 or bp.max() >= cfg.qubit_count):
            raise ConfigurationError("blueprint slot out of range")
        kind = bp // (cfg.size_of_individual * cfg.size_of_population)
        n = cfg.number_of_wires
        axes = np.asarray(self.axes)
        rot = kind < n
        codes = np.where(rot, 3 * kind + np.where(rot, axes[np.minimum(bp, axes.size - 1)], 0), 3 * n + (kind - n))
        return codes.astype(np.uint8), np.asarray(self.thetas, dtype=np.float64)[bp]


def construct_segments(pop: PopulationState, cfg: PopulationConfig, templates, rng, device: int = 0) -> SegmentBank:
    """engine.py:156-171: Born measurement (n_meas draws, plurality, ties to the
    lower axis) of every qutrit row on its (seed, generation, slot) stream."""
    st = _streams(rng)
    q = np.ascontiguousarray(pop.qutrits, dtype=np.complex128)
    if q.shape != (cfg.qutrit_count, 3):
        raise ConfigurationError("qutrits shape does not match the configuration")
    axes = np.empty(cfg.qutrit_count, dtype=np.int8)
    lib = _lib.load()
    _lib.check(lib.isq_construct_segments(cfg.number_of_wires, cfg.size_of_individual, cfg.size_of_population,
                                          cfg.n_meas, st.seed, st.generation, _lib.ptr(q), _lib.ptr(axes),
                                          _device(device)))
    return SegmentBank(cfg, templates, np.array(pop.thetas, dtype=np.float64), axes.astype(np.int64))


def sample_circuits(cfg: PopulationConfig, rng, count: int, device: int = 0) -> np.ndarray:
    """Blueprints of circuits rng.index .. rng.index + count - 1 of generation
    rng.generation: (count, L) flat slots (engine.py:174-184)."""
    st = _streams(rng)
    out = np.empty((int(count), cfg.size_of_individual), dtype=np.int64)
    lib = _lib.load()
    _lib.check(lib.isq_sample_circuits(cfg.number_of_wires, cfg.size_of_individual, cfg.size_of_population,
                                       st.seed, st.generation, st.index, int(count), _lib.ptr(out),
                                       _device(device)))
    return out


def sample_circuit(cfg: PopulationConfig, rng, device: int = 0) -> np.ndarray:
    """engine.py:174-184: one blueprint (a flat slot per circuit position)."""
    return sample_circuits(cfg, rng, 1, device)[0]


def evaluate_circuits(blueprints: np.ndarray, bank: SegmentBank, target: np.ndarray, device: int = 0,
                      precision: str = "fp64") -> np.ndarray:
    """evaluate_circuit for every row of (count, L) blueprints, one device launch."""
    n = bank.cfg.number_of_wires
    target = np.asarray(target)
    if target.shape[0] != 2 ** n:
        raise ConfigurationError(f"target dimension {target.shape[0]} != 2^{n}")
    bp = np.asarray(blueprints, dtype=np.int64)
    if bp.ndim == 1:
        bp = bp[None, :]
    codes, thetas = bank.gate_arrays(bp)
    return fitness_batch(codes, thetas, target, n, device=device, precision=precision)


def evaluate_circuit(blueprint: np.ndarray, bank: SegmentBank, target: np.ndarray) -> float:
    """engine.py:187-199: compose the blueprint (position 0 first) and score it."""
    return float(evaluate_circuits(np.asarray(blueprint)[None, :], bank, target)[0])




class SegmentFitnessTable:
    """engine.py:202-222 on the device: entries keyed by (flat, position) in a
    device hash, slot_max as u64 atomicMax (fitness >= 0)."""

    def __init__(self, cfg: PopulationConfig, device: int = 0):
        self.cfg = cfg
        self.device = int(device)
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._lib.isq_table_create(cfg.qubit_count, cfg.size_of_individual, self.device,
                                              ctypes.byref(h)))
        self._h = h
        # host copy of slot_max handed out by .slot_max; callers may write it in
        # place (table.slot_max[:] = 1.0, pkg/tests/test_engine.py:192), so it is
        # uploaded before every device update while it is alive
        self._mirror: Optional[np.ndarray] = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value is not None:
            try:
                self._lib.isq_table_destroy(h)
            except Exception:
                pass
            self._h = None

    def _push(self):
        if self._mirror is not None:
            m = np.ascontiguousarray(self._mirror, dtype=np.float64)
            _lib.check(self._lib.isq_table_set_slot_max(self._h, _lib.ptr(m)))

    @property
    def slot_max(self) -> np.ndarray:
        if self._mirror is None:
            m = np.empty(self.cfg.qubit_count)
            _lib.check(self._lib.isq_table_read(self._h, _lib.ptr(m), None, None, None))
            self._mirror = m
        return self._mirror

    @property
    def entries(self) -> Dict[Tuple[int, int], float]:
        n = ctypes.c_int64()
        _lib.check(self._lib.isq_table_read(self._h, None, ctypes.byref(n), None, None))
        keys = np.empty(n.value, dtype=np.int64)
        vals = np.empty(n.value)
        _lib.check(self._lib.isq_table_read(self._h, None, ctypes.byref(n), _lib.ptr(keys), _lib.ptr(vals)))
        L = self.cfg.size_of_individual
        return {(int(k // L), int(k % L)): float(v) for k, v in zip(keys, vals)}

    def update_batch(self, blueprints: np.ndarray, fitnesses: Sequence[float]) -> Set[int]:
        """update() for several circuits in order; returns the union of their improved sets."""
        bp = np.ascontiguousarray(blueprints, dtype=np.int64)
        if bp.ndim == 1:
            bp = bp[None, :]
        fits = np.ascontiguousarray(fitnesses, dtype=np.float64).reshape(-1)
        if bp.shape != (fits.size, self.cfg.size_of_individual):
            raise ConfigurationError("blueprints must be (count, sizeOfIndividual) with one fitness per row")
        self._push()
        improved = np.empty(bp.shape, dtype=np.uint8)
        _lib.check(self._lib.isq_table_update(self._h, fits.size, _lib.ptr(bp), _lib.ptr(fits),
                                              _lib.ptr(improved)))
        if self._mirror is not None:  # the same array object stays current, as the reference's attribute
            _lib.check(self._lib.isq_table_read(self._h, _lib.ptr(self._mirror), None, None, None))
        return {int(f) for f in np.unique(bp[improved.astype(bool)])}

    def update(self, blueprint: np.ndarray, fit: float) -> Set[int]:
        """Elitist keep-best merge; returns the flat slots that improved."""
        return self.update_batch(np.asarray(blueprint)[None, :], [fit])


def mutate_population(pop: PopulationState, table: SegmentFitnessTable, cfg: PopulationConfig, rng,
                      device: int = 0) -> Dict[int, Snapshot]:
    """engine.py:228-263, in place on `pop`: each slot masked with
    probabilityOfMutation (skipped at slot_max >= 1), a fair coin picking the
    qutrit (rotation region) or angle mutation, scaled by (1 - slot_max);
    returns the pre-mutation snapshots of the mutated slots."""
    st = _streams(rng)
    th0 = np.array(pop.thetas, dtype=np.float64)
    q0 = np.array(pop.qutrits, dtype=np.complex128)
    if th0.shape != (cfg.qubit_count,) or q0.shape != (cfg.qutrit_count, 3):
        raise ConfigurationError("population shape does not match the configuration")
    th, q = th0.copy(), np.ascontiguousarray(q0)
    q = q.copy()
    smax = np.ascontiguousarray(table.slot_max, dtype=np.float64)
    mutated = np.empty(cfg.qubit_count, dtype=np.uint8)
    conf = _lib.QeqeaConfig(number_of_wires=cfg.number_of_wires, size_of_individual=cfg.size_of_individual,
                            size_of_population=cfg.size_of_population,
                            probability_of_mutation=cfg.probability_of_mutation,
                            mutation_range=cfg.mutation_range, n_meas=cfg.n_meas, rank=0,
                            max_generations=cfg.max_generations, target_fitness=cfg.target_fitness,
                            seed=st.seed, world=1, precision=0)
    lib = _lib.load()
    _lib.check(lib.isq_mutate_population(ctypes.byref(conf), st.generation, _lib.ptr(th), _lib.ptr(q),
                                         _lib.ptr(smax), _lib.ptr(mutated), _device(device)))
    pop.thetas[:] = th
    pop.qutrits[:] = q
    Qt = cfg.qutrit_count
    return {int(s): (float(th0[s]), q0[s].copy() if s < Qt else None) for s in np.flatnonzero(mutated)}


# --------------------------------------------------------------------- GA --

def random_genome(cfg: GaConfig, rng, device: int = 0) -> CircuitGenome:
    """ga.py:68-73: genome rng.index, each gene a uniform gate choice with a
    uniform angle (per-gene streams)."""
    st = _streams(rng)
    L = cfg.size_of_individual
    codes = np.empty(L, dtype=np.uint8)
    thetas = np.empty(L)
    lib = _lib.load()
    _lib.check(lib.isq_ga_random_genomes(cfg.number_of_wires, L, st.seed, st.index, 1, _lib.ptr(codes),
                                         _lib.ptr(thetas), _device(device)))
    return tuple(gate_from_code(k, t, cfg.number_of_wires) for k, t in zip(codes, thetas))


def decode_genome(genome: CircuitGenome, number_of_wires: int) -> np.ndarray:
    """ga.py:76-78: the genome's unitary (device composition)."""
    return compose_gates(list(genome), number_of_wires)


def two_point_crossover(a: CircuitGenome, b: CircuitGenome, rng,
                        device: int = 0) -> Tuple[CircuitGenome, CircuitGenome]:
    """ga.py:81-92: swap the slice [p, q) of sorted(integers(0, L + 1, size=2))."""
    if len(a) != len(b):
        raise ConfigurationError("crossover requires equal genome lengths")
    if len(a) < 2:
        return a, b
    st = _streams(rng)
    cuts = np.empty(2, dtype=np.int32)
    lib = _lib.load()
    _lib.check(lib.isq_ga_crossover_cuts(len(a), st.seed, st.generation, st.index, 1, _lib.ptr(cuts),
                                         _device(device)))
    p, q = int(cuts[0]), int(cuts[1])
    return a[:p] + b[p:q] + a[q:], b[:p] + a[p:q] + b[q:]


def sus_select(fitnesses: List[float], count: int, rng, device: int = 0) -> List[int]:
    """ga.py:95-116: stochastic universal sampling, uniform picks when every
    fitness is zero."""
    st = _streams(rng)
    f = np.ascontiguousarray(fitnesses, dtype=np.float64)
    picks = np.empty(int(count), dtype=np.int64)
    lib = _lib.load()
    _lib.check(lib.isq_ga_sus_select(f.size, _lib.ptr(f), int(count), st.seed, st.generation, _lib.ptr(picks),
                                     _device(device)))
    return [int(x) for x in picks]


def ga_mutate(genome: CircuitGenome, cfg: GaConfig, rng, device: int = 0) -> CircuitGenome:
    """ga.py:119-138: per-gene Bernoulli mutation of child rng.index of
    generation rng.generation (angle step or, with structural_rate, a new gate
    identity keeping the angle)."""
    st = _streams(rng)
    codes, thetas = encode_gates(list(genome), cfg.number_of_wires)
    conf = _lib.GaConfigC(number_of_wires=cfg.number_of_wires, size_of_individual=len(genome), population=1,
                          mutation_rate=cfg.mutation_rate, mutation_range=cfg.mutation_range,
                          structural_rate=cfg.structural_rate, max_generations=cfg.max_generations,
                          target_fitness=cfg.target_fitness, seed=st.seed, rank=0, world=1, precision=0,
                          reserved=0)
    lib = _lib.load()
    _lib.check(lib.isq_ga_mutate_genomes(ctypes.byref(conf), st.generation, st.index, 1, _lib.ptr(codes),
                                         _lib.ptr(thetas), _device(device)))
    return tuple(gate_from_code(k, t, cfg.number_of_wires) for k, t in zip(codes, thetas))


__all__ = [
    "CounterStreams", "SegmentBank", "SegmentFitnessTable", "construct_segments", "decode_genome",
    "enumerate_templates", "evaluate_circuit", "evaluate_circuits", "ga_mutate", "init_population",
    "mutate_population", "random_genome", "sample_circuit", "sample_circuits", "sus_select",
    "two_point_crossover",
]
