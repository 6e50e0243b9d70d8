"""QEQEA generation loop restated in numpy (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/isingsynth/engine.py step() (318-361)
phase by phase, eagerly over the whole bank exactly as the reference does,
with every random draw taken from the per-unit Philox streams of
oracle/streams.py.  Arithmetic follows the reference's own formulas:
dense Kronecker-expanded rotations and row-scaled interactions
(gates.py:101-116,154-184), trace fidelity (fitness.py:36-49), angle and
qutrit mutation (encoding.py:45-53,87-132).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache
from itertools import combinations
from typing import Dict, List, Optional, Tuple

import numpy as np

from .streams import (
    DOM_MEASURE,
    DOM_MUTATE,
    DOM_SAMPLE,
    TWO_PI,
    init_slot,
    stream,
)

# encoding.py:23 — three mixing angles in (0, pi/2), five phases in (0, 2pi)
SU3_RANGES = np.array([math.pi / 2] * 3 + [TWO_PI] * 5)

_PAULI = (
    np.array([[0, 1], [1, 0]], dtype=np.complex128),
    np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    np.array([[1, 0], [0, -1]], dtype=np.complex128),
)


# ---------------------------------------------------------------- layout ---

@dataclass(frozen=True)
class Layout:
    """engine.py:33-94 slot accounting."""

    n: int
    L: int
    P: int
    p_mut: float = 0.3
    mutation_range: float = math.pi / 4
    n_meas: int = 1
    max_generations: int = 10_000_000
    target_fitness: float = 0.999

    @property
    def K(self) -> int:  # slot kinds: n rotations + C(n,2) interactions (engine.py:65-72)
        return self.n + self.n * (self.n - 1) // 2

    @property
    def Q(self) -> int:  # qubit_count (engine.py:74-76)
        return self.K * self.P * self.L

    @property
    def Qt(self) -> int:  # qutrit_count (engine.py:78-80)
        return self.n * self.P * self.L

    def flat(self, kind, ind, pos):  # engine.py:82-87
        return kind * self.L * self.P + ind * self.L + pos

    def decode(self, flat: int) -> Tuple[int, int, int]:  # engine.py:89-94
        kind, rest = divmod(int(flat), self.L * self.P)
        ind, pos = divmod(rest, self.L)
        return kind, ind, pos


def pairs(n: int):
    return list(combinations(range(1, n + 1), 2))


def gate_code(layout: Layout, flat: int, axis: int) -> int:
    """Slot -> gate code (include/isq.h), via SegmentBank.descriptor (engine.py:134-146)."""
    kind = int(flat) // (layout.L * layout.P)
    if kind < layout.n:
        return 3 * kind + int(axis)
    return 3 * layout.n + (kind - layout.n)


# ------------------------------------------------------------- gates/fit ---

def rotation_2x2(axis: int, theta: float) -> np.ndarray:  # gates.py:60-64
    c = math.cos(theta / 2.0)
    s = math.sin(theta / 2.0)
    return c * np.eye(2, dtype=np.complex128) - 1j * s * _PAULI[axis]


@lru_cache(maxsize=16384)
def _expanded(axis: int, theta: float, wire: int, n: int) -> np.ndarray:  # gates.py:101-116,154-160
    g = rotation_2x2(axis, theta)
    left, right = 2 ** (wire - 1), 2 ** (n - wire)
    if left > 1:
        g = np.kron(np.eye(left, dtype=np.complex128), g)
    if right > 1:
        g = np.kron(g, np.eye(right, dtype=np.complex128))
    g.setflags(write=False)
    return g


@lru_cache(maxsize=16384)
def _interaction(pair: Tuple[int, int], theta: float, n: int) -> np.ndarray:  # gates.py:67-98,163-170
    k = np.arange(2 ** n)
    bi = (k >> (n - pair[0])) & 1
    bj = (k >> (n - pair[1])) & 1
    signs = np.where(bi == bj, 1, -1)
    d = np.exp(-0.5j * theta * signs)
    d.setflags(write=False)
    return d


def apply_code(acc: np.ndarray, code: int, theta: float, n: int) -> np.ndarray:  # gates.py:173-184
    code = int(code)
    if code < 3 * n:
        return _expanded(code % 3, float(theta), code // 3 + 1, n) @ acc
    return _interaction(pairs(n)[code - 3 * n], float(theta), n)[:, None] * acc


def compose(codes, thetas, n: int) -> np.ndarray:  # gates.py:187-195
    acc = np.eye(2 ** n, dtype=np.complex128)
    for c, t in zip(codes, thetas):
        acc = apply_code(acc, c, t, n)
    return acc


def fitness_value(s: np.ndarray, t: np.ndarray) -> float:  # fitness.py:36-49
    size = s.shape[0]
    overlap = abs(np.sum(s.conj() * t))
    radicand = max(0.0, (size - overlap) / size)
    return min(1.0, max(0.0, 1.0 - math.sqrt(radicand)))


def circuit_fitness(codes, thetas, target: np.ndarray, n: int) -> float:
    return fitness_value(compose(codes, thetas, n), target)


# -------------------------------------------------------------- encoding ---

def mutate_angle(theta: float, f: float, rng_: float, g: np.random.Generator) -> float:
    """encoding.py:45-53."""
    sign = 1.0 if g.random() < 0.5 else -1.0
    return (theta + sign * (1.0 - f) * rng_) % TWO_PI


def su3_operator(p) -> np.ndarray:
    """encoding.py:87-116 (Eq. 11), parameters (t1, t2, t3, f1..f5)."""
    t1, t2, t3, f1, f2, f3, f4, f5 = p
    c1, c2, c3 = math.cos(t1), math.cos(t2), math.cos(t3)
    s1, s2, s3 = math.sin(t1), math.sin(t2), math.sin(t3)
    e = np.exp
    return np.array(
        [
            [e(1j * f1) * c1 * c2, e(1j * f3) * s1, e(1j * f4) * c1 * s2],
            [
                e(-1j * f4 - 1j * f5) * s2 * s3 - e(1j * (f1 + f2 - f3)) * s1 * c2 * c3,
                e(1j * f2) * c1 * c3,
                -e(-1j * f1 - 1j * f5) * c2 * s3 - e(1j * (f2 - f3 + f4)) * s1 * s2 * c3,
            ],
            [
                -e(-1j * f2 - 1j * f4) * s2 * c3 - e(1j * (f1 - f3 + f5)) * s1 * c2 * s3,
                e(1j * f5) * c1 * s3,
                e(-1j * f1 - 1j * f2) * c2 * c3 - e(1j * (-f3 + f4 + f5)) * s1 * s2 * s3,
            ],
        ],
        dtype=np.complex128,
    )


def mutate_qutrit(state: np.ndarray, f: float, g: np.random.Generator) -> np.ndarray:
    """encoding.py:119-132: one of the eight SU(3) parameters, drawn from its
    domain shrunk by (1 - f), then renormalised."""
    which = int(g.integers(8))
    value = g.uniform(0.0, SU3_RANGES[which] * (1.0 - f))
    params = [0.0] * 8
    params[which] = value
    new = su3_operator(params) @ state
    return new / np.linalg.norm(new)


def measure_axes(qutrits: np.ndarray, n_meas: int, seed: int, gen: int, slots) -> np.ndarray:
    """construct_segments (engine.py:167-170) for the given rotation slots, one
    multinomial row per slot stream."""
    slots = np.asarray(slots, dtype=np.int64)
    if slots.size == 0:
        return np.zeros(0, dtype=np.int64)
    probs = np.abs(qutrits[slots]) ** 2
    probs /= probs.sum(axis=1, keepdims=True)
    axes = np.empty(slots.size, dtype=np.int64)
    for i, s in enumerate(slots):
        counts = stream(seed, DOM_MEASURE, gen, int(s)).multinomial(n_meas, probs[i])
        axes[i] = int(np.argmax(counts))
    return axes


def sample_blueprint(layout: Layout, seed: int, gen: int, c: int) -> np.ndarray:
    """sample_circuit (engine.py:174-184) on stream (seed, DOM_SAMPLE, gen, c)."""
    g = stream(seed, DOM_SAMPLE, gen, c)
    L = layout.L
    which_individual = g.integers(layout.P, size=L)
    which_kind = g.integers(layout.K, size=L)
    return which_kind * L * layout.P + which_individual * L + np.arange(L)


# ---------------------------------------------------------------- engine ---

@dataclass
class GenerationTrace:
    blueprints: np.ndarray         # (P, L) int64
    axes: np.ndarray               # (Qt,) int64 measured axes of this generation
    fitness: np.ndarray            # (P,)
    improved: np.ndarray           # sorted int64 slots
    gen_best: float
    gen_mean: float


class OracleQeqea:
    """Eager restatement of QeqeaEngine (engine.py:266-384) on Philox streams."""

    def __init__(self, layout: Layout, target: np.ndarray, seed: int,
                 thetas: Optional[np.ndarray] = None, qutrits: Optional[np.ndarray] = None):
        self.layout = layout
        self.target = np.asarray(target, dtype=np.complex128)
        self.seed = int(seed)
        if thetas is None:
            thetas = np.empty(layout.Q)
            qutrits = np.empty((layout.Qt, 3), dtype=np.complex128)
            for s in range(layout.Q):
                th, q = init_slot(seed, s, s < layout.Qt)
                thetas[s] = th
                if q is not None:
                    qutrits[s] = q
        self.thetas = np.array(thetas, dtype=np.float64, copy=True)
        self.qutrits = np.array(qutrits, dtype=np.complex128, copy=True)
        self.slot_max = np.zeros(layout.Q)
        self.pending: Dict[int, Tuple[float, Optional[np.ndarray]]] = {}
        self.generation = 0
        self.best_fitness = 0.0
        self.best_codes: List[int] = []
        self.best_thetas: List[float] = []
        self.stop_reason: Optional[str] = None

    @property
    def done(self) -> bool:
        return self.stop_reason is not None

    # The generation is split into phases so a population-sharded driver can
    # score a subset of the circuits and finish on the gathered fitness vector.
    def begin_generation(self):
        lay, g = self.layout, self.generation
        # construct_segments (engine.py:156-171)
        self._axes = measure_axes(self.qutrits, lay.n_meas, self.seed, g, np.arange(lay.Qt))
        self._bank_thetas = self.thetas.copy()
        # sample_circuit x P (engine.py:322-325)
        self._bps = np.stack([sample_blueprint(lay, self.seed, g, c) for c in range(lay.P)])
        self._codes = np.array([[gate_code(lay, f, self._axes[f] if f < lay.Qt else 0) for f in bp]
                                for bp in self._bps], dtype=np.int64)

    def evaluate(self, c0: int, c1: int) -> np.ndarray:
        """evaluate_circuit for circuits [c0, c1) (engine.py:187-199, 326-336)."""
        return np.array([circuit_fitness(self._codes[c], self._bank_thetas[self._bps[c]], self.target,
                                         self.layout.n) for c in range(c0, c1)])

    def finish_generation(self, fits: np.ndarray, trace: bool = False):
        lay, g = self.layout, self.generation
        bps, codes_all, bank_thetas = self._bps, self._codes, self._bank_thetas
        # table update + best tracking (engine.py:202-222, 338-343)
        improved = set()
        for c in range(lay.P):
            fit = fits[c]
            for flat in bps[c]:
                flat = int(flat)
                if fit > self.slot_max[flat]:
                    self.slot_max[flat] = fit
                    improved.add(flat)
            if fit > self.best_fitness:
                self.best_fitness = float(fit)
                self.best_codes = [int(x) for x in codes_all[c]]
                self.best_thetas = [float(bank_thetas[f]) for f in bps[c]]
        # elitist revert of last generation's mutations (engine.py:345-351)
        for flat, (theta, qutrit) in self.pending.items():
            if flat not in improved:
                self.thetas[flat] = theta
                if qutrit is not None:
                    self.qutrits[flat] = qutrit
        # mutate_population (engine.py:228-263) with one stream per slot
        self.pending = self.mutate(g)
        self.generation += 1
        if self.best_fitness >= lay.target_fitness:
            self.stop_reason = "target-reached"
        elif self.generation >= lay.max_generations:
            self.stop_reason = "generation-limit"
        gen_best = float(max(fits))
        gen_mean = float(np.mean(fits))
        if trace:
            return gen_best, gen_mean, GenerationTrace(
                bps, self._axes, np.asarray(fits), np.array(sorted(improved), dtype=np.int64),
                gen_best, gen_mean)
        return gen_best, gen_mean

    def step(self, trace: bool = False):
        self.begin_generation()
        return self.finish_generation(self.evaluate(0, self.layout.P), trace=trace)

    def mutate(self, g: int) -> Dict[int, Tuple[float, Optional[np.ndarray]]]:
        lay = self.layout
        snapshots: Dict[int, Tuple[float, Optional[np.ndarray]]] = {}
        for flat in range(lay.Q):
            st = stream(self.seed, DOM_MUTATE, g, flat)
            masked = st.random() < lay.p_mut
            coin = st.random() < 0.5
            if not masked:
                continue
            f = float(self.slot_max[flat])
            if f >= 1.0:
                continue
            has_q = flat < lay.Qt
            snapshots[flat] = (float(self.thetas[flat]), self.qutrits[flat].copy() if has_q else None)
            if coin and has_q:
                self.qutrits[flat] = mutate_qutrit(self.qutrits[flat], f, st)
            else:
                self.thetas[flat] = mutate_angle(self.thetas[flat], f, lay.mutation_range, st)
        return snapshots
