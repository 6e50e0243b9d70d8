"""GPUGA baseline restated in numpy (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/isingsynth/ga.py: genomes as (code, theta)
arrays (gate_choices order, ga.py:47-59), fitness of the decoded genome
(ga.py:76-78,167-170), elite (171-174), SUS (95-116), pairwise two-point
crossover (81-92, 177-187) and per-gene mutation (119-138), with draws from
the per-unit Philox streams of oracle/streams.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .qeqea import circuit_fitness
from .streams import DOM_GA_INIT, DOM_GA_MUT, DOM_GA_PAIR, DOM_GA_SUS, TWO_PI, stream


@dataclass(frozen=True)
class GaLayout:
    n: int
    L: int
    P: int
    rate: float = 0.1
    mutation_range: float = math.pi / 8
    structural: float = 0.1
    max_generations: int = 10_000_000
    target_fitness: float = 0.999

    @property
    def n_choices(self) -> int:
        return 3 * self.n + self.n * (self.n - 1) // 2


def sus_select(fits, count: int, g: np.random.Generator) -> List[int]:
    """ga.py:95-116."""
    total = float(np.sum(fits))
    if total <= 0.0:
        return [int(g.integers(len(fits))) for _ in range(count)]
    spacing = total / count
    pointer = g.uniform(0.0, spacing)
    picks, cumulative, index = [], 0.0, 0
    for _ in range(count):
        while index < len(fits) - 1 and cumulative + fits[index] <= pointer:
            cumulative += fits[index]
            index += 1
        picks.append(index)
        pointer += spacing
    return picks


def crossover_cuts(L: int, g: np.random.Generator):
    """ga.py:81-92: sorted(integers(0, L+1, size=2)); no draw when L < 2."""
    if L < 2:
        return 0, 0
    p, q = sorted(g.integers(0, L + 1, size=2))
    return int(p), int(q)


def mutate_gene(code: int, theta: float, cfg: GaLayout, g: np.random.Generator):
    """ga.py:126-137 for one gene."""
    if g.random() >= cfg.rate:
        return code, theta
    if g.random() < cfg.structural:
        return int(g.integers(cfg.n_choices)), theta
    return code, (theta + g.uniform(-cfg.mutation_range, cfg.mutation_range)) % TWO_PI


class OracleGa:
    def __init__(self, cfg: GaLayout, target: np.ndarray, seed: int):
        self.cfg = cfg
        self.target = np.asarray(target, dtype=np.complex128)
        self.seed = int(seed)
        self.codes = np.empty((cfg.P, cfg.L), dtype=np.uint8)
        self.thetas = np.empty((cfg.P, cfg.L))
        for i in range(cfg.P):  # random_genome (ga.py:68-73), one stream per gene
            for j in range(cfg.L):
                g = stream(seed, DOM_GA_INIT, 0, i, j)
                self.codes[i, j] = int(g.integers(cfg.n_choices))
                self.thetas[i, j] = g.uniform(0.0, TWO_PI)
        self.generation = 0
        self.best_fitness = 0.0
        self.best_codes: List[int] = []
        self.best_thetas: List[float] = []
        self.stop_reason: Optional[str] = None

    @property
    def done(self) -> bool:
        return self.stop_reason is not None

    def evaluate(self, c0: int, c1: int) -> np.ndarray:
        """Fitness of genomes [c0, c1) (ga.py:167-170)."""
        return np.array([circuit_fitness(self.codes[i], self.thetas[i], self.target, self.cfg.n)
                         for i in range(c0, c1)])

    def step(self, trace: bool = False):
        return self.finish_generation(self.evaluate(0, self.cfg.P), trace=trace)

    def finish_generation(self, fits: np.ndarray, trace: bool = False):
        cfg, gen = self.cfg, self.generation
        fits = np.asarray(fits)
        elite = int(np.argmax(fits))
        if fits[elite] > self.best_fitness:
            self.best_fitness = float(fits[elite])
            self.best_codes = [int(x) for x in self.codes[elite]]
            self.best_thetas = [float(x) for x in self.thetas[elite]]
        parents = sus_select(list(fits), cfg.P, stream(self.seed, DOM_GA_SUS, gen))
        nc = np.empty_like(self.codes)
        nt = np.empty_like(self.thetas)
        nc[0], nt[0] = self.codes[elite], self.thetas[elite]
        i, k = 1, 0
        while i < cfg.P:
            a = parents[(2 * k) % cfg.P]
            b = parents[(2 * k + 1) % cfg.P]
            p, q = crossover_cuts(cfg.L, stream(self.seed, DOM_GA_PAIR, gen, k))
            for first, second in ((a, b), (b, a)):
                if i >= cfg.P:
                    break
                cc = self.codes[first].copy()
                ct = self.thetas[first].copy()
                cc[p:q] = self.codes[second][p:q]
                ct[p:q] = self.thetas[second][p:q]
                for j in range(cfg.L):
                    cc[j], ct[j] = mutate_gene(int(cc[j]), float(ct[j]), cfg,
                                               stream(self.seed, DOM_GA_MUT, gen, i, j))
                nc[i], nt[i] = cc, ct
                i += 1
            k += 1
        self.codes, self.thetas = nc, nt
        self.generation += 1
        if self.best_fitness >= cfg.target_fitness:
            self.stop_reason = "target-reached"
        elif self.generation >= cfg.max_generations:
            self.stop_reason = "generation-limit"
        gb, gm = float(fits.max()), float(np.mean(fits))
        if trace:
            return gb, gm, fits, np.array(parents)
        return gb, gm
