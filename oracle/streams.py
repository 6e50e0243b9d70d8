"""Counter-based stream scheme (TEST INFRASTRUCTURE ONLY).

Every random draw of the generation loop comes from numpy's own
Generator(Philox(key=[seed, domain], counter=[0, gen, index, sub])) — one
stream per unit of work — instead of the reference's single sequential
default_rng(seed) (engine.py:283) and per-circuit SeedSequence streams
(engine.py:311-316).  The device reproduces these streams bit for bit
(csrc/np_random.cuh).  Domain numbers are shared with the device.
"""
from __future__ import annotations

import math

import numpy as np

DOM_SAMPLE = 1    # (gen, circuit, 0)  sample_circuit          engine.py:174-184
DOM_MEASURE = 2   # (gen, slot, 0)     construct_segments row  engine.py:167-170
DOM_MUTATE = 3    # (gen, slot, 0)     mutate_population slot  engine.py:241-262
DOM_INIT = 4      # (0, slot, 0)       init_population slot    engine.py:105-112
DOM_GA_INIT = 5   # (0, genome, gene)  random_genome gene      ga.py:68-73
DOM_GA_SUS = 6    # (gen, 0, 0)        sus_select              ga.py:95-116
DOM_GA_PAIR = 7   # (gen, pair, 0)     two_point_crossover     ga.py:81-92
DOM_GA_MUT = 8    # (gen, child, gene) ga_mutate gene          ga.py:119-138

TWO_PI = 2.0 * math.pi


def stream(seed: int, domain: int, gen: int = 0, index: int = 0, sub: int = 0) -> np.random.Generator:
    # explicit uint64 arrays: a Python list holding ints >= 2^63 would be
    # routed through float64 by numpy and lose bits
    key = np.array([int(seed), int(domain)], dtype=np.uint64)
    ctr = np.array([0, int(gen), int(index), int(sub)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key, counter=ctr))


def init_slot(seed: int, slot: int, with_qutrit: bool):
    """Per-slot initial genome unit (replaces init_population's bulk draws,
    engine.py:105-112 + encoding.py:56-63): theta = uniform(0, 2pi); the
    qutrit is a normalised complex Gaussian drawn by Box-Muller from six
    further uniforms (distributionally the reference's normal draws)."""
    g = stream(seed, DOM_INIT, 0, slot)
    theta = g.uniform(0.0, TWO_PI)
    if not with_qutrit:
        return theta, None
    re = np.empty(3)
    im = np.empty(3)
    for k in range(3):
        u1 = g.random()
        u2 = g.random()
        r = math.sqrt(-2.0 * math.log(1.0 - u1))
        re[k] = r * math.cos(TWO_PI * u2)
        im[k] = r * math.sin(TWO_PI * u2)
    amps = re + 1j * im
    return theta, amps / np.linalg.norm(amps)
