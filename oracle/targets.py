"""Deterministic wide targets for the n >= 9 fixtures (TEST INFRASTRUCTURE
ONLY).  A 2^13 x 2^13 complex target is 1 GB, so the fixtures store a seed
and both the generator (oracle/gen_golden_xwide.py, reference side) and the
tests rebuild the same matrix with plain numpy."""
from __future__ import annotations

import numpy as np


def _near_identity(rng: np.random.Generator) -> np.ndarray:
    """exp(-i a/2 (n . sigma)) with a random axis n and a in [0, 0.6): near
    the identity, so short circuits score well away from zero."""
    a = rng.uniform(0.0, 0.6)
    v = rng.normal(size=3)
    nx, ny, nz = v / np.linalg.norm(v)
    c, s = np.cos(a / 2), np.sin(a / 2)
    return np.array([[c - 1j * s * nz, -1j * s * nx - s * ny],
                     [-1j * s * nx + s * ny, c + 1j * s * nz]], dtype=np.complex128)


def product_target(n: int, seed: int) -> np.ndarray:
    """Kronecker product of n seeded near-identity 2 x 2 unitaries (wire 1 =
    most significant factor) times a ZZ-type diagonal phase on wires 1, 2."""
    rng = np.random.default_rng(seed)
    m = np.ones((1, 1), dtype=np.complex128)
    for _ in range(n):
        m = np.kron(m, _near_identity(rng))
    r = np.arange(2 ** n)
    par = ((r >> (n - 1)) ^ (r >> (n - 2))) & 1
    m *= np.exp(1j * 0.35 * (1 - 2 * par))[:, None]
    return m


def sus_fitness(P: int, seed: int, kind: str) -> np.ndarray:
    """Fitness vectors for the large-population SUS fixtures
    (oracle/gen_golden_sus.py): `skewed` spans many binades, `zeros` adds 30 %
    exact zeros, `ties` are dyadic multiples of 1/8 (exact sums, pointer ties)."""
    rng = np.random.default_rng(seed)
    if kind == "skewed":
        return rng.random(P) ** 6
    if kind == "zeros":
        f = rng.random(P) ** 2
        f[rng.random(P) < 0.3] = 0.0
        return f
    if kind == "ties":
        return rng.integers(0, 5, P) * 0.125
    if kind in ("range", "dyadic", "tie40"):
        return sus_fitness_extra(P, seed, kind)
    raise ValueError(kind)


def sus_fitness_extra(P: int, seed: int, kind: str) -> np.ndarray:
    """More SUS fixtures: `range` spans 1e-300 .. 1 (many binade crossings,
    subnormal-free), `dyadic` are multiples of 1/8 with a power-of-two count
    (an exactly dyadic spacing: a whole binade of exact rounding ties in the
    pointer sum)."""
    rng = np.random.default_rng(seed)
    if kind == "range":
        return 10.0 ** rng.uniform(-300.0, 0.0, P)
    if kind == "dyadic":
        return rng.integers(1, 9, P) * 0.125
    if kind == "tie40":  # k 2^-40: while the running sum is in [2^13, 2^14), half the adds are exact ties
        return rng.integers(1, 1 << 40, P).astype(np.float64) * 2.0 ** -40
    raise ValueError(kind)
