"""The reference's encoding module (encoding.py:1-132: phase-encoded angle
carriers and qutrit axis selectors) on the device.

Same names, constants and signatures; `rng` is a `CounterStreams` position
(`paper_1809_11134_b200.functional`) instead of a sequential Generator, so a
call computes exactly what the engines compute for that unit:

    mutate_angle(theta, f, range, CounterStreams(seed, g, s))   the angle step mutate_population
    mutate_qutrit(state, f, CounterStreams(seed, g, s))          gives slot s at the end of generation g
    estimate_axis(state, n_meas, CounterStreams(seed, g, s))     slot s's measurement in generation g
    measure_qutrit(state, CounterStreams(seed, g, s))            one Born draw (stream sub 1)
    random_angle(CounterStreams(seed, index=s))                  slot s's initial angle
    random_qutrit(CounterStreams(seed, index=s))                 slot s's initial qutrit (Box-Muller)

Every operator also takes arrays (a leading batch axis); element i is then
unit `rng.index + i`.  The engines' streams: csrc/np_random.cuh, DESIGN §5.1.
"""
from __future__ import annotations

import math
from dataclasses import astuple, dataclass

import numpy as np

from . import _lib
from .functional import CounterStreams, _streams  # noqa: F401  (CounterStreams re-exported)
from .gates import Axis

TWO_PI = 2.0 * math.pi

# encoding.py:21-23: three mixing angles in (0, pi/2), five phases in (0, 2 pi)
SU3_RANGES = np.array([math.pi / 2] * 3 + [TWO_PI] * 5)


@dataclass(frozen=True)
class SU3Params:
    """Eight parameters of the 3x3 special-unitary mutation operator (encoding.py:26-37)."""

    theta1: float = 0.0
    theta2: float = 0.0
    theta3: float = 0.0
    phi1: float = 0.0
    phi2: float = 0.0
    phi3: float = 0.0
    phi4: float = 0.0
    phi5: float = 0.0


def read_angle(theta: float) -> float:
    """encoding.py:40-42: the stored angle is read back exactly."""
    return theta


def _batch(x, dtype, tail=()):
    a = np.ascontiguousarray(x, dtype=dtype)
    scalar = a.shape == tail
    return a.reshape((-1,) + tail), scalar


def mutate_angle(theta, segment_fitness, mutation_range: float, rng, device: int = 0):
    """encoding.py:45-53: (theta + sign (1 - f) range) mod 2 pi, sign from the
    slot's mutation stream (bit-exact)."""
    st = _streams(rng)
    th, scalar = _batch(theta, np.float64)
    f = np.ascontiguousarray(np.broadcast_to(np.asarray(segment_fitness, dtype=np.float64), th.shape[:1]))
    out = np.empty_like(th)
    _lib.check(_lib.load().isq_mutate_angles(th.shape[0], _lib.ptr(th), _lib.ptr(f), float(mutation_range),
                                             st.seed, st.generation, st.index, _lib.ptr(out), int(device)))
    return float(out[0]) if scalar else out


def mutate_qutrit(state, segment_fitness, rng, device: int = 0) -> np.ndarray:
    """encoding.py:119-132: one of the eight SU(3) parameters (integers(8)),
    drawn from its range shrunk by (1 - f), applied and renormalised."""
    st = _streams(rng)
    q, scalar = _batch(state, np.complex128, (3,))
    f = np.ascontiguousarray(np.broadcast_to(np.asarray(segment_fitness, dtype=np.float64), q.shape[:1]))
    out = np.empty_like(q)
    _lib.check(_lib.load().isq_mutate_qutrits(q.shape[0], _lib.ptr(q), _lib.ptr(f), st.seed, st.generation,
                                              st.index, _lib.ptr(out), int(device)))
    return out[0] if scalar else out


def random_angle(rng, device: int = 0) -> float:
    """encoding.py:56-57: uniform on [0, 2 pi) -- slot rng.index's initial angle."""
    st = _streams(rng)
    th = np.empty(1)
    _lib.check(_lib.load().isq_init_slots(1, st.seed, st.index, 0, _lib.ptr(th), None, int(device)))
    return float(th[0])


def random_qutrit(rng, device: int = 0) -> np.ndarray:
    """encoding.py:60-63: a normalised complex Gaussian 3-vector -- slot
    rng.index's initial qutrit (Box-Muller: distributionally, not bitwise,
    numpy's normal())."""
    st = _streams(rng)
    th = np.empty(1)
    q = np.empty((1, 3), dtype=np.complex128)
    _lib.check(_lib.load().isq_init_slots(1, st.seed, st.index, 1, _lib.ptr(th), _lib.ptr(q), int(device)))
    return q[0]


def born_probabilities(state, device: int = 0) -> np.ndarray:
    """encoding.py:66-71: |amplitude|^2 / norm^2; InvariantViolation when the
    norm^2 deviates from 1 by more than 1e-6."""
    q, scalar = _batch(state, np.complex128, (3,))
    out = np.empty(q.shape, dtype=np.float64)
    _lib.check(_lib.load().isq_born_probabilities(q.shape[0], _lib.ptr(q), _lib.ptr(out), int(device)))
    return out[0] if scalar else out


def _axes(fn, state, rng, *args, device: int = 0):
    st = _streams(rng)
    q, scalar = _batch(state, np.complex128, (3,))
    out = np.empty(q.shape[0], dtype=np.int8)
    _lib.check(getattr(_lib.load(), fn)(q.shape[0], _lib.ptr(q), *args, st.seed, st.generation, st.index,
                                        _lib.ptr(out), int(device)))
    return Axis(int(out[0])) if scalar else out.astype(np.int64)


def measure_qutrit(state, rng, device: int = 0):
    """encoding.py:74-77: one Born-rule draw, Generator.choice(3, p=born); the
    stored state is not collapsed."""
    return _axes("isq_measure_qutrits", state, rng, device=device)


def estimate_axis(state, n_meas: int, rng, device: int = 0):
    """encoding.py:80-84: plurality of multinomial(n_meas, born), ties toward
    X < Y < Z -- the axis construct_segments measures for the slot."""
    if int(n_meas) < 1:
        from .errors import ConfigurationError

        raise ConfigurationError("nMeas must be ≥ 1")
    return _axes("isq_estimate_axes", state, rng, int(n_meas), device=device)


def su3_operator(p, device: int = 0) -> np.ndarray:
    """encoding.py:87-116: the 3x3 special-unitary template.  `p` is an
    SU3Params, 8 numbers, or an (N, 8) array (-> (N, 3, 3))."""
    prm = np.asarray(astuple(p) if isinstance(p, SU3Params) else p, dtype=np.float64)
    prm, scalar = _batch(prm, np.float64, (8,))
    out = np.empty((prm.shape[0], 3, 3), dtype=np.complex128)
    _lib.check(_lib.load().isq_su3_operators(prm.shape[0], _lib.ptr(prm), _lib.ptr(out), int(device)))
    return out[0] if scalar else out
