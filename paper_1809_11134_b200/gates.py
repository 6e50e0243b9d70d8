"""Ising-model gate descriptors and the device composition entry point.

Mirrors the reference's gate vocabulary (gates.py:30-151): `Axis`, `GateOp`,
`InteractionTemplate`, `pair_signs`, `enumerate_templates`, `rotation_gate`,
`interaction_diagonal`.  Composition (`compose_gates`, gates.py:187-195) runs on
the GPU through libisq; the small 2x2 / diagonal helpers here only describe
gates (they are what tests and readers use to reason about conventions).

Wire 1 is the most significant basis bit; position 0 of a gate list is applied
first (it is the rightmost factor).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import IntEnum
from itertools import combinations
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import ConfigurationError


class Axis(IntEnum):
    X = 0
    Y = 1
    Z = 2

    @property
    def label(self) -> str:
        return "xyz"[self.value]

    @classmethod
    def from_label(cls, label: str) -> "Axis":
        return cls("xyz".index(label.lower()))


_PAULI = {
    0: np.array([[0, 1], [1, 0]], dtype=np.complex128),
    1: np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    2: np.array([[1, 0], [0, -1]], dtype=np.complex128),
}


@dataclass(frozen=True)
class InteractionTemplate:
    """+-1 diagonal of Z_i Z_j over the 2^n basis (gates.py:44-57)."""

    pair: Tuple[int, int]
    signs: np.ndarray

    def __post_init__(self):
        i, j = self.pair
        if not 1 <= i < j:
            raise ConfigurationError(f"invalid wire pair {self.pair}")


def rotation_gate(axis: Axis, theta: float) -> np.ndarray:
    """2x2 rotation cos(th/2) I - i sin(th/2) sigma_axis (gates.py:60-64)."""
    c = math.cos(theta / 2.0)
    s = math.sin(theta / 2.0)
    return c * np.eye(2, dtype=np.complex128) - 1j * s * _PAULI[int(axis)]


def pair_signs(pair: Tuple[int, int], number_of_wires: int) -> np.ndarray:
    """Z_i Z_j diagonal as +-1 over basis states (gates.py:67-73)."""
    i, j = pair
    k = np.arange(2 ** number_of_wires)
    bit_i = (k >> (number_of_wires - i)) & 1
    bit_j = (k >> (number_of_wires - j)) & 1
    return np.where(bit_i == bit_j, 1, -1)


def wire_pairs(number_of_wires: int) -> List[Tuple[int, int]]:
    """All C(n,2) wire pairs in lexicographic order (gates.py:85-88)."""
    return list(combinations(range(1, number_of_wires + 1), 2))


def enumerate_templates(number_of_wires: int) -> List[InteractionTemplate]:
    if number_of_wires < 2:
        raise ConfigurationError(
            f"need at least 2 wires for interactions, got {number_of_wires}"
        )
    return [InteractionTemplate(p, pair_signs(p, number_of_wires)) for p in wire_pairs(number_of_wires)]


def interaction_diagonal(template: InteractionTemplate, theta: float) -> np.ndarray:
    """Entry k = exp(-i th signs[k] / 2) (gates.py:91-93)."""
    return np.exp(-0.5j * theta * template.signs)


@dataclass(frozen=True)
class GateOp:
    """One decoded circuit segment (gates.py:119-151)."""

    kind: str
    theta: float
    wire: Optional[int] = None
    axis: Optional[Axis] = None
    pair: Optional[Tuple[int, int]] = None

    def to_dict(self) -> dict:
        d = {"kind": self.kind, "theta": self.theta}
        if self.kind == "rotation":
            d["wire"] = self.wire
            d["axis"] = self.axis.label
        else:
            d["pair"] = list(self.pair)
        return d

    @classmethod
    def from_dict(cls, d: dict) -> "GateOp":
        if d["kind"] == "rotation":
            return cls(kind="rotation", theta=d["theta"], wire=d["wire"], axis=Axis.from_label(d["axis"]))
        return cls(kind="interaction", theta=d["theta"], pair=tuple(d["pair"]))


# ---- gate codes (include/isq.h) -------------------------------------------

def gate_code_count(number_of_wires: int) -> int:
    n = number_of_wires
    return 3 * n + n * (n - 1) // 2


def gate_code(gate: GateOp, number_of_wires: int) -> int:
    """ga.py:47-59 gate_choices index of `gate`'s identity."""
    n = number_of_wires
    if gate.kind == "rotation":
        if not 1 <= gate.wire <= n:
            raise ConfigurationError(f"wire {gate.wire} out of range 1..{n}")
        return 3 * (gate.wire - 1) + int(gate.axis)
    pairs = wire_pairs(n)
    pair = tuple(gate.pair)
    if pair not in pairs:
        raise ConfigurationError(f"invalid wire pair {gate.pair} for {n} wires")
    return 3 * n + pairs.index(pair)


def gate_from_code(code: int, theta: float, number_of_wires: int) -> GateOp:
    n = number_of_wires
    code = int(code)
    if code < 3 * n:
        return GateOp(kind="rotation", theta=float(theta), wire=code // 3 + 1, axis=Axis(code % 3))
    return GateOp(kind="interaction", theta=float(theta), pair=wire_pairs(n)[code - 3 * n])


def encode_gates(gates: Sequence[GateOp], number_of_wires: int) -> Tuple[np.ndarray, np.ndarray]:
    codes = np.array([gate_code(g, number_of_wires) for g in gates], dtype=np.uint8)
    thetas = np.array([float(g.theta) for g in gates], dtype=np.float64)
    return codes, thetas


def compose_gates(gates: Sequence[GateOp], number_of_wires: int) -> np.ndarray:
    """Circuit unitary of an ordered gate list, composed on the GPU
    (gates.py:187-195: position 0 applied first)."""
    from .fitness import compose_batch

    codes, thetas = encode_gates(gates, number_of_wires)
    return compose_batch(codes[None, :], thetas[None, :], number_of_wires)[0]


def apply_gates(acc: np.ndarray, gates: Sequence[GateOp], number_of_wires: int, device: int = 0) -> np.ndarray:
    """acc left-multiplied by every gate in order (position 0 first), on the
    GPU (isq_apply_gates: each gate applied as row-pair butterflies / row
    phases with its exact matrix).  acc: (D, D) or (count, D, D)."""
    from . import _lib

    n = number_of_wires
    a = np.ascontiguousarray(acc, dtype=np.complex128)
    single = a.ndim == 2
    if single:
        a = a[None]
    d = 2 ** n
    if a.shape[1:] != (d, d):
        raise ConfigurationError(f"accumulator shape {a.shape[1:]} != ({d}, {d})")
    codes, thetas = encode_gates(gates, n)
    count = a.shape[0]
    codes = np.ascontiguousarray(np.broadcast_to(codes, (count, codes.size)))
    thetas = np.ascontiguousarray(np.broadcast_to(thetas, (count, thetas.size)))
    out = np.empty_like(a)
    lib = _lib.load()
    _lib.check(lib.isq_apply_gates(n, codes.shape[1], count, _lib.ptr(codes), _lib.ptr(thetas), _lib.ptr(a),
                                   _lib.ptr(out), int(device)))
    return out[0] if single else out


def apply_gate(acc: np.ndarray, gate: GateOp, number_of_wires: int) -> np.ndarray:
    """gates.py:173-184: the accumulator left-multiplied by the expanded gate."""
    return apply_gates(acc, [gate], number_of_wires)


def expand_rotation(axis: Axis, theta: float, wire: int, number_of_wires: int) -> np.ndarray:
    """gates.py:101-116: a single-wire rotation embedded in the 2^n width."""
    if not 1 <= wire <= number_of_wires:
        raise ConfigurationError(f"wire {wire} out of range 1..{number_of_wires}")
    gate = GateOp(kind="rotation", theta=theta, wire=wire, axis=Axis(int(axis)))
    return apply_gate(np.eye(2 ** number_of_wires, dtype=np.complex128), gate, number_of_wires)


def interaction_gate(template: InteractionTemplate, theta: float) -> np.ndarray:
    """gates.py:96-98: the dense diagonal matrix of J_ij(theta)."""
    n = int(round(math.log2(template.signs.size)))
    gate = GateOp(kind="interaction", theta=theta, pair=tuple(template.pair))
    return apply_gate(np.eye(2 ** n, dtype=np.complex128), gate, n)
