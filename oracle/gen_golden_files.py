"""Target files and circuit text written by the REFERENCE itself (TEST
INFRASTRUCTURE ONLY; build container, /root/reference/pkg/src importable).

  tests/golden/fredkin_ref.mat   fitness.write_target_file of the Fredkin
                                 permutation (C3's target, fitness.py:116-126)
  tests/golden/haar5_ref.mat     the C5 Haar target (conftest.random_unitary(32,
                                 default_rng(12345))), same writer
  tests/golden/circuit_text.json report.render_circuit of seeded gate lists
                                 (report.py:80-96) with the gates themselves

Usage:  python oracle/gen_golden_files.py
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
sys.path.insert(0, str(REF))

from isingsynth.fitness import TargetSpec, write_target_file  # noqa: E402
from isingsynth.gates import Axis, GateOp  # noqa: E402
from isingsynth.report import render_circuit  # noqa: E402


def main():
    m = np.eye(8, dtype=np.complex128)
    m[[5, 6], [5, 6]] = 0.0
    m[5, 6] = m[6, 5] = 1.0
    write_target_file(OUT / "fredkin_ref.mat", TargetSpec("Fredkin", 3, m))
    rng = np.random.default_rng(12345)
    z = rng.normal(size=(32, 32)) + 1j * rng.normal(size=(32, 32))
    q, r = np.linalg.qr(z)
    write_target_file(OUT / "haar5_ref.mat", TargetSpec("haar5", 5, q * (np.diag(r) / np.abs(np.diag(r)))))
    rng = np.random.default_rng(7)
    cases = []
    for n in (2, 3, 5):
        for L in (1, 4, 17):
            gates = []
            for _ in range(L):
                if rng.random() < 0.5:
                    gates.append(GateOp(kind="rotation", theta=float(rng.uniform(0, 2 * math.pi)),
                                        wire=int(rng.integers(1, n + 1)), axis=Axis(int(rng.integers(3)))))
                else:
                    i = int(rng.integers(1, n))
                    j = int(rng.integers(i + 1, n + 1))
                    gates.append(GateOp(kind="interaction", theta=float(rng.uniform(0, 2 * math.pi)), pair=(i, j)))
            cases.append({"n": n, "gates": [g.to_dict() for g in gates], "text": render_circuit(gates)})
    (OUT / "circuit_text.json").write_text(json.dumps(cases, indent=1))
    print("wrote fredkin_ref.mat, haar5_ref.mat, circuit_text.json")


if __name__ == "__main__":
    main()
