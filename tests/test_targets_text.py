"""Target-file ingestion (fitness.py:84-126) and the circuit text format
(report.py:80-124), against files and text the reference wrote itself
(oracle/gen_golden_files.py) and the reference tests' cases
(pkg/tests/test_fitness.py:125-148, pkg/tests/test_harness.py:36-60)."""
import json
import math

import numpy as np
import pytest

from conftest import GOLDEN, random_unitary

from paper_1809_11134_b200.errors import ConfigurationError
from paper_1809_11134_b200.fitness import TargetSpec, load_target_file, target_matrix, write_target_file
from paper_1809_11134_b200.gates import Axis, GateOp
from paper_1809_11134_b200.report import parse_circuit_text, render_circuit


def test_reference_written_fredkin_file_equals_named_fredkin():
    spec = load_target_file(GOLDEN / "fredkin_ref.mat")
    assert spec.number_of_wires == 3
    assert np.array_equal(spec.matrix, target_matrix("Fredkin").matrix)
    # target_matrix accepts a file path as the reference does (fitness.py:76-80)
    assert np.array_equal(target_matrix(str(GOLDEN / "fredkin_ref.mat"), 3).matrix, spec.matrix)
    with pytest.raises(ConfigurationError):
        target_matrix(str(GOLDEN / "fredkin_ref.mat"), 4)


def test_reference_written_haar_file_loads_bit_exact():
    from paper_1809_11134_b200.synthetic import haar_target

    spec = load_target_file(GOLDEN / "haar5_ref.mat")
    assert spec.number_of_wires == 5
    assert np.array_equal(spec.matrix, haar_target(5))  # %.17g round trip is exact


def test_target_file_round_trip(tmp_path, rng):
    spec = target_matrix("CNOT")
    write_target_file(tmp_path / "cnot.mat", spec)
    loaded = load_target_file(tmp_path / "cnot.mat")
    assert loaded.number_of_wires == 2 and np.array_equal(loaded.matrix, spec.matrix)
    u = random_unitary(8, rng)
    write_target_file(tmp_path / "u.mat", TargetSpec("u", 3, u))
    assert np.array_equal(load_target_file(tmp_path / "u.mat").matrix, u)
    # our writer's output is the reference writer's format byte for byte
    write_target_file(tmp_path / "f.mat", target_matrix("Fredkin"))
    assert (tmp_path / "f.mat").read_text() == (GOLDEN / "fredkin_ref.mat").read_text()


def test_target_file_rejects_garbage(tmp_path):
    bad = tmp_path / "bad.mat"
    bad.write_text("2\n1 0 0 0\n0 1 0 0\n0 0 1 0\n")
    with pytest.raises(ConfigurationError):
        load_target_file(bad)
    nonunitary = tmp_path / "nu.mat"
    nonunitary.write_text("1\n1+0j 0+0j\n0+0j 2+0j\n")
    with pytest.raises(ConfigurationError, match="not unitary"):
        load_target_file(nonunitary)
    # the unitarity check is at 1e-9 (fitness.py:107-112): just inside passes, just outside fails
    for eps, ok in ((1e-10, True), (1e-8, False)):
        f = tmp_path / f"eps{eps}.mat"
        f.write_text(f"1\n{1 + eps!r}+0j 0+0j\n0+0j 1+0j\n")
        if ok:
            load_target_file(f)
        else:
            with pytest.raises(ConfigurationError, match="not unitary"):
                load_target_file(f)
    with pytest.raises(ConfigurationError):
        target_matrix("no-such-gate")


def test_render_circuit_exact_text():
    gates = [
        GateOp(kind="rotation", theta=math.pi / 2, wire=1, axis=Axis.Y),
        GateOp(kind="interaction", theta=3 * math.pi / 2, pair=(1, 2)),
        GateOp(kind="rotation", theta=3 * math.pi / 2, wire=1, axis=Axis.X),
    ]
    assert render_circuit(gates) == "R1y(θ=1.570796)J12(θ=4.712389)R1x(θ=4.712389)"


def test_render_matches_reference_text_and_parses_back():
    cases = json.loads((GOLDEN / "circuit_text.json").read_text())
    assert len(cases) >= 9
    for case in cases:
        gates = [GateOp.from_dict(d) for d in case["gates"]]
        assert render_circuit(gates) == case["text"]
        back = parse_circuit_text(case["text"])
        assert len(back) == len(gates)
        for a, b in zip(back, gates):
            assert (a.kind, a.wire, a.axis, a.pair) == (b.kind, b.wire, b.axis, b.pair)
            assert abs(a.theta - b.theta) <= 5e-7  # 6 decimals
        assert render_circuit(back) == case["text"]


def test_parse_rejects_garbage():
    with pytest.raises(ValueError):
        parse_circuit_text("R1q(θ=1.0)")
    assert parse_circuit_text("") == []


@pytest.mark.gpu
def test_file_target_scores_like_the_named_target():
    from paper_1809_11134_b200.fitness import fitness_batch

    rng = np.random.default_rng(3)
    codes = rng.integers(0, 12, size=(256, 16)).astype(np.uint8)
    thetas = rng.uniform(0, 2 * math.pi, size=(256, 16))
    a = fitness_batch(codes, thetas, load_target_file(GOLDEN / "fredkin_ref.mat"), 3)
    b = fitness_batch(codes, thetas, target_matrix("Fredkin"), 3)
    assert np.array_equal(a, b)
