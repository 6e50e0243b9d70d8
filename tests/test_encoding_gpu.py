"""encoding.py's per-unit operators on the device (paper_1809_11134_b200.encoding)
against the reference's own encoding functions on the engines' counter streams
(tests/golden/encoding.npz, oracle/gen_golden_encoding.py)."""
import math

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _g():
    g = golden("encoding")
    seed, first = (int(x) for x in g["meta"])
    return g, seed, first


@pytest.mark.parametrize("gen", [0, 7])
def test_mutations_match_reference(gen):
    from paper_1809_11134_b200.encoding import CounterStreams, mutate_angle, mutate_qutrit

    g, seed, first = _g()
    th = mutate_angle(g["thetas"], g["fits"], 0.7, CounterStreams(seed, gen, first))
    assert np.array_equal(th, g[f"g{gen}_mutate_angle"])  # bit-exact (encoding.py:45-53)
    q = mutate_qutrit(g["qutrits"], g["fits"], CounterStreams(seed, gen, first))
    np.testing.assert_allclose(q, g[f"g{gen}_mutate_qutrit"], rtol=0, atol=1e-14)
    # one unit at a time: the same stream position
    assert mutate_angle(float(g["thetas"][5]), float(g["fits"][5]), 0.7,
                        CounterStreams(seed, gen, first + 5)) == g[f"g{gen}_mutate_angle"][5]


@pytest.mark.parametrize("gen", [0, 7])
@pytest.mark.parametrize("n_meas", [1, 3, 11, 61, 1000])
def test_estimate_axis_matches_reference(gen, n_meas):
    from paper_1809_11134_b200.encoding import CounterStreams, estimate_axis
    from paper_1809_11134_b200.gates import Axis

    g, seed, first = _g()
    axes = estimate_axis(g["qutrits"], n_meas, CounterStreams(seed, gen, first))
    assert np.array_equal(axes, g[f"g{gen}_estimate_nm{n_meas}"])
    one = estimate_axis(g["qutrits"][4], n_meas, CounterStreams(seed, gen, first + 4))
    assert isinstance(one, Axis) and int(one) == g[f"g{gen}_estimate_nm{n_meas}"][4]


@pytest.mark.parametrize("gen", [0, 7])
def test_measure_qutrit_matches_reference(gen):
    from paper_1809_11134_b200.encoding import CounterStreams, measure_qutrit

    g, seed, first = _g()
    assert np.array_equal(measure_qutrit(g["qutrits"], CounterStreams(seed, gen, first)), g[f"g{gen}_measure"])


def test_born_su3_and_random_angle_match_reference():
    from paper_1809_11134_b200.encoding import (CounterStreams, SU3Params, born_probabilities, random_angle,
                                                su3_operator)

    g, seed, first = _g()
    np.testing.assert_allclose(born_probabilities(g["qutrits"]), g["born"], rtol=0, atol=1e-16)
    np.testing.assert_allclose(su3_operator(g["su3_params"]), g["su3"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(su3_operator(SU3Params(*g["su3_params"][3])), g["su3"][3], rtol=0, atol=1e-14)
    for i in (0, 9, 63):
        assert random_angle(CounterStreams(seed, index=first + i)) == g["random_angle"][i]


def test_random_qutrit_is_a_normalised_gaussian_direction():
    """random_qutrit draws Box-Muller normals (numpy's normal() is a ziggurat):
    distributional parity -- unit norm, E|q_k|^2 = 1/3."""
    from paper_1809_11134_b200.encoding import CounterStreams, random_qutrit

    qs = np.array([random_qutrit(CounterStreams(5, index=i)) for i in range(400)])
    assert np.allclose(np.linalg.norm(qs, axis=1), 1.0, atol=1e-12)
    assert np.allclose((np.abs(qs) ** 2).mean(axis=0), 1 / 3, atol=0.05)


def test_invariants_and_generators():
    from paper_1809_11134_b200.encoding import (CounterStreams, born_probabilities, estimate_axis, measure_qutrit,
                                                mutate_angle, read_angle)
    from paper_1809_11134_b200.errors import ConfigurationError, InvariantViolation

    bad = np.array([1.0, 0.01, 0.0], dtype=np.complex128)  # norm^2 = 1.0001
    for call in (lambda: born_probabilities(bad), lambda: estimate_axis(bad, 3, CounterStreams(1)),
                 lambda: measure_qutrit(bad, CounterStreams(1))):
        with pytest.raises(InvariantViolation):
            call()
    with pytest.raises(ConfigurationError):
        estimate_axis(np.array([1, 0, 0], dtype=np.complex128), 0, CounterStreams(1))
    with pytest.raises(TypeError):
        mutate_angle(1.0, 0.5, 0.7, np.random.default_rng(0))
    assert read_angle(math.pi / 3) == math.pi / 3
