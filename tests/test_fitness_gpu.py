"""Device fitness / composition parity against the reference's golden vectors
and the CPU oracle.  Tolerance (north_star): |d fit| <= 1e-9 |fit_ref| + 1e-12
in fp64; composed unitaries within 1e-12 absolute."""
import math

import numpy as np
import pytest

from conftest import fit_close, golden, random_unitary
from oracle import qeqea as O

pytestmark = pytest.mark.gpu


def _cases():
    g = golden("fitness")
    keys = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_fit")})
    return g, keys


def test_fitness_batch_matches_reference_goldens():
    from paper_1809_11134_b200.fitness import fitness_batch

    g, keys = _cases()
    assert len(keys) >= 50
    for k in keys:
        n = int(k.split("_")[0][1:])
        out = fitness_batch(g[k + "_codes"], g[k + "_thetas"], g[k + "_target"], n)
        ok = fit_close(out, g[k + "_fit"])
        assert ok.all(), (k, out[~ok], g[k + "_fit"][~ok])


def test_compose_batch_matches_reference_goldens():
    from paper_1809_11134_b200.fitness import compose_batch

    g, keys = _cases()
    for k in keys:
        if k + "_unitary" not in g.files:
            continue
        n = int(k.split("_")[0][1:])
        u = compose_batch(g[k + "_codes"], g[k + "_thetas"], n)
        np.testing.assert_allclose(u, g[k + "_unitary"], rtol=0, atol=1e-12, err_msg=k)


@pytest.mark.parametrize("n,L", [(2, 7), (3, 16), (4, 32), (5, 64), (5, 200), (4, 1)])
def test_fitness_batch_matches_oracle_random(n, L):
    from paper_1809_11134_b200.fitness import fitness_batch

    rng = np.random.default_rng(100 + n * 7 + L)
    count = 300
    nc = 3 * n + n * (n - 1) // 2
    codes = rng.integers(0, nc, size=(count, L)).astype(np.uint8)
    thetas = rng.uniform(0, 2 * math.pi, size=(count, L))
    T = random_unitary(2 ** n, rng)
    out = fitness_batch(codes, thetas, T, n)
    ref = np.array([O.circuit_fitness(codes[c], thetas[c], T, n) for c in range(count)])
    assert fit_close(out, ref).all()


def test_fitness_near_one_and_phase_invariance():
    from paper_1809_11134_b200.fitness import fitness_batch, fitness_value

    # a circuit equal to its target up to a global phase has fitness 1
    codes = np.array([[2, 5, 9, 1]], dtype=np.uint8)  # n=3 gates
    thetas = np.array([[0.3, 1.1, 2.0, 4.0]])
    U = O.compose(codes[0], thetas[0], 3)
    out = fitness_batch(codes, thetas, np.exp(0.77j) * U, 3)
    assert out[0] == pytest.approx(1.0, abs=1e-7)
    assert fitness_value(U, U) == pytest.approx(1.0, abs=1e-7)
    x = np.array([[0, 1], [1, 0]], dtype=complex)
    assert fitness_value(x, np.eye(2)) == 0.0
    T = np.eye(4)[[0, 1, 3, 2]].astype(complex)
    assert fitness_value(np.eye(4), T) == pytest.approx(0.2928932188134524, abs=1e-15)


def test_large_batch_c5_shape_properties():
    """At C5 shape (n=5, L=64), 2^16 candidates: fitness in [0,1], equal rows
    give identical fitness (determinism), a sample matches the oracle."""
    from paper_1809_11134_b200.fitness import fitness_batch

    rng = np.random.default_rng(3)
    count, L, n = 1 << 16, 64, 5
    codes = rng.integers(0, 25, size=(count, L)).astype(np.uint8)
    thetas = rng.uniform(0, 2 * math.pi, size=(count, L))
    codes[1::2] = codes[0::2]
    thetas[1::2] = thetas[0::2]
    T = random_unitary(32, np.random.default_rng(12345))
    out = fitness_batch(codes, thetas, T, n)
    assert np.all((out >= 0) & (out <= 1))
    assert np.array_equal(out[0::2], out[1::2])
    idx = rng.choice(count, 40, replace=False)
    ref = np.array([O.circuit_fitness(codes[c], thetas[c], T, n) for c in idx])
    assert fit_close(out[idx], ref).all()


def test_compose_gates_api_matches_oracle():
    from paper_1809_11134_b200.gates import Axis, GateOp, compose_gates

    gates = [GateOp("rotation", 0.4, wire=1, axis=Axis.Y), GateOp("interaction", 2.2, pair=(1, 3)),
             GateOp("rotation", 5.0, wire=3, axis=Axis.X), GateOp("rotation", 1.0, wire=2, axis=Axis.Z)]
    u = compose_gates(gates, 3)
    ref = O.compose([1, 9 + 1, 6, 5], [0.4, 2.2, 5.0, 1.0], 3)
    np.testing.assert_allclose(u, ref, atol=1e-13)
    np.testing.assert_allclose(compose_gates([], 3), np.eye(8), atol=0)


FP32_RTOL, FP32_ATOL = 1e-4, 1e-6  # include/isq.h ISQ_PRECISION_FP32 bound


def test_fp32_variant_matches_reference_goldens_within_stated_bound():
    from paper_1809_11134_b200.fitness import fitness_batch

    g, keys = _cases()
    worst = 0.0
    for k in keys:
        n = int(k.split("_")[0][1:])
        ref = g[k + "_fit"]
        out = fitness_batch(g[k + "_codes"], g[k + "_thetas"], g[k + "_target"], n, precision="fp32")
        err = np.abs(out - ref)
        assert (err <= FP32_RTOL * np.abs(ref) + FP32_ATOL).all(), (k, out, ref)
        worst = max(worst, float(err.max()))
    assert worst > 0.0  # it really is a different arithmetic


@pytest.mark.parametrize("n,L", [(3, 16), (4, 32), (5, 64)])
def test_fp32_variant_matches_oracle_random(n, L):
    from paper_1809_11134_b200.fitness import fitness_batch

    rng = np.random.default_rng(500 + n)
    count = 200
    nc = 3 * n + n * (n - 1) // 2
    codes = rng.integers(0, nc, size=(count, L)).astype(np.uint8)
    thetas = rng.uniform(0, 2 * math.pi, size=(count, L))
    T = random_unitary(2 ** n, rng)
    out = fitness_batch(codes, thetas, T, n, precision="fp32")
    ref = np.array([O.circuit_fitness(codes[c], thetas[c], T, n) for c in range(count)])
    assert (np.abs(out - ref) <= FP32_RTOL * np.abs(ref) + FP32_ATOL).all()


def test_invalid_gate_codes_fail_loudly():
    """A code outside the wire count's gate set: ConfigurationError from the
    host-buffer API (validated on the device, not by a host scan), NaN for
    exactly that circuit from the device API."""
    import torch

    from paper_1809_11134_b200 import _lib
    from paper_1809_11134_b200.errors import ConfigurationError
    from paper_1809_11134_b200.fitness import fitness_batch

    rng = np.random.default_rng(3)
    codes = rng.integers(0, 12, size=(40, 16)).astype(np.uint8)
    thetas = rng.uniform(0, 2 * math.pi, size=(40, 16))
    T = random_unitary(8, rng)
    good = fitness_batch(codes, thetas, T, 3)
    bad = codes.copy()
    bad[17, 5] = 12  # n = 3 has 12 gate choices (ga.py:47-59)
    with pytest.raises(ConfigurationError):
        fitness_batch(bad, thetas, T, 3)
    dev = torch.device("cuda:0")
    c = torch.from_numpy(bad).to(dev)
    t = torch.from_numpy(thetas).to(dev)
    tt = torch.from_numpy(np.ascontiguousarray(T)).to(dev)
    out = torch.empty(40, dtype=torch.float64, device=dev)
    lib = _lib.load()
    _lib.check(lib.isq_fitness_batch_device_ex(3, 16, 40, c.data_ptr(), t.data_ptr(), tt.data_ptr(),
                                               out.data_ptr(), 0, None))
    got = out.cpu().numpy()
    assert np.isnan(got[17]) and not np.isnan(np.delete(got, 17)).any()
    assert np.array_equal(np.delete(got, 17), np.delete(good, 17))
