"""Pins the CPU oracle (oracle/) against the reference: golden vectors the
reference itself produced (oracle/gen_golden.py) and the reference tests'
known-answer values.  CPU only."""
import math

import numpy as np
import pytest

from conftest import golden
from oracle import qeqea as O
from oracle import ga as OG
from oracle.streams import DOM_SAMPLE, init_slot, stream


def test_philox_kat_numpy_counter_convention():
    # numpy Philox increments the counter before each block: the first word of
    # Philox(key=0, counter=0) is Random123's philox4x64_10(ctr=(1,0,0,0), key=0).
    g = np.random.Generator(np.random.Philox(key=[0, 0], counter=[0, 0, 0, 0]))
    assert g.bit_generator.random_raw() == 0x02F4BA6408E4D89B
    # Random123 KAT: ctr = key = 0 -> 16554d9eca36314c db20fe9d672d0fdc ...
    g = np.random.Generator(np.random.Philox(key=[0, 0], counter=[2**64 - 1, 2**64 - 1, 2**64 - 1, 2**64 - 1]))
    assert g.bit_generator.random_raw() == 0x16554D9ECA36314C


@pytest.mark.parametrize("key", ["n2_CNOT", "n3_Toffoli", "n3_Fredkin", "n4_CCCNOT", "n5_haar", "n3_haar"])
def test_oracle_fitness_matches_reference(key):
    g = golden("fitness")
    for L in (0, 1, 3, 16, 33, 64):
        k = f"{key}_L{L}"
        n = int(key[1])
        T = g[k + "_target"]
        for c in range(g[k + "_codes"].shape[0]):
            f = O.circuit_fitness(g[k + "_codes"][c], g[k + "_thetas"][c], T, n)
            assert f == pytest.approx(g[k + "_fit"][c], rel=1e-13, abs=1e-15)


def test_fitness_known_answers():
    cnot = O.compose([0, 3 * 2], [math.pi, 0.0], 2)  # any unitary; check KAT below
    assert cnot.shape == (4, 4)
    T = np.eye(4)[[0, 1, 3, 2]].astype(np.complex128)
    # reference test_fitness.py:62-67: fitness(I4, CNOT) = 1 - sqrt(1/2)
    assert O.fitness_value(np.eye(4, dtype=np.complex128), T) == pytest.approx(0.2928932188134524, abs=1e-15)
    # length-3 CNOT cap (test_output.txt:12)
    assert 1 - math.sqrt(1 - math.sqrt(2) / 2) == pytest.approx(0.4588038998538031, abs=1e-15)
    # reference CNOT circuit (harness.py:158-162) under the default convention
    f = O.circuit_fitness([3 * 0 + 1, 6, 3 * 0 + 0], [math.pi / 2, 3 * math.pi / 2, 3 * math.pi / 2], T, 2)
    assert f == pytest.approx(0.1339745962155614, abs=1e-12)


def test_oracle_sampling_matches_reference():
    g = golden("sampling")
    for key in g.files:
        n, L, P, s, gen = (int(t[1:]) for t in key.split("_"))
        lay = O.Layout(n, L, P)
        bps = g[key]
        for c in range(bps.shape[0]):
            assert np.array_equal(O.sample_blueprint(lay, s, gen, c), bps[c])


def test_oracle_measurement_matches_reference():
    g = golden("measure")
    for nm in (1, 3, 11, 61, 100, 1000):
        q = g[f"nm{nm}_qutrits"]
        for gen in (0, 9):
            axes = O.measure_axes(q, nm, 11, gen, np.arange(q.shape[0]))
            assert np.array_equal(axes, g[f"nm{nm}_g{gen}_axes"])
    # pinned qutrits measure deterministically (test_encoding.py:86-92)
    assert list(g["nm1_g0_axes"][:3]) == [0, 1, 2]


def test_oracle_mutation_matches_reference():
    g = golden("mutate")
    lay = O.Layout(3, 16, 8, p_mut=0.5)
    for gen in (0, 4):
        eng = O.OracleQeqea(lay, np.eye(8), 3, g["thetas0"], g["qutrits0"])
        eng.slot_max = g["slot_max"].copy()
        snaps = eng.mutate(gen)
        mutated = np.zeros(lay.Q, dtype=bool)
        mutated[list(snaps)] = True
        assert np.array_equal(mutated, g[f"g{gen}_mutated"])
        assert np.array_equal(eng.thetas, g[f"g{gen}_thetas"])  # angle path is bit-exact
        np.testing.assert_allclose(eng.qutrits, g[f"g{gen}_qutrits"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("name", ["cnot", "toffoli_c1", "fredkin_c3", "cccnot", "haar5", "identity_conv", "nmeas100",
                                  "nmeas61_n4", "long", "n5_l64"])
def test_oracle_qeqea_trajectory_matches_reference(name):
    g = golden(f"traj_qeqea_{name}")
    lay = O.Layout(int(g["n"]), int(g["L"]), int(g["P"]), p_mut=float(g["p_mut"]),
                   mutation_range=float(g["mutation_range"]), n_meas=int(g["n_meas"]),
                   max_generations=int(g["gens"]), target_fitness=float(g["target_fitness"]))
    eng = O.OracleQeqea(lay, g["target"], int(g["seed"]), g["init_thetas"], g["init_qutrits"])
    recs = []
    ptr = g["improved_ptr"]
    gen = 0
    while not eng.done:
        gb, gm, tr = eng.step(trace=True)
        recs.append((gb, gm, eng.best_fitness))
        assert np.array_equal(tr.blueprints, g["blueprints"][gen])
        assert np.array_equal(tr.improved, g["improved"][ptr[gen]:ptr[gen + 1]])
        np.testing.assert_allclose(tr.fitness, g["fitness"][gen], rtol=1e-12, atol=1e-14)
        if gen == 0:
            assert np.array_equal(tr.axes, g["axes0"])
        gen += 1
    assert gen == int(g["generations_run"])
    assert str(eng.stop_reason) == str(g["stop_reason"])
    np.testing.assert_allclose(np.array(recs), g["records"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(eng.thetas, g["final_thetas"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(eng.qutrits, g["final_qutrits"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(eng.slot_max, g["final_slot_max"], rtol=1e-12, atol=1e-14)
    assert list(eng.best_codes) == list(g["best_codes"])
    np.testing.assert_allclose(eng.best_thetas, g["best_thetas"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("name", ["cnot", "toffoli_c2", "odd13", "l1", "long", "n4", "n5"])
def test_oracle_ga_trajectory_matches_reference(name):
    g = golden(f"traj_ga_{name}")
    cfg = OG.GaLayout(int(g["n"]), int(g["L"]), int(g["P"]), rate=float(g["rate"]),
                      mutation_range=float(g["mrange"]), structural=float(g["structural"]),
                      max_generations=int(g["gens"]), target_fitness=float(g["target_fitness"]))
    eng = OG.OracleGa(cfg, g["target"], int(g["seed"]))
    assert np.array_equal(eng.codes, g["init_codes"])
    assert np.array_equal(eng.thetas, g["init_thetas"])
    recs = []
    gen = 0
    while not eng.done:
        gb, gm, fits, parents = eng.step(trace=True)
        recs.append((gb, gm, eng.best_fitness))
        np.testing.assert_allclose(fits, g["fitness"][gen], rtol=1e-12, atol=1e-14)
        assert np.array_equal(parents, g["parents"][gen])
        gen += 1
    np.testing.assert_allclose(np.array(recs), g["records"], rtol=1e-12, atol=1e-14)
    assert np.array_equal(eng.codes, g["final_codes"])
    np.testing.assert_allclose(eng.thetas, g["final_thetas"], rtol=1e-12, atol=1e-13)
    assert list(eng.best_codes) == list(g["best_codes"])


def test_init_slot_distribution():
    th, q = zip(*[init_slot(3, s, True) for s in range(2000)])
    th = np.array(th)
    q = np.array(q)
    assert np.all((th >= 0) & (th < 2 * math.pi))
    np.testing.assert_allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-12)
    # uniform on the sphere: E|q_k|^2 = 1/3
    np.testing.assert_allclose((np.abs(q) ** 2).mean(axis=0), 1 / 3, atol=0.03)


def test_sampling_stream_layout():
    # integers(P, size=L) consumes u32 halves low-first; the next call continues
    # from the buffered half.
    g = stream(5, DOM_SAMPLE, 2, 9)
    raw = np.random.Generator(np.random.Philox(key=[5, DOM_SAMPLE], counter=[0, 2, 9, 0]))
    words = [raw.bit_generator.random_raw() for _ in range(4)]
    u32 = []
    for w in words:
        u32 += [w & 0xFFFFFFFF, w >> 32]
    a = g.integers(1024, size=3)
    b = g.integers(15, size=2)
    assert list(a) == [(u * 1024) >> 32 for u in u32[:3]]
    assert list(b) == [(u * 15) >> 32 for u in u32[3:5]]


def test_exp_log_identity_on_binomial_q():
    """numpy's random_binomial_inversion computes qn = exp(n * log(q)) with the
    C library; for n = 1 (the default n_meas) the device takes qn = q
    (csrc/np_random.cuh binomial_inversion).  That is exact iff the C
    library's exp(log(q)) returns q for every q = 1 - p, p in [0, 0.5]."""
    import math
    import random
    import struct

    def step(x, k):
        return struct.unpack("<d", struct.pack("<q", struct.unpack("<q", struct.pack("<d", x))[0] + k))[0]

    rng = random.Random(5)
    qs = [1.0 - 0.5 * rng.random() for _ in range(200_000)]
    qs += [step(0.5, k) for k in range(50_000)] + [step(1.0, -k) for k in range(50_000)] + [0.5, 1.0]
    assert all(math.exp(1.0 * math.log(q)) == q for q in qs)


def test_binomial_restatement_matches_numpy():
    """oracle/binomial.py (inversion + BTPE, the device's transcription source)
    against numpy's own Generator draws on Philox streams, including the BTPE
    branch (n * min(p, 1 - p) > 30) that nMeas > 60 reaches."""
    from oracle.binomial import binomial, multinomial3
    from oracle.streams import stream

    rng = np.random.default_rng(1)
    for trial in range(3000):
        n = int(rng.choice([61, 100, 257, 1000, 100000]))
        p = float(rng.uniform(0.01, 0.99))
        assert stream(7, 2, trial, 0).binomial(n, p) == binomial(stream(7, 2, trial, 0), p, n)
    for trial in range(3000):
        n = int(rng.choice([1, 11, 61, 100, 1000]))
        q = rng.normal(size=3) + 1j * rng.normal(size=3)
        pr = np.abs(q) ** 2
        pr /= pr.sum()
        assert list(stream(7, 2, trial, 1).multinomial(n, pr)) == multinomial3(stream(7, 2, trial, 1), n, list(pr))


def _sus_cases():
    g = golden("sus_large")
    return g, sorted({k.rsplit("_", 1)[0] for k in g.files})


def test_oracle_sus_select_matches_reference_at_large_populations():
    """oracle/ga.sus_select (the restatement the device is checked against)
    against the reference's own picks at P up to 300k (oracle/gen_golden_sus.py)."""
    import hashlib

    from oracle.streams import DOM_GA_SUS
    from oracle.targets import sus_fitness

    g, names = _sus_cases()
    assert len(names) == 9
    for name in names:
        P, count, seed, gen = (int(x) for x in g[name + "_meta"])
        f = sus_fitness(P, seed, str(g[name + "_kind"]))
        assert float(np.sum(list(map(float, f)))) == float(g[name + "_total"])
        picks = np.asarray(OG.sus_select(list(map(float, f)), count, stream(seed, DOM_GA_SUS, gen)), dtype=np.int64)
        assert hashlib.sha256(picks.astype("<i8").tobytes()).hexdigest() == str(g[name + "_sha"]), name


def test_oracle_encoding_matches_reference_goldens():
    """The oracle's encoding restatement (mutate_angle, mutate_qutrit,
    su3_operator) and the measurement recipe it uses against the reference's
    own functions on the same streams (tests/golden/encoding.npz)."""
    from oracle.streams import DOM_MEASURE, DOM_MUTATE

    g = golden("encoding")
    seed, first = (int(x) for x in g["meta"])
    th, q, f = g["thetas"], g["qutrits"], g["fits"]
    for gen in (0, 7):
        ma, mq = [], []
        for i in range(th.size):
            st = stream(seed, DOM_MUTATE, gen, first + i)
            st.random(), st.random()
            ma.append(O.mutate_angle(float(th[i]), float(f[i]), 0.7, st))
            st = stream(seed, DOM_MUTATE, gen, first + i)
            st.random(), st.random()
            mq.append(O.mutate_qutrit(q[i], float(f[i]), st))
        assert np.array_equal(np.array(ma), g[f"g{gen}_mutate_angle"])
        np.testing.assert_allclose(np.array(mq), g[f"g{gen}_mutate_qutrit"], rtol=0, atol=1e-15)
        for nm in (1, 11, 1000):
            want = [int(np.argmax(stream(seed, DOM_MEASURE, gen, first + i).multinomial(
                nm, np.abs(q[i]) ** 2 / (np.abs(q[i]) ** 2).sum()))) for i in range(th.size)]
            assert np.array_equal(np.array(want), g[f"g{gen}_estimate_nm{nm}"])
    np.testing.assert_allclose(np.array([O.su3_operator(p) for p in g["su3_params"]]), g["su3"], rtol=0, atol=0)
