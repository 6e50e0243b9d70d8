"""QEQEA engine parity on the device (QeqeaEngine, engine.py:266-384).

Trajectories are compared generation by generation with the fixtures the
reference produced itself (oracle/gen_golden.py: the reference engine driven by
the same Philox streams, started from the reference's own init_population):
blueprints bit-exact, fitness / records within the fp64 tolerance, final bank,
table, best circuit and stop reason."""
import math
import pickle

import numpy as np
import pytest

from conftest import fit_close, golden, random_unitary
from oracle import qeqea as O

pytestmark = pytest.mark.gpu

TRAJ = ["cnot", "toffoli_c1", "fredkin_c3", "cccnot", "haar5", "identity_conv", "nmeas100", "nmeas61_n4", "long",
        "n5_l64"]


def _engine_from_golden(g, **kw):
    from paper_1809_11134_b200.engine import PopulationConfig, PopulationState, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    cfg = PopulationConfig(
        number_of_wires=int(g["n"]), size_of_individual=int(g["L"]), size_of_population=int(g["P"]),
        probability_of_mutation=float(g["p_mut"]), mutation_range=float(g["mutation_range"]),
        n_meas=int(g["n_meas"]), max_generations=int(g["gens"]), target_fitness=float(g["target_fitness"]))
    spec = TargetSpec("golden", cfg.number_of_wires, g["target"])
    pop = PopulationState(g["init_thetas"].copy(), g["init_qutrits"].copy())
    return QeqeaEngine(cfg, spec, int(g["seed"]), population=pop, **kw)


@pytest.mark.parametrize("name", TRAJ)
@pytest.mark.parametrize("mode", ["auto", "kernels", "fused"])
def test_trajectory_matches_reference(name, mode):
    g = golden(f"traj_qeqea_{name}")
    eng = _engine_from_golden(g)
    eng.set_launch_mode(mode)
    gen = 0
    recs = []
    while not eng.done:
        flats, codes, thetas = eng.sample()
        assert np.array_equal(flats, g["blueprints"][gen]), f"blueprints differ at generation {gen}"
        gb, gm = eng.step()
        recs.append((gb, gm, eng.best_fitness))
        fit = eng.last_fitness()
        ok = fit_close(fit, g["fitness"][gen])
        assert ok.all(), (gen, fit[~ok], g["fitness"][gen][~ok])
        gen += 1
    assert gen == int(g["generations_run"])
    assert eng.stop_reason == str(g["stop_reason"])
    assert fit_close(np.array(recs), g["records"]).all()
    pop = eng.pop
    np.testing.assert_allclose(pop.thetas, g["final_thetas"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(pop.qutrits, g["final_qutrits"], rtol=0, atol=1e-11)
    assert fit_close(eng.table.slot_max, g["final_slot_max"]).all()
    from paper_1809_11134_b200.gates import encode_gates

    bc, bt = encode_gates(eng.best_gates, eng.cfg.number_of_wires)
    assert list(bc) == list(g["best_codes"])
    np.testing.assert_allclose(bt, g["best_thetas"], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("mode", ["auto", "kernels", "graph", "fused"])
def test_batched_steps_equal_single_steps(mode):
    """steps(n) in every launch mode (CUDA graphs of 16 generations, one fused
    launch, ...) equals n single steps on the plain kernels, bit for bit."""
    g = golden("traj_qeqea_toffoli_c1")
    a = _engine_from_golden(g)
    b = _engine_from_golden(g)
    a.set_launch_mode("kernels")
    b.set_launch_mode(mode)
    ra = [a.step() for _ in range(40)]
    rb = b.steps(40)
    assert [x[0] for x in ra] == list(rb["gen_best"])
    assert [x[1] for x in ra] == list(rb["gen_mean"])
    assert np.array_equal(a.pop.thetas, b.pop.thetas)
    assert np.array_equal(a.table.slot_max, b.table.slot_max)
    assert [x.to_dict() for x in a.best_gates] == [x.to_dict() for x in b.best_gates]


def test_device_init_matches_oracle_init():
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import target_matrix

    cfg = PopulationConfig(number_of_wires=3, size_of_individual=8, size_of_population=7)
    eng = QeqeaEngine(cfg, target_matrix("Toffoli"), seed=11)
    pop = eng.pop
    from oracle.streams import init_slot

    for s in range(cfg.qubit_count):
        th, q = init_slot(11, s, s < cfg.qutrit_count)
        assert pop.thetas[s] == th  # uniform(0, 2pi): bit-exact
        if q is not None:
            np.testing.assert_allclose(pop.qutrits[s], q, rtol=0, atol=1e-14)


def test_oracle_trajectory_from_device_init():
    """Device init -> oracle replay over many generations (C1 shape)."""
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import target_matrix

    cfg = PopulationConfig(number_of_wires=3, size_of_individual=16, size_of_population=5,
                           max_generations=150)
    t = target_matrix("Toffoli")
    eng = QeqeaEngine(cfg, t, seed=21)
    pop = eng.pop
    lay = O.Layout(3, 16, 5, max_generations=150)
    ora = O.OracleQeqea(lay, t.matrix, 21, pop.thetas, pop.qutrits)
    dev = eng.steps(150)
    ref = [ora.step() for _ in range(150)]
    assert fit_close(dev["gen_best"], np.array([r[0] for r in ref])).all()
    assert fit_close(dev["gen_mean"], np.array([r[1] for r in ref])).all()
    assert fit_close(eng.best_fitness, ora.best_fitness)
    np.testing.assert_allclose(eng.pop.thetas, ora.thetas, rtol=1e-11, atol=1e-12)


def test_single_individual_population_consumes_no_individual_draws():
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import target_matrix

    cfg = PopulationConfig(number_of_wires=2, size_of_individual=3, size_of_population=1,
                           max_generations=30)
    t = target_matrix("CNOT")
    eng = QeqeaEngine(cfg, t, seed=4)
    pop = eng.pop
    ora = O.OracleQeqea(O.Layout(2, 3, 1, max_generations=30), t.matrix, 4, pop.thetas, pop.qutrits)
    for _ in range(30):
        flats, _, _ = eng.sample()
        gb, gm, tr = ora.step(trace=True)
        assert np.array_equal(flats, tr.blueprints)
        d = eng.step()
        assert fit_close(d[0], gb)


def test_pickle_round_trip_continues_identically():
    g = golden("traj_qeqea_cnot")
    a = _engine_from_golden(g)
    for _ in range(20):
        a.step()
    b = pickle.loads(pickle.dumps(a))
    ta = [a.step() for _ in range(20)]
    tb = [b.step() for _ in range(20)]
    assert ta == tb
    assert a.best_fitness == b.best_fitness
    assert a.best_gates == b.best_gates


def test_errors_and_echo():
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.errors import ConfigurationError
    from paper_1809_11134_b200.fitness import target_matrix

    cfg = PopulationConfig(number_of_wires=2, size_of_individual=3, size_of_population=4)
    with pytest.raises(ConfigurationError):
        QeqeaEngine(cfg, target_matrix("Toffoli"), seed=1)
    with pytest.raises(ConfigurationError):
        QeqeaEngine(cfg, target_matrix("CNOT"), seed=-1)
    with pytest.raises(ConfigurationError):
        PopulationConfig(number_of_wires=1, size_of_individual=3, size_of_population=4)
    with pytest.raises(ConfigurationError):
        PopulationConfig(number_of_wires=2, size_of_individual=3, size_of_population=4, n_meas=0)
    # nMeas > 60 reaches numpy's BTPE binomial branch, reproduced on the device
    big = QeqeaEngine(PopulationConfig(number_of_wires=2, size_of_individual=3, size_of_population=4,
                                       n_meas=1000), target_matrix("CNOT"), seed=1)
    assert big.steps(5).size == 5
    e = QeqeaEngine(cfg, target_matrix("CNOT"), seed=0, workers=2)
    echo = e.config_echo()
    assert echo["sizeOfIndividual"] == 3 and echo["workers"] == 2
    assert echo["probabilityOfMutation"] == pytest.approx(0.3)


def test_c4_shape_sample_and_fitness_against_oracle():
    """C4 (n=4, L=32, P=65536): device blueprints / codes / fitness of a sample
    of circuits match the oracle's sample_circuit + reference arithmetic."""
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import target_matrix

    P = 65536
    cfg = PopulationConfig(number_of_wires=4, size_of_individual=32, size_of_population=P,
                           max_generations=10)
    t = target_matrix("CCCNOT")
    eng = QeqeaEngine(cfg, t, seed=5)
    lay = O.Layout(4, 32, P)
    bests = []
    for gen in range(3):
        idx = np.array([0, 1, 777, 4097, P - 1])
        flats, codes, thetas = eng.sample()
        for c in idx:
            assert np.array_equal(flats[c], O.sample_blueprint(lay, 5, gen, int(c)))
        eng.step()
        fit = eng.last_fitness()
        assert np.all((fit >= 0) & (fit <= 1))
        ref = np.array([O.circuit_fitness(codes[c], thetas[c], t.matrix, 4) for c in idx])
        assert fit_close(fit[idx], ref).all()
        bests.append(eng.best_fitness)
    assert bests == sorted(bests)


def test_fp32_engine_first_generation_within_bound():
    """precision="fp32": same blueprints and gates as fp64 (they do not depend
    on fitness in generation 0), fitness within the stated fp32 bound."""
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    T = random_unitary(32, np.random.default_rng(9))
    cfg = PopulationConfig(number_of_wires=5, size_of_individual=64, size_of_population=4096,
                           target_fitness=1.0)
    a = QeqeaEngine(cfg, TargetSpec("haar", 5, T), seed=4)
    b = QeqeaEngine(cfg, TargetSpec("haar", 5, T), seed=4, precision="fp32")
    fa, ca, ta = a.sample()
    fb, cb, tb = b.sample()
    assert np.array_equal(fa, fb) and np.array_equal(ca, cb) and np.array_equal(ta, tb)
    a.step()
    b.step()
    x, y = a.last_fitness(), b.last_fitness()
    assert (np.abs(x - y) <= 1e-4 * np.abs(x) + 1e-6).all()
    assert not np.array_equal(x, y)
    b.steps(5)  # keeps running on the fp32 path
    assert b.generation == 6


def test_handles_release_their_device_memory():
    """Create / run / close engines repeatedly (QEQEA on the fused path, CUDA
    graphs and plain kernels; GA): device memory returns to where it started."""
    import torch

    from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

    t = target_matrix("Toffoli")

    def cycle():
        for P in (5, 4096, 1 << 16):
            e = QeqeaEngine(PopulationConfig(3, 16, P, max_generations=40), t, 1)
            e.steps(20)
            _ = e.best_gates
            e.close()
        g = GaEngine(GaConfig(3, 16, 50, max_generations=40), t, 1)
        g.steps(20)
        g.close()

    cycle()  # first use allocates the runtime's own pools
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(3):
        cycle()
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert abs(free1 - free0) < 64 << 20, (free0, free1)


@pytest.mark.parametrize("n_meas", [1, 3, 11, 61, 1000])
def test_device_measurement_matches_reference_goldens(n_meas):
    """construct_segments on the device (Born probabilities, multinomial by
    binomial inversion, argmax) against the reference's own measurements
    (measure.npz: engine.construct_segments per slot stream, generations 0
    and 9).  probability_of_mutation = 0 keeps the bank fixed across the
    generations, so every touched rotation slot's gate code carries the axis
    the reference measured for it."""
    from paper_1809_11134_b200.engine import PopulationConfig, PopulationState, QeqeaEngine
    from paper_1809_11134_b200.fitness import target_matrix

    g = golden("measure")
    q = g[f"nm{n_meas}_qutrits"]
    cfg = PopulationConfig(number_of_wires=3, size_of_individual=8, size_of_population=25, n_meas=n_meas,
                           probability_of_mutation=0.0)
    assert q.shape == (cfg.qutrit_count, 3)
    pop = PopulationState(np.zeros(cfg.qubit_count), q.copy())
    eng = QeqeaEngine(cfg, target_matrix("Toffoli"), seed=11, population=pop)
    checked = 0
    for gen in range(10):
        if gen in (0, 9):
            flats, codes, _ = eng.sample()
            rot = flats < cfg.qutrit_count
            assert np.array_equal(codes[rot] % 3, g[f"nm{n_meas}_g{gen}_axes"][flats[rot]]), gen
            checked += int(rot.sum())
        eng.step()
    assert checked > 100


def test_configuration_larger_than_the_device_is_refused_up_front():
    """A bank that cannot fit (n = 2, L = 4096, P = 300k: ≈262 GB with the
    per-touch arrays) is a ConfigurationError naming the sizes, raised before
    any allocation -- never a CPU fallback."""
    from paper_1809_11134_b200 import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.errors import ConfigurationError

    with pytest.raises(ConfigurationError, match="GB of device memory"):
        QeqeaEngine(PopulationConfig(2, 4096, 300_000), np.eye(4, dtype=np.complex128), 1)
