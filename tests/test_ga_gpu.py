"""GA engine parity on the device (GaEngine, ga.py:141-214) against the
fixtures the reference produced with the same Philox streams
(oracle/gen_golden.py PhiloxGaEngine): initial genomes and SUS parents
bit-exact, fitness / records within the fp64 tolerance, final genomes and best
circuit."""
import pickle

import numpy as np
import pytest

from conftest import fit_close, golden
from oracle import ga as OG

pytestmark = pytest.mark.gpu


def _engine(g):
    from paper_1809_11134_b200.fitness import TargetSpec
    from paper_1809_11134_b200.ga import GaConfig, GaEngine

    cfg = GaConfig(number_of_wires=int(g["n"]), size_of_individual=int(g["L"]), population=int(g["P"]),
                   mutation_rate=float(g["rate"]), mutation_range=float(g["mrange"]),
                   structural_rate=float(g["structural"]), max_generations=int(g["gens"]),
                   target_fitness=float(g["target_fitness"]))
    return GaEngine(cfg, TargetSpec("golden", cfg.number_of_wires, g["target"]), int(g["seed"]))


@pytest.mark.parametrize("name", ["cnot", "toffoli_c2", "odd13", "p300", "p1024", "l1", "long", "n4", "n5"])
@pytest.mark.parametrize("mode", ["auto", "kernels", "fused"])
def test_ga_trajectory_matches_reference(name, mode):
    g = golden(f"traj_ga_{name}")
    eng = _engine(g)
    eng.set_launch_mode(mode)
    codes, thetas = eng.genome_arrays()
    assert np.array_equal(codes, g["init_codes"])
    assert np.array_equal(thetas, g["init_thetas"])
    gen = 0
    recs = []
    while not eng.done:
        gb, gm = eng.step()
        recs.append((gb, gm, eng.best_fitness))
        assert fit_close(eng.last_fitness(), g["fitness"][gen]).all(), gen
        assert np.array_equal(eng.last_parents(), g["parents"][gen]), gen
        gen += 1
    assert gen == int(g["generations_run"])
    assert eng.stop_reason == str(g["stop_reason"])
    assert fit_close(np.array(recs), g["records"]).all()
    codes, thetas = eng.genome_arrays()
    assert np.array_equal(codes, g["final_codes"])
    np.testing.assert_allclose(thetas, g["final_thetas"], rtol=1e-12, atol=1e-13)
    from paper_1809_11134_b200.gates import encode_gates

    bc, bt = encode_gates(eng.best_gates, eng.cfg.number_of_wires)
    assert list(bc) == list(g["best_codes"])


def test_ga_against_oracle_long_run():
    from paper_1809_11134_b200.fitness import target_matrix
    from paper_1809_11134_b200.ga import GaConfig, GaEngine

    cfg = GaConfig(number_of_wires=3, size_of_individual=16, population=50, max_generations=120)
    t = target_matrix("Toffoli")
    eng = GaEngine(cfg, t, seed=31)
    ora = OG.OracleGa(OG.GaLayout(3, 16, 50, max_generations=120), t.matrix, 31)
    dev = eng.steps(120)
    ref = [ora.step() for _ in range(120)]
    assert fit_close(dev["gen_best"], np.array([r[0] for r in ref])).all()
    assert fit_close(dev["gen_mean"], np.array([r[1] for r in ref])).all()
    codes, _ = eng.genome_arrays()
    assert np.array_equal(codes, ora.codes)


def test_ga_pickle_round_trip():
    from paper_1809_11134_b200.fitness import target_matrix
    from paper_1809_11134_b200.ga import GaConfig, GaEngine

    cfg = GaConfig(number_of_wires=2, size_of_individual=5, population=10, max_generations=100)
    a = GaEngine(cfg, target_matrix("CNOT"), seed=2)
    for _ in range(30):
        a.step()
    b = pickle.loads(pickle.dumps(a))
    assert [a.step() for _ in range(30)] == [b.step() for _ in range(30)]
    assert a.best_gates == b.best_gates


def test_ga_population_and_elitism():
    from paper_1809_11134_b200.fitness import target_matrix
    from paper_1809_11134_b200.ga import GaConfig, GaEngine

    cfg = GaConfig(number_of_wires=2, size_of_individual=5, population=13, max_generations=60)
    eng = GaEngine(cfg, target_matrix("CNOT"), seed=6)
    bests = []
    while not eng.done:
        gb, gm = eng.step()
        assert 0.0 <= gm <= gb <= 1.0
        bests.append(gb)
        assert len(eng.genomes) == 13
    assert all(b >= a - 1e-12 for a, b in zip(bests, bests[1:]))
    assert eng.stop_reason == "generation-limit"
    assert len(eng.gate_choices if hasattr(eng, "gate_choices") else cfg.gate_choices) == 7


@pytest.mark.parametrize("mode", ["auto", "kernels", "graph", "fused"])
def test_ga_batched_steps_equal_single_steps(mode):
    g = golden("traj_ga_toffoli_c2")
    a, b = _engine(g), _engine(g)
    a.set_launch_mode("kernels")
    b.set_launch_mode(mode)
    ra = [a.step() for _ in range(int(g["gens"]))]
    rb = b.steps(int(g["gens"]))
    assert [x[0] for x in ra] == list(rb["gen_best"])
    assert [x[1] for x in ra] == list(rb["gen_mean"])
    ca, ta = a.genome_arrays()
    cb, tb = b.genome_arrays()
    assert np.array_equal(ca, cb) and np.array_equal(ta, tb)


@pytest.mark.parametrize("mode", ["graph", "auto"])
def test_large_population_graph_modes_equal_plain_kernels(mode):
    """The grid-wide SUS (P - 1 >= 2^17: tile sums, maps, serial carry, apply,
    pairwise parts) captured into the generation graphs gives the plain
    launches' parents and genomes."""
    from paper_1809_11134_b200 import GaConfig, GaEngine, target_matrix

    P = (1 << 17) + 2
    a = GaEngine(GaConfig(2, 4, P, max_generations=100, target_fitness=1.0), target_matrix("CNOT"), 6)
    b = GaEngine(GaConfig(2, 4, P, max_generations=100, target_fitness=1.0), target_matrix("CNOT"), 6)
    a.set_launch_mode("kernels")
    b.set_launch_mode(mode)
    ra = [a.step() for _ in range(4)]
    rb = b.steps(4)
    assert [x[0] for x in ra] == list(rb["gen_best"]) and [x[1] for x in ra] == list(rb["gen_mean"])
    assert np.array_equal(a.last_parents(), b.last_parents())
    ca, ta = a.genome_arrays()
    cb, tb = b.genome_arrays()
    assert np.array_equal(ca, cb) and np.array_equal(ta, tb)


@pytest.mark.parametrize("P", [513, 1 << 17, (1 << 17) + 1, (1 << 17) + 2, 1 << 20])
def test_large_population_parents_match_the_oracle_walk(P):
    """P > 512 selects on the block SUS + search kernels (kernels_ga.cu
    ga_reduce_sus_large_kernel; from P - 1 = 2^17 the running sums and the
    total are grid-wide, sus.cuh launch_exact_chain_grid); its parents must be the sequential walk's
    (oracle/ga.sus_select, pinned to the reference by tests/golden/sus_large)
    on the engine's own fitness, generation by generation."""
    from oracle.ga import sus_select
    from oracle.streams import DOM_GA_SUS, stream
    from paper_1809_11134_b200 import GaConfig, GaEngine, target_matrix

    eng = GaEngine(GaConfig(2, 4, P, max_generations=100, target_fitness=1.0), target_matrix("CNOT"), 5)
    eng.set_launch_mode("kernels")
    for gen in range(3):
        eng.step()
        fit = eng.last_fitness()
        want = sus_select(list(map(float, fit)), P, stream(5, DOM_GA_SUS, gen))
        assert np.array_equal(eng.last_parents(), np.asarray(want)), gen
