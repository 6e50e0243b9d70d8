"""The reference's functional API on the device (paper_1809_11134_b200.functional)
against the reference's own outputs (tests/golden, written by oracle/gen_golden.py
from isingsynth itself on the same counter streams) and the reference tests'
Generator-independent cases (pkg/tests/test_engine.py:45-208,
pkg/tests/test_ga.py:38-90)."""
import math

import numpy as np
import pytest

from conftest import fit_close, golden
from oracle import ga as OG
from oracle.streams import DOM_GA_MUT, DOM_GA_PAIR, init_slot, stream

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from paper_1809_11134_b200 import PopulationConfig

    base = dict(number_of_wires=2, size_of_individual=3, size_of_population=4)
    base.update(kw)
    return PopulationConfig(**base)


def test_generators_are_refused_with_an_explanation():
    from paper_1809_11134_b200 import sample_circuit

    with pytest.raises(TypeError, match="counter-based"):
        sample_circuit(_cfg(), np.random.default_rng(0))


def test_sample_circuit_matches_reference_goldens():
    from paper_1809_11134_b200 import CounterStreams, PopulationConfig
    from paper_1809_11134_b200.functional import sample_circuits

    g = golden("sampling")
    for key in g.files:
        n, L, P, s, gen = (int(t[1:]) for t in key.split("_"))
        cfg = PopulationConfig(number_of_wires=n, size_of_individual=L, size_of_population=P)
        bps = g[key]
        assert np.array_equal(sample_circuits(cfg, CounterStreams(s, gen, 0), bps.shape[0]), bps), key


def test_sample_circuit_equals_the_engines_blueprints():
    from paper_1809_11134_b200 import CounterStreams, QeqeaEngine, sample_circuit, target_matrix

    cfg = _cfg(number_of_wires=3, size_of_individual=16, size_of_population=300)
    eng = QeqeaEngine(cfg, target_matrix("Toffoli"), seed=4)
    eng.steps(2)
    flats, _, _ = eng.sample()
    for c in (0, 1, 151, 299):
        assert np.array_equal(sample_circuit(cfg, CounterStreams(4, 2, c)), flats[c])


def test_sample_circuit_bounds_and_positions():
    from paper_1809_11134_b200 import CounterStreams
    from paper_1809_11134_b200.functional import sample_circuits

    cfg = _cfg(size_of_individual=7)
    bps = sample_circuits(cfg, CounterStreams(1, 0, 0), 100)
    assert bps.shape == (100, 7)
    for bp in bps:
        assert [cfg.decode_flat(int(f))[2] for f in bp] == list(range(7))
        assert all(0 <= f < cfg.qubit_count for f in bp)


@pytest.mark.parametrize("n_meas", [1, 3, 11, 61, 100, 1000])
def test_construct_segments_matches_reference_goldens(n_meas):
    from paper_1809_11134_b200 import CounterStreams, PopulationConfig, PopulationState, construct_segments
    from paper_1809_11134_b200.gates import enumerate_templates

    g = golden("measure")
    cfg = PopulationConfig(number_of_wires=3, size_of_individual=8, size_of_population=25, n_meas=n_meas)
    q = g[f"nm{n_meas}_qutrits"]
    pop = PopulationState(np.zeros(cfg.qubit_count), q)
    for gen in (0, 9):
        bank = construct_segments(pop, cfg, enumerate_templates(3), CounterStreams(11, gen))
        assert np.array_equal(bank.axes, g[f"nm{n_meas}_g{gen}_axes"]), gen


def test_construct_segments_respects_born_weights():
    from paper_1809_11134_b200 import CounterStreams, construct_segments, init_population
    from paper_1809_11134_b200.gates import Axis, enumerate_templates

    cfg = _cfg(size_of_individual=50, size_of_population=10, n_meas=11)
    pop = init_population(cfg, CounterStreams(3))
    pop.qutrits[:] = 0.0
    pop.qutrits[:, 2] = 1.0  # every selector pinned to Z
    bank = construct_segments(pop, cfg, enumerate_templates(2), CounterStreams(3, 5))
    assert np.all(bank.axes == Axis.Z)


def test_init_population_matches_the_init_streams():
    from paper_1809_11134_b200 import CounterStreams, init_population

    cfg = _cfg(number_of_wires=3, size_of_individual=5, size_of_population=6)
    pop = init_population(cfg, CounterStreams(11))
    assert pop.thetas.shape == (cfg.qubit_count,) and pop.qutrits.shape == (cfg.qutrit_count, 3)
    assert np.all((pop.thetas >= 0) & (pop.thetas < 2 * math.pi))
    np.testing.assert_allclose(np.linalg.norm(pop.qutrits, axis=1), 1.0, atol=1e-12)
    for s in range(cfg.qubit_count):
        th, q = init_slot(11, s, s < cfg.qutrit_count)
        assert pop.thetas[s] == th
        if q is not None:
            np.testing.assert_allclose(pop.qutrits[s], q, rtol=0, atol=1e-14)


def test_segment_bank_descriptors():
    from paper_1809_11134_b200 import CounterStreams, construct_segments, init_population
    from paper_1809_11134_b200.gates import enumerate_templates

    cfg = _cfg()
    pop = init_population(cfg, CounterStreams(2))
    bank = construct_segments(pop, cfg, enumerate_templates(2), CounterStreams(2, 0))
    op = bank.descriptor(cfg.flat_index(1, 2, 0))
    assert op.kind == "rotation" and op.wire == 2 and op.theta == pop.thetas[cfg.flat_index(1, 2, 0)]
    op = bank.descriptor(cfg.flat_index(2, 0, 1))
    assert op.kind == "interaction" and op.pair == (1, 2)
    for flat in (cfg.flat_index(1, 2, 0), cfg.flat_index(2, 0, 1)):
        u = bank.unitary(flat)
        np.testing.assert_allclose(u.conj().T @ u, np.eye(4), atol=1e-12)


def test_evaluate_circuit_matches_compose_and_the_fitness_goldens():
    from paper_1809_11134_b200 import (CounterStreams, compose_gates, construct_segments, evaluate_circuit,
                                       fitness_value, init_population, target_matrix)
    from paper_1809_11134_b200.functional import evaluate_circuits, sample_circuits
    from paper_1809_11134_b200.gates import enumerate_templates

    cfg = _cfg()
    pop = init_population(cfg, CounterStreams(5))
    bank = construct_segments(pop, cfg, enumerate_templates(2), CounterStreams(5, 0))
    t = target_matrix("CNOT").matrix
    bps = sample_circuits(cfg, CounterStreams(5, 0, 0), 20)
    batch = evaluate_circuits(bps, bank, t)
    for bp, f in zip(bps, batch):
        u = compose_gates([bank.descriptor(int(x)) for x in bp], 2)
        assert evaluate_circuit(bp, bank, t) == f
        assert f == pytest.approx(fitness_value(u, t), abs=1e-12)


def test_segment_table_keeps_best():
    """pkg/tests/test_engine.py:159-171, verbatim semantics."""
    from paper_1809_11134_b200 import SegmentFitnessTable

    table = SegmentFitnessTable(_cfg())
    bp = np.array([0, 5, 10])
    assert table.update(bp, 0.4) == {0, 5, 10}
    assert table.update(bp, 0.3) == set()  # lower score never overwrites
    assert table.entries[(5, 1)] == 0.4
    assert table.update(np.array([1, 5, 10]), 0.6) == {1, 5, 10}
    assert table.entries[(5, 1)] == 0.6
    assert table.slot_max[5] == 0.6
    assert (0, 1) not in table.entries  # same slot at another position is a separate entry


def test_segment_table_batches_match_the_sequential_reference_rule():
    """update_batch over many circuits == the reference's per-circuit loop
    (engine.py:211-222), restated here on a dict."""
    from paper_1809_11134_b200 import SegmentFitnessTable

    cfg = _cfg(number_of_wires=3, size_of_individual=5, size_of_population=7)
    rng = np.random.default_rng(8)
    table = SegmentFitnessTable(cfg)
    entries, slot_max = {}, np.zeros(cfg.qubit_count)
    for _ in range(6):
        bps = rng.integers(0, cfg.qubit_count, size=(40, cfg.size_of_individual))
        fits = np.round(rng.uniform(0, 1, size=40), 2)  # ties included
        want = set()
        for bp, fit in zip(bps, fits):
            for pos, flat in enumerate(bp):
                key = (int(flat), pos)
                if fit > entries.get(key, 0.0):
                    entries[key] = fit
                    want.add(int(flat))
                slot_max[flat] = max(slot_max[flat], fit)
        assert table.update_batch(bps, fits) == want
        assert np.array_equal(table.slot_max, slot_max)
        assert table.entries == entries


def test_mutate_population_matches_reference_goldens():
    from paper_1809_11134_b200 import (CounterStreams, PopulationConfig, PopulationState, SegmentFitnessTable,
                                       mutate_population)

    g = golden("mutate")
    cfg = PopulationConfig(number_of_wires=3, size_of_individual=16, size_of_population=8,
                           probability_of_mutation=0.5)
    table = SegmentFitnessTable(cfg)
    table.slot_max[:] = g["slot_max"]
    for gen in (0, 4):
        pop = PopulationState(g["thetas0"].copy(), g["qutrits0"].copy())
        snaps = mutate_population(pop, table, cfg, CounterStreams(3, gen))
        mutated = np.zeros(cfg.qubit_count, dtype=bool)
        mutated[list(snaps)] = True
        assert np.array_equal(mutated, g[f"g{gen}_mutated"])
        assert np.array_equal(pop.thetas, g[f"g{gen}_thetas"])  # angle path bit-exact
        np.testing.assert_allclose(pop.qutrits, g[f"g{gen}_qutrits"], rtol=0, atol=1e-15)


def test_mutation_snapshots_and_revert():
    """pkg/tests/test_engine.py:174-197."""
    from paper_1809_11134_b200 import CounterStreams, SegmentFitnessTable, init_population, mutate_population

    cfg = _cfg(probability_of_mutation=1.0)
    pop = init_population(cfg, CounterStreams(6))
    table = SegmentFitnessTable(cfg)
    before, before_q = pop.thetas.copy(), pop.qutrits.copy()
    snapshots = mutate_population(pop, table, cfg, CounterStreams(6, 0))
    assert set(snapshots) == set(range(cfg.qubit_count))
    assert np.nonzero(~np.isclose(pop.thetas, before))[0].size > 0
    for flat, (theta, qutrit) in snapshots.items():
        assert theta == before[flat]
        if flat < cfg.qutrit_count:
            assert np.array_equal(qutrit, before_q[flat])
        else:
            assert qutrit is None
    for flat, (theta, qutrit) in snapshots.items():
        pop.thetas[flat] = theta
        if qutrit is not None:
            pop.qutrits[flat] = qutrit
    assert np.array_equal(pop.thetas, before) and np.array_equal(pop.qutrits, before_q)


def test_mutation_skips_perfect_slots():
    """pkg/tests/test_engine.py:200-208."""
    from paper_1809_11134_b200 import CounterStreams, SegmentFitnessTable, init_population, mutate_population

    cfg = _cfg(probability_of_mutation=1.0)
    pop = init_population(cfg, CounterStreams(7))
    table = SegmentFitnessTable(cfg)
    table.slot_max[:] = 1.0
    before = pop.thetas.copy()
    assert mutate_population(pop, table, cfg, CounterStreams(7, 0)) == {}
    assert np.array_equal(pop.thetas, before)


@pytest.mark.parametrize("name", ["cnot", "toffoli_c2", "p300"])
def test_ga_operators_match_reference_goldens(name):
    """random_genome = the reference's initial genomes, sus_select = the
    reference's parents for the reference's fitness, every generation."""
    from paper_1809_11134_b200 import CounterStreams, GaConfig, random_genome, sus_select
    from paper_1809_11134_b200.gates import encode_gates

    g = golden(f"traj_ga_{name}")
    n, L, P, seed = int(g["n"]), int(g["L"]), int(g["P"]), int(g["seed"])
    cfg = GaConfig(number_of_wires=n, size_of_individual=L, population=P)
    for i in (0, 1, P - 1):
        codes, thetas = encode_gates(random_genome(cfg, CounterStreams(seed, index=i)), n)
        assert np.array_equal(codes, g["init_codes"][i]) and np.array_equal(thetas, g["init_thetas"][i])
    for gen in range(int(g["generations_run"])):
        assert sus_select(list(g["fitness"][gen]), P, CounterStreams(seed, gen)) == list(g["parents"][gen])


def test_sus_select_at_large_populations_matches_reference():
    """The block SUS (sus.cuh: pairwise total by subtrees, the two running sums
    on staged tiles, the picks by binary search) against the reference's own
    picks, P = 600 .. 300k, count = P / about P/2 / 2P, with zeros and ties
    (oracle/gen_golden_sus.py)."""
    import hashlib

    from oracle.targets import sus_fitness
    from paper_1809_11134_b200 import CounterStreams, sus_select

    g = golden("sus_large")
    names = sorted({k.rsplit("_", 1)[0] for k in g.files})
    for name in names:
        P, count, seed, gen = (int(x) for x in g[name + "_meta"])
        f = sus_fitness(P, seed, str(g[name + "_kind"]))
        picks = np.asarray(sus_select(f, count, CounterStreams(seed, gen)), dtype=np.int64)
        assert np.array_equal(picks[:64], g[name + "_head"]) and np.array_equal(picks[-64:], g[name + "_tail"]), name
        assert hashlib.sha256(picks.astype("<i8").tobytes()).hexdigest() == str(g[name + "_sha"]), name


@pytest.mark.parametrize("P,count,kind", [(1, 1, "one"), (1, 7, "one"), (2, 5, "u"), (3, 1, "u"), (700, 700, "zero"),
                                           (9000, 3, "u"), (5, 9000, "u"), (4096, 4096, "spike"), (900, 900, "neg")])
def test_sus_select_edge_shapes_match_the_walk(P, count, kind):
    """Single values, more pointers than values and the reverse, all-zero
    fitness at a size above the shared-memory walk, one dominant value, and
    negative values (non-monotone sums: the walk itself runs)."""
    from oracle.ga import sus_select as walk
    from oracle.streams import DOM_GA_SUS
    from paper_1809_11134_b200 import CounterStreams, sus_select

    r = np.random.default_rng(P + count)
    f = {"one": np.array([0.3] * P), "u": r.random(P), "zero": np.zeros(P),
         "spike": np.where(np.arange(P) == P // 3, 1.0, 1e-9 * r.random(P)),
         "neg": r.random(P) - 0.2}[kind]  # not a fitness, but the reference's walk accepts it
    want = walk(list(map(float, f)), count, stream(8, DOM_GA_SUS, 2))
    assert sus_select(f, count, CounterStreams(8, 2)) == want


@pytest.mark.parametrize("kind", ["zero_prefix", "dyadic", "spikes", "wide", "tiny"])
def test_sus_select_grid_wide_sums_match_the_walk(kind):
    """From P - 1 = 2^17 values the running sums and numpy's total run over
    the whole GPU (sus.cuh launch_exact_chain_grid / launch_pairwise_parts):
    tiles advanced by their composite map where the binade provably holds,
    the rest (binade crossings, a zero or subnormal-range running sum) by
    the exact block form.  Families that exercise each branch."""
    from oracle.ga import sus_select as walk
    from oracle.streams import DOM_GA_SUS
    from paper_1809_11134_b200 import CounterStreams, sus_select

    P = (1 << 17) + 3 * 8192 + 5
    r = np.random.default_rng(42)
    u = r.random(P)
    f = {"zero_prefix": np.where(np.arange(P) < P // 2, 0.0, u),
         "dyadic": np.floor(u * 64) / 64,
         "spikes": np.where(u < 0.3, 0.0, np.where(u > 0.9999, 1e6 * u, u)),
         "wide": np.ldexp(u, (np.arange(P) % 40) - 20),
         "tiny": 1e-310 * u}[kind]
    want = walk(list(map(float, f)), P, stream(9, DOM_GA_SUS, 4))
    assert sus_select(f, P, CounterStreams(9, 4)) == want


def test_sus_all_zero_falls_back_to_uniform_draws():
    from paper_1809_11134_b200 import CounterStreams, sus_select

    picks = sus_select([0.0] * 9, 9, CounterStreams(3, 1))
    want = [int(x) for x in (lambda s: [s.integers(9) for _ in range(9)])(stream(3, 6, 1))]
    assert picks == want


def test_crossover_and_mutation_match_the_streams():
    from paper_1809_11134_b200 import CounterStreams, GaConfig, ga_mutate, random_genome, two_point_crossover
    from paper_1809_11134_b200.gates import encode_gates

    cfg = GaConfig(number_of_wires=3, size_of_individual=16, mutation_rate=0.5, structural_rate=0.4)
    lay = OG.GaLayout(3, 16, 50, rate=0.5, structural=0.4)
    a = random_genome(cfg, CounterStreams(1, index=0))
    b = random_genome(cfg, CounterStreams(1, index=1))
    for k in range(20):
        ca, cb = two_point_crossover(a, b, CounterStreams(1, 3, k))
        p, q = OG.crossover_cuts(16, stream(1, DOM_GA_PAIR, 3, k))
        assert ca == a[:p] + b[p:q] + a[q:] and cb == b[:p] + a[p:q] + b[q:]
    for i in range(10):
        m = ga_mutate(a, cfg, CounterStreams(1, 2, i))
        codes, thetas = encode_gates(list(a), 3)
        mc, mt = encode_gates(list(m), 3)
        for j in range(16):
            wc, wt = OG.mutate_gene(int(codes[j]), float(thetas[j]), lay, stream(1, DOM_GA_MUT, 2, i, j))
            assert mc[j] == wc and mt[j] == wt
    short = random_genome(GaConfig(number_of_wires=2, size_of_individual=1), CounterStreams(0))
    assert two_point_crossover(short, short, CounterStreams(0, 0, 0)) == (short, short)


def test_decode_genome_is_shared_composition():
    from paper_1809_11134_b200 import CounterStreams, GaConfig, compose_gates, decode_genome, random_genome

    cfg = GaConfig(number_of_wires=2, size_of_individual=5)
    g = random_genome(cfg, CounterStreams(4))
    u = decode_genome(g, 2)
    assert np.array_equal(u, compose_gates(list(g), 2))
    np.testing.assert_allclose(u.conj().T @ u, np.eye(4), atol=1e-12)


def test_module_level_names_resolve_like_the_reference():
    from paper_1809_11134_b200.engine import (SegmentFitnessTable, construct_segments, evaluate_circuit,
                                              init_population, mutate_population, sample_circuit)
    from paper_1809_11134_b200.ga import decode_genome, ga_mutate, random_genome, sus_select, two_point_crossover

    assert all(callable(f) for f in (SegmentFitnessTable, construct_segments, evaluate_circuit, init_population,
                                     mutate_population, sample_circuit, decode_genome, ga_mutate, random_genome,
                                     sus_select, two_point_crossover))


def test_apply_gate_expand_rotation_interaction_gate_match_the_reference_definitions():
    """gates.py:96-116,173-184: dense Kronecker expansion / diagonal, left
    multiplication of an arbitrary accumulator (pkg/tests/test_gates.py:112-132)."""
    from paper_1809_11134_b200.gates import (Axis, GateOp, apply_gate, apply_gates, compose_gates,
                                             enumerate_templates, expand_rotation, interaction_gate,
                                             interaction_diagonal, rotation_gate)

    rng = np.random.default_rng(4)
    for n in (2, 3, 5, 6):
        d = 2 ** n
        acc = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
        for wire in (1, n):
            for axis in Axis:
                th = float(rng.uniform(0, 2 * math.pi))
                left, right = 2 ** (wire - 1), 2 ** (n - wire)
                dense = np.kron(np.kron(np.eye(left), rotation_gate(axis, th)), np.eye(right))
                np.testing.assert_allclose(expand_rotation(axis, th, wire, n), dense, atol=1e-14)
                g = GateOp(kind="rotation", theta=th, wire=wire, axis=axis)
                np.testing.assert_allclose(apply_gate(acc, g, n), dense @ acc, atol=1e-12)
        tpl = enumerate_templates(n)[-1]
        th = float(rng.uniform(0, 2 * math.pi))
        np.testing.assert_allclose(interaction_gate(tpl, th), np.diag(interaction_diagonal(tpl, th)), atol=1e-14)
        gates = [GateOp(kind="rotation", theta=0.3, wire=1, axis=Axis.Y),
                 GateOp(kind="interaction", theta=1.1, pair=tpl.pair)]
        np.testing.assert_allclose(apply_gates(np.eye(d), gates, n), compose_gates(gates, n), atol=1e-13)


def test_target_is_valid():
    from paper_1809_11134_b200.fitness import TargetSpec, target_is_valid, target_matrix

    assert target_is_valid(target_matrix("Toffoli"))
    assert not target_is_valid(TargetSpec("bad", 1, np.array([[1, 0], [0, 2]], dtype=complex)))
