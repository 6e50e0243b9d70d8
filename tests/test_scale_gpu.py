"""Generation-level parity at the scale the product runs (many blocks,
colliding touches), against fixtures the reference produced itself
(oracle/gen_golden_scale.py: the reference's sample_circuit,
construct_segments, evaluate_circuit, SegmentFitnessTable.update, elitist
revert and mutate_angle / mutate_qutrit on the per-unit Philox streams).

Per generation: blueprints (SHA-256, bit-exact), every circuit's fitness
(fp64 bound), the improved set (engine.py:202-222; here the slots whose
slot_max rose, SHA-256 bit-exact), and the live bank after the generation
(engine.pop: committed values with the new pending mutations applied,
engine.py:345-352 + 228-263) through 256 range sums of theta / qutrit
components / slot_max and the exact values of a seeded slot sample (half of
it improved slots).  Run in the plain-kernel and CUDA-graph launch modes.
"""
import hashlib

import numpy as np
import pytest

from conftest import fit_close, golden

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def _bucket_sums(x, buckets):
    n = x.shape[0]
    edges = (np.arange(buckets + 1) * n) // buckets
    c = np.concatenate([np.zeros((1,) + x.shape[1:]), np.cumsum(x, axis=0)])
    return c[edges[1:]] - c[edges[:-1]]


@pytest.mark.parametrize("name", ["n4", "n5", "c4"])
@pytest.mark.parametrize("mode", ["kernels", "graph"])
def test_multiblock_generations_match_reference(name, mode):
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec
    from paper_1809_11134_b200.gates import encode_gates

    g = golden(f"traj_scale_{name}")
    cfg = PopulationConfig(
        number_of_wires=int(g["n"]), size_of_individual=int(g["L"]), size_of_population=int(g["P"]),
        probability_of_mutation=float(g["p_mut"]), mutation_range=float(g["mutation_range"]),
        n_meas=int(g["n_meas"]), max_generations=int(g["gens"]), target_fitness=float(g["target_fitness"]))
    eng = QeqeaEngine(cfg, TargetSpec("golden", cfg.number_of_wires, g["target"]), int(g["seed"]))
    eng.set_launch_mode(mode)
    B = int(g["buckets"])
    Qt = cfg.qutrit_count
    assert int(g["colliding_slots"].min()) > 100  # the fixture does exercise collisions
    gen = 0
    while not eng.done:
        flats, _, _ = eng.sample()
        assert _sha(flats) == str(g["blueprint_sha"][gen]), f"blueprints differ at generation {gen}"
        before = eng.table.slot_max
        gb, gm = eng.step()
        fit = eng.last_fitness()
        if "fitness_idx" in g:
            fit = fit[g["fitness_idx"]]
        ok = fit_close(fit, g["fitness"][gen])
        assert ok.all(), (gen, int((~ok).sum()), fit[~ok][:5], g["fitness"][gen][~ok][:5])
        assert fit_close([gb, gm, eng.best_fitness], g["records"][gen]).all()
        after = eng.table.slot_max
        improved = np.flatnonzero(after > before)
        assert improved.size == int(g["improved_count"][gen]), (gen, improved.size, int(g["improved_count"][gen]))
        assert _sha(improved) == str(g["improved_sha"][gen]), gen
        pop = eng.pop
        np.testing.assert_allclose(_bucket_sums(pop.thetas, B), g["theta_sums"][gen], rtol=0, atol=1e-7)
        np.testing.assert_allclose(_bucket_sums(pop.qutrits.real, B), g["qre_sums"][gen], rtol=0, atol=1e-7)
        np.testing.assert_allclose(_bucket_sums(pop.qutrits.imag, B), g["qim_sums"][gen], rtol=0, atol=1e-7)
        np.testing.assert_allclose(_bucket_sums(after, B), g["slot_max_sums"][gen], rtol=0, atol=1e-7)
        idx = g["sample_idx"][gen]
        s = idx >= 0
        np.testing.assert_allclose(pop.thetas[idx[s]], g["sample_thetas"][gen][s], rtol=1e-11, atol=1e-12)
        assert fit_close(after[idx[s]], g["sample_slot_max"][gen][s]).all()
        rot = s & (idx < Qt)
        np.testing.assert_allclose(pop.qutrits[idx[rot]], g["sample_qutrits"][gen][rot], rtol=0, atol=1e-11)
        gen += 1
    assert gen == int(g["generations_run"])
    assert eng.stop_reason == str(g["stop_reason"])
    bc, bt = encode_gates(eng.best_gates, cfg.number_of_wires)
    assert list(bc) == list(g["best_codes"])
    np.testing.assert_allclose(bt, g["best_thetas"], rtol=1e-11, atol=1e-12)


def test_c5_run_invariants():
    """BASELINE config 5 (n = 5, L = 64, P = 2^20, 36 GB bank) for 40
    generations through the engine's batched steps: the records are
    consistent (best-so-far = running max of the generation bests, fitness
    values in [0, 1], mean <= best), `steps(k)` and the stop rule agree, and
    circuits of generation 25 sampled on their own (`sample`, the gates the
    generation evaluates) and rescored with fitness_batch give the fitness
    the generation recorded."""
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec, fitness_batch
    from paper_1809_11134_b200.synthetic import haar_target

    n, L, P, gens = 5, 64, 1 << 20, 40
    T = haar_target(n)
    eng = QeqeaEngine(PopulationConfig(n, L, P, max_generations=gens, target_fitness=1.0),
                      TargetSpec("haar", n, T), 7)
    rec = eng.steps(25)
    c0 = P // 3
    _, codes, thetas = eng.sample(c0, c0 + 48)
    gb, gm = eng.step()
    again = fitness_batch(codes, thetas, T, n)
    assert fit_close(again, eng.last_fitness()[c0:c0 + 48]).all()
    rec2 = eng.steps(100)  # stops at the generation limit
    assert len(rec) == 25 and len(rec2) == gens - 26
    assert eng.done and eng.stop_reason == "generation-limit" and eng.generation == gens
    best = np.concatenate([rec["gen_best"], [gb], rec2["gen_best"]])
    mean = np.concatenate([rec["gen_mean"], [gm], rec2["gen_mean"]])
    bsf = np.concatenate([rec["best_fitness"], [max(rec["best_fitness"][-1], gb)], rec2["best_fitness"]])
    assert np.all((best >= 0) & (best <= 1)) and np.all(mean <= best) and np.all(mean >= 0)
    assert np.array_equal(bsf, np.maximum.accumulate(best))
    assert eng.best_fitness == bsf[-1]
    fit = eng.last_fitness()
    assert fit.shape == (P,) and fit.max() == best[-1]
    eng.close()
