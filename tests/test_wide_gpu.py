"""numberOfWires 6..8 (the reference allows up to its 4^n <= 2^26 cap; the
tier's configurations are n = 3..5): the block-per-circuit kernel
(kernels_fitness.cu fitness_generic_kernel) against fixtures the reference
produced itself (oracle/gen_golden_wide.py)."""
import numpy as np
import pytest

from conftest import fit_close, golden

pytestmark = pytest.mark.gpu


def test_fitness_and_composition_match_reference_goldens():
    from paper_1809_11134_b200.fitness import compose_batch, fitness_batch

    g = golden("fitness_wide")
    keys = sorted({k.rsplit("_", 1)[0] for k in g.files})
    assert len(keys) >= 5
    for key in keys:
        n = int(key.split("_")[0][1:])
        codes, thetas, T = g[key + "_codes"], g[key + "_thetas"], g[key + "_target"]
        fit = fitness_batch(codes, thetas, T, n)
        assert fit_close(fit, g[key + "_fit"]).all(), (key, fit, g[key + "_fit"])
        if key + "_unitary" in g.files:
            np.testing.assert_allclose(compose_batch(codes, thetas, n), g[key + "_unitary"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", ["auto", "kernels", "graph"])
def test_qeqea_trajectory_n6_matches_reference(mode):
    from test_qeqea_gpu import _engine_from_golden

    g = golden("traj_qeqea_n6")
    eng = _engine_from_golden(g)
    eng.set_launch_mode(mode)
    if mode == "graph":  # batches of generations (graph mode is plain launches above 5 wires)
        b = _engine_from_golden(g)
        b.set_launch_mode(mode)
        rec = b.steps(int(g["gens"]))
        assert fit_close(rec["gen_best"], g["records"][:, 0]).all()
    gen = 0
    while not eng.done:
        flats, _, _ = eng.sample()
        assert np.array_equal(flats, g["blueprints"][gen])
        eng.step()
        assert fit_close(eng.last_fitness(), g["fitness"][gen]).all(), gen
        gen += 1
    assert gen == int(g["generations_run"])
    pop = eng.pop
    np.testing.assert_allclose(pop.thetas, g["final_thetas"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(pop.qutrits, g["final_qutrits"], rtol=0, atol=1e-11)
    assert fit_close(eng.table.slot_max, g["final_slot_max"]).all()


def test_fused_launch_is_refused_above_five_wires():
    from paper_1809_11134_b200.errors import ConfigurationError
    from test_qeqea_gpu import _engine_from_golden

    eng = _engine_from_golden(golden("traj_qeqea_n6"))
    eng.set_launch_mode("fused")
    with pytest.raises(ConfigurationError):
        eng.steps(1)


@pytest.mark.parametrize("mode", ["auto", "kernels"])
def test_ga_trajectory_n6_matches_reference(mode):
    from test_ga_gpu import _engine

    g = golden("traj_ga_n6")
    eng = _engine(g)
    eng.set_launch_mode(mode)
    codes, thetas = eng.genome_arrays()
    assert np.array_equal(codes, g["init_codes"])
    gen = 0
    while not eng.done:
        eng.step()
        assert fit_close(eng.last_fitness(), g["fitness"][gen]).all(), gen
        assert np.array_equal(eng.last_parents(), g["parents"][gen]), gen
        gen += 1
    codes, thetas = eng.genome_arrays()
    assert np.array_equal(codes, g["final_codes"])
    np.testing.assert_allclose(thetas, g["final_thetas"], rtol=1e-12, atol=1e-13)
