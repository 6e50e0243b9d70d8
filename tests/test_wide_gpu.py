"""numberOfWires 6..13 (13 is the reference's default 4^n <= 2^26 cap; the
tier's configurations are n = 3..5): the block-per-circuit kernel
(kernels_fitness.cu fitness_generic_kernel) against fixtures the reference
produced itself (oracle/gen_golden_wide.py for n = 6..8,
oracle/gen_golden_xwide.py for n = 9..13, whose targets are rebuilt from a
seed by oracle/targets.py: 1 GB at n = 13)."""
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


def _wide_golden(name):
    """A trajectory fixture with its target (rebuilt when only the seed is stored)."""
    from oracle.targets import product_target

    g = dict(golden(name))
    if "target" not in g:
        g["target"] = product_target(int(g["n"]), int(g["target_seed"]))
    return g


def test_fitness_up_to_the_reference_cap_matches_reference_goldens():
    """n = 9..13 (one resident matrix 4 MB .. 1 GB; the launch bounds its
    scratch by the free memory)."""
    from oracle.targets import product_target
    from paper_1809_11134_b200.fitness import fitness_batch

    g = golden("fitness_xwide")
    keys = sorted({k.split("_")[0] + "_" + k.split("_")[1] for k in g.files})
    assert sorted(int(k.split("_")[0][1:]) for k in keys) == [9, 10, 11, 12, 13]
    for key in keys:
        n = int(key.split("_")[0][1:])
        T = product_target(n, int(g[key + "_target_seed"]))
        fit = fitness_batch(g[key + "_codes"], g[key + "_thetas"], T, n)
        assert fit_close(fit, g[key + "_fit"]).all(), (key, fit, g[key + "_fit"])


@pytest.mark.parametrize("name,mode", [("n6", "auto"), ("n6", "kernels"), ("n6", "graph"), ("n11", "auto")])
def test_qeqea_trajectory_wide_matches_reference(name, mode):
    from test_qeqea_gpu import _engine_from_golden

    g = _wide_golden(f"traj_qeqea_{name}")
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


@pytest.mark.parametrize("name,mode", [("n6", "auto"), ("n6", "kernels"), ("n11", "auto")])
def test_ga_trajectory_wide_matches_reference(name, mode):
    from test_ga_gpu import _engine

    g = _wide_golden(f"traj_ga_{name}")
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
