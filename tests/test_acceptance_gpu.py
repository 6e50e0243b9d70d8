"""The reference's acceptance criteria on the device engines
(pkg/tests/test_acceptance.py criteria 1-3; recorded outcomes in
pkg/test_output.txt:12-18).  Counter-based streams make the individual runs
differ from the reference's PCG64 runs; the outcomes must not."""
import math
import statistics

import pytest

pytestmark = pytest.mark.gpu

SEEDS = (1, 2, 3, 4, 5)
CNOT_L3_CAP = 1 - math.sqrt(1 - math.sqrt(2) / 2)  # 0.4588..., test_output.txt:12


def _run(engine):
    while not engine.done:
        engine.steps(4096)
    return engine.best_fitness, engine.generation


def test_criterion_1_qeqea_cnot_reaches_the_length3_cap():
    from paper_1809_11134_b200 import PopulationConfig, QeqeaEngine, target_matrix

    for s in SEEDS:
        best, gen = _run(QeqeaEngine(PopulationConfig(2, 3, 5, max_generations=50_000, target_fitness=0.999),
                                     target_matrix("CNOT"), s))
        assert CNOT_L3_CAP - 1e-3 < best <= CNOT_L3_CAP + 1e-12, (s, best)
        assert gen == 50_000


def test_criterion_2_ga_synthesizes_cnot():
    """The reference asserts 5/5 successes on seeds 1..5 (test_acceptance.py:185-191).
    Per seed that is a Bernoulli draw: the reference's own GA succeeds on
    34/40 seeds (tests/golden/ga_cnot_outcomes_reference.json, made by
    oracle/gen_ga_cnot_outcomes.py; 3 of its failures sit at the 0.4588
    local optimum).  So the device GA must match the RATE over the same 40
    seeds: within 2.6 standard deviations of the reference's proportion."""
    import json
    from pathlib import Path

    from paper_1809_11134_b200 import GaConfig, GaEngine, target_matrix

    ref = json.loads((Path(__file__).parent / "golden" / "ga_cnot_outcomes_reference.json").read_text())
    ok = 0
    for s in range(1, ref["seeds"] + 1):
        best, gen = _run(GaEngine(GaConfig(2, 6, 50, mutation_rate=0.2, mutation_range=math.pi / 8,
                                           structural_rate=0.2, max_generations=10_000, target_fitness=0.999),
                                  target_matrix("CNOT"), s))
        assert (best >= 0.999) == (gen < 10_000), (s, best, gen)
        ok += best >= 0.999
    p = ref["successes"] / ref["seeds"]
    assert ok >= ref["seeds"] * p - 2.6 * math.sqrt(ref["seeds"] * p * (1 - p)), (ok, ref["successes"])


def test_criterion_3_ga_beats_qeqea_on_toffoli():
    from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

    t = target_matrix("Toffoli")
    ga = [_run(GaEngine(GaConfig(3, 16, 50, max_generations=20_000), t, s))[0] for s in SEEDS]
    qe = [_run(QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=20_000), t, s))[0] for s in SEEDS]
    assert statistics.median(ga) >= statistics.median(qe)
    assert 0.40 < statistics.median(qe) < 0.55  # the reference's plateau (README: 0.45-0.52)


@pytest.mark.parametrize("kind", ["c3_ga_toffoli", "c3_qeqea_toffoli", "c12_qeqea_CCCNOT_2000",
                                  "c12_qeqea_Peres_2000", "c12_ga_Peres_1000"])
def test_outcome_distributions_match_the_reference_over_40_seeds(kind):
    """Criteria 3 (Toffoli, 20k generations) and 12 (smoke runs) as
    distributions of the best fitness over seeds 1..40, against the
    reference's own engines run on the same configurations and seeds
    (tests/golden/acceptance_outcomes_reference.json, written by
    oracle/gen_acceptance_outcomes.py): a two-sided Mann-Whitney U test must
    not reject equality at the 1 % level."""
    import json
    from pathlib import Path

    from scipy.stats import mannwhitneyu

    from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

    ref = json.loads((Path(__file__).parent / "golden" / "acceptance_outcomes_reference.json").read_text())
    seeds = range(1, ref["seeds"] + 1)
    if kind.startswith("c3"):
        t = target_matrix("Toffoli")
        make = ((lambda s: GaEngine(GaConfig(3, 16, 50, max_generations=20_000), t, s)) if "ga" in kind else
                (lambda s: QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=20_000), t, s)))
    else:
        _, algo, name, gens = kind.split("_")
        spec = target_matrix(name)
        make = ((lambda s: QeqeaEngine(PopulationConfig(spec.number_of_wires, 16, 5, max_generations=int(gens)),
                                       spec, s)) if algo == "qeqea" else
                (lambda s: GaEngine(GaConfig(spec.number_of_wires, 16, 20, max_generations=int(gens)), spec, s)))
    device = [_run(make(s))[0] for s in seeds]
    reference = [ref[kind][str(s)] for s in seeds]
    assert mannwhitneyu(device, reference).pvalue > 0.01, (statistics.median(device), statistics.median(reference))
