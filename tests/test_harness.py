"""Engine factory for the reference's RunConfig (harness.py:25-50)."""
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import pytest


@dataclass
class RunConfigLike:
    """Field-for-field mirror of the reference's RunConfig (config.py:18-41)."""

    algo: str = "qeqea"
    target: str = "CNOT"
    number_of_wires: Optional[int] = None
    size_of_individual: int = 3
    size_of_population: int = 5
    probability_of_mutation: float = 0.3
    mutation_range: float = math.pi / 4
    n_meas: int = 1
    max_generations: int = 10_000_000
    target_fitness: float = 0.999
    ga_population: int = 50
    ga_mutation_rate: float = 0.1
    ga_mutation_range: float = math.pi / 8
    ga_structural_rate: float = 0.1
    seed: int = 0
    out_dir: str = "runs"
    checkpoint_every: int = 0
    workers: int = 1
    verbose_log: bool = False


def test_unknown_algo_is_a_configuration_error():
    from paper_1809_11134_b200.errors import ConfigurationError
    from paper_1809_11134_b200.harness import build_engine

    with pytest.raises(ConfigurationError):
        build_engine(RunConfigLike(algo="sa", target="Toffoli"))


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["qeqea", "ga"])
def test_build_engine_runs_the_device_engine(algo):
    from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix
    from paper_1809_11134_b200.harness import build_engine, run

    cfg = RunConfigLike(algo=algo, target="Toffoli", size_of_individual=16, max_generations=60, seed=3)
    eng = build_engine(cfg)
    assert eng.algorithm == algo
    assert eng.config_echo()["maxGenerations"] == 60
    eng.close()
    report = run(cfg)
    t = target_matrix("Toffoli")
    if algo == "qeqea":
        ref = QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=60), t, 3)
    else:
        ref = GaEngine(GaConfig(3, 16, 50, max_generations=60), t, 3)
    rec = ref.steps(60)
    assert report.stop_reason == ref.stop_reason == "generation-limit"
    assert [r.best_fitness for r in report.records] == list(rec["best_fitness"])
    assert report.final_fitness == ref.best_fitness
    assert [g.to_dict() for g in report.best_gates] == [g.to_dict() for g in ref.best_gates]
