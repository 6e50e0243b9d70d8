"""Stop rule after a stop: resume with a larger max_generations and step()
after a stop, as the reference behaves.

* harness.resume_experiment (reference harness.py:95-139) replaces
  engine.cfg with a larger max_generations and clears stop_reason; the
  continued run must equal an uninterrupted one
  (reference pkg/tests/test_harness.py:185-212, same configuration).
* engine.step() after a stop still runs one generation (engine.py:318-361,
  ga.py:165-194) and keeps the stop reason."""
import math
import pickle
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("algo", ["qeqea", "ga"])
def test_resume_matches_uninterrupted_run(tmp_path, algo):
    from paper_1809_11134_b200.harness import resume_experiment, run_experiment
    from paper_1809_11134_b200.report import RunReport

    base = dict(algo=algo, target="CNOT", seed=13, size_of_individual=3, size_of_population=5,
                target_fitness=1.0)
    full = run_experiment(RunConfigLike(max_generations=1000, out_dir=str(tmp_path / "full"), **base))
    part_dir = tmp_path / "part"
    part = run_experiment(RunConfigLike(max_generations=400, out_dir=str(part_dir), checkpoint_every=400, **base))
    assert len(part.records) == 400 and part.stop_reason == "generation-limit"
    resumed = resume_experiment(part_dir / "checkpoint.pkl", max_generations=1000)
    assert len(resumed.records) == 1000
    assert [r.best_fitness for r in resumed.records] == [r.best_fitness for r in full.records]
    assert [r.mean_fitness for r in resumed.records] == [r.mean_fitness for r in full.records]
    assert resumed.final_fitness == full.final_fitness
    assert resumed.stop_reason == full.stop_reason == "generation-limit"
    assert [g.to_dict() for g in resumed.best_gates] == [g.to_dict() for g in full.best_gates]
    assert len((part_dir / "generations.log").read_text().splitlines()) == 1000
    assert RunReport.load(part_dir / "report.json").final_fitness == full.final_fitness
    assert "stopReason:   generation-limit" in (part_dir / "summary.txt").read_text()


def _engines(algo, max_generations, seed=5):
    from paper_1809_11134_b200 import GaConfig, GaEngine, PopulationConfig, QeqeaEngine, target_matrix

    t = target_matrix("Toffoli")
    if algo == "qeqea":
        return QeqeaEngine(PopulationConfig(3, 16, 7, max_generations=max_generations), t, seed)
    return GaEngine(GaConfig(3, 16, 20, max_generations=max_generations), t, seed)


@pytest.mark.parametrize("algo", ["qeqea", "ga"])
def test_step_after_generation_limit_runs_a_generation(algo):
    a = _engines(algo, 10)
    ra = a.steps(10)
    assert a.done and a.stop_reason == "generation-limit"
    extra = [a.step() for _ in range(3)]
    assert a.generation == 13 and a.stop_reason == "generation-limit"
    b = _engines(algo, 13)
    rb = b.steps(13)
    assert np.array_equal(ra, rb[:10])
    assert [(float(r["gen_best"]), float(r["gen_mean"])) for r in rb[10:]] == extra
    assert a.best_fitness == b.best_fitness
    assert [g.to_dict() for g in a.best_gates] == [g.to_dict() for g in b.best_gates]


@pytest.mark.parametrize("algo", ["qeqea", "ga"])
def test_step_after_target_reached_keeps_the_reason(algo):
    from paper_1809_11134_b200 import GaConfig, PopulationConfig

    a = _engines(algo, 1000)
    a.cfg = replace(a.cfg, target_fitness=1e-6)  # pushed to the device: stops after generation 1
    a.steps(5)
    assert a.generation == 1 and a.stop_reason == "target-reached"
    a.step()
    assert a.generation == 2 and a.stop_reason == "target-reached"
    with pytest.raises(Exception):
        a.cfg = replace(a.cfg, size_of_individual=4)  # only the stop rule may change
    assert isinstance(a.cfg, (GaConfig, PopulationConfig))


@pytest.mark.parametrize("algo", ["qeqea", "ga"])
def test_pickled_engine_resumes_with_larger_limit(algo):
    a = _engines(algo, 30)
    a.steps(30)
    blob = pickle.dumps(a)
    b = pickle.loads(blob)
    assert b.done and b.generation == 30
    b.cfg = replace(b.cfg, max_generations=50)
    b.stop_reason = None
    rb = b.steps(100)
    assert rb.size == 20 and b.generation == 50 and b.stop_reason == "generation-limit"
    c = _engines(algo, 50)
    rc = c.steps(50)
    assert np.array_equal(rb, rc[30:])
    assert [g.to_dict() for g in b.best_gates] == [g.to_dict() for g in c.best_gates]
