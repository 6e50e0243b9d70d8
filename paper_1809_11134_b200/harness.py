"""Engine factory for the reference's run configuration (harness.py:21-50).

`build_engine(cfg)` takes the reference's `RunConfig` (config.py:18-41) — or
any object with the same attributes — and returns the device engine for
`cfg.algo`, so the reference's run / resume / checkpoint plumbing
(harness.py:73-139, report.py:127-168) drives the B200 generation loop
unchanged: it only calls `engine.step()`, reads `generation`, `best_fitness`,
`best_gates`, `stop_reason`, `config_echo()` and pickles the engine.  The
reference's config-file parsing, convention sweep and compare stay with the
reference.
"""
from __future__ import annotations

from typing import Optional

from .engine import PopulationConfig, QeqeaEngine
from .errors import ConfigurationError
from .fitness import TargetSpec, target_matrix
from .ga import GaConfig, GaEngine
from .report import RunReport, run_engine


def resolve_target(cfg) -> TargetSpec:
    """harness.py:21-22: named target or target file, sized by numberOfWires."""
    return target_matrix(cfg.target, cfg.number_of_wires)


def build_engine(cfg, target: Optional[TargetSpec] = None, *, device: int = 0, precision: str = "fp64"):
    """harness.py:25-50 with the device engines (same field mapping)."""
    spec = target if target is not None else resolve_target(cfg)
    n = spec.number_of_wires
    if cfg.algo == "qeqea":
        pop_cfg = PopulationConfig(
            number_of_wires=n,
            size_of_individual=cfg.size_of_individual,
            size_of_population=cfg.size_of_population,
            probability_of_mutation=cfg.probability_of_mutation,
            mutation_range=cfg.mutation_range,
            n_meas=cfg.n_meas,
            max_generations=cfg.max_generations,
            target_fitness=cfg.target_fitness,
        )
        return QeqeaEngine(pop_cfg, spec, cfg.seed, workers=cfg.workers, device=device, precision=precision)
    if cfg.algo != "ga":
        raise ConfigurationError(f"unknown algo {cfg.algo!r} (expected 'qeqea' or 'ga')")
    ga_cfg = GaConfig(
        number_of_wires=n,
        size_of_individual=cfg.size_of_individual,
        population=cfg.ga_population,
        mutation_rate=cfg.ga_mutation_rate,
        mutation_range=cfg.ga_mutation_range,
        structural_rate=cfg.ga_structural_rate,
        max_generations=cfg.max_generations,
        target_fitness=cfg.target_fitness,
    )
    return GaEngine(ga_cfg, spec, cfg.seed, workers=cfg.workers, device=device, precision=precision)


def run(cfg, target: Optional[TargetSpec] = None, **kw) -> RunReport:
    """build_engine + report.run_engine (the loop of harness.run_experiment,
    without its file outputs)."""
    return run_engine(build_engine(cfg, target, **kw))
