"""Engine factory for the reference's run configuration (harness.py:21-50).

`build_engine(cfg)` takes the reference's `RunConfig` (config.py:18-41) — or
any object with the same attributes — and returns the device engine for
`cfg.algo`, so the reference's run / resume / checkpoint plumbing
(harness.py:73-139, report.py:127-168) drives the B200 generation loop
unchanged: it only calls `engine.step()`, reads `generation`, `best_fitness`,
`best_gates`, `stop_reason`, `config_echo()` and pickles the engine.
`run_experiment` / `resume_experiment` (harness.py:73-139) write the same
files (generations.log, report.json, summary.txt, checkpoint.pkl); a resume
with a larger max_generations replaces `engine.cfg` and clears
`stop_reason`, which the device engines push to their handles.  The
reference's config-file parsing, convention sweep and compare stay with the
reference.
"""
from __future__ import annotations

import dataclasses
import pickle
from pathlib import Path
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


def _write_atomic(path: Path, data: bytes) -> None:
    tmp = path.parent / (path.name + ".tmp")
    tmp.write_bytes(data)
    tmp.replace(path)


def _outputs(out: Path, report: RunReport) -> None:
    """report.json + summary.txt (harness.py:59-70 keys and order)."""
    out.joinpath("report.json").write_text(report.to_json())
    fields = (("algorithm", report.algorithm), ("target", report.target), ("seed", report.seed),
              ("generations", len(report.records)), ("finalFitness", f"{report.final_fitness:.6f}"),
              ("stopReason", report.stop_reason),
              ("bestCircuit", report.to_dict()["bestCircuitText"]))
    out.joinpath("summary.txt").write_text("".join(f"{(k + ':').ljust(14)}{v}\n" for k, v in fields))


def _drive(engine, cfg, out: Path, report: Optional[RunReport], log_mode: str) -> RunReport:
    def checkpoint(eng, rep):
        _write_atomic(out / "checkpoint.pkl", pickle.dumps({"engine": eng, "report": rep, "config": cfg}))

    every = int(getattr(cfg, "checkpoint_every", 0) or 0)
    with open(out / "generations.log", log_mode) as log:
        report = run_engine(engine, log_fh=log, checkpoint_fn=checkpoint if every > 0 else None,
                            checkpoint_every=every, report=report)
    _outputs(out, report)
    return report


def run_experiment(cfg, target: Optional[TargetSpec] = None, **kw) -> RunReport:
    """harness.py:73-92: one configured run with its log, report and
    checkpoints under cfg.out_dir, on the device engines."""
    out = Path(cfg.out_dir)
    try:
        out.mkdir(parents=True, exist_ok=True)
    except OSError as exc:
        raise IOError(f"cannot create output directory {out}: {exc}") from exc
    return _drive(build_engine(cfg, target, **kw), cfg, out, None, "w")


def resume_experiment(checkpoint_path, max_generations: Optional[int] = None) -> RunReport:
    """harness.py:95-139: continue a checkpointed run.  The unpickled device
    engine carries its whole state (bank, table, generation, best), so the
    trajectory equals an uninterrupted run's."""
    try:
        saved = pickle.loads(Path(checkpoint_path).read_bytes())
    except OSError as exc:
        raise IOError(f"cannot read checkpoint {checkpoint_path}: {exc}") from exc
    engine, report, cfg = saved["engine"], saved["report"], saved["config"]
    if max_generations is not None:
        engine.cfg = dataclasses.replace(engine.cfg, max_generations=max_generations)
        if engine.stop_reason == "generation-limit" and engine.generation < max_generations:
            engine.stop_reason = None
    out = Path(cfg.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    return _drive(engine, cfg, out, report, "a")
