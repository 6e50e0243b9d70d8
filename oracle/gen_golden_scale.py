"""Multi-block trajectory fixtures from the REFERENCE implementation itself.

TEST INFRASTRUCTURE ONLY (build container; /root/reference does not exist on
the GPU box, so the outputs are committed as fixtures under tests/golden/).

The round-1 trajectory goldens (oracle/gen_golden.py) have P <= 6: one values
tile and one commit block on the device.  These cover the shapes the product
runs at, where the device splits a generation over hundreds of blocks and
many touches of one generation collide on the same slot (claim-stamped
qutrit commits, unarbitrated angle stores, the slot_max atomicMax, the lazy
revert):

  traj_scale_n4.npz   n=4, L=32, P=4096, CCCNOT, 5 generations
                      (131k touches per generation, ~6k colliding slots)
  traj_scale_n5.npz   n=5, L=64, P=1024, Haar target, 5 generations
  traj_scale_c4.npz   BASELINE config 4: n=4, L=32, P=65536, CCCNOT, 3 generations
                      (per-circuit fitness kept for a seeded sample of 8192)
  traj_ga_p300.npz    GA, P=300  (cooperative launch, P > 256 variant)
  traj_ga_p1024.npz   GA, P=1024 (single-thread SUS walk, P > 512)

QEQEA generations are the reference's own functions (sample_circuit,
construct_segments, SegmentBank, evaluate_circuit, SegmentFitnessTable.update,
the elitist revert of QeqeaEngine.step, mutate_angle / mutate_qutrit) on the
per-unit Philox streams of oracle/streams.py (gen_golden.PhiloxQeqeaEngine).
Two shortcuts that do not change any value:
  * only the rotation slots a circuit touches are measured: every slot has
    its own measurement stream, and evaluate_circuit reads only the
    descriptors of blueprint slots;
  * the initial bank is oracle.streams.init_slot per slot (the device's own
    init, pinned on the GPU by test_device_init_matches_oracle_init), so the
    fixture does not have to carry a 36 MB initial bank.

The fixtures are compact (whole banks would be tens of MB): per generation
the fitness of every circuit, SHA-256 of the blueprints and of the sorted
improved set, 256 contiguous-range bucket sums of the live bank (theta,
qutrit components, slot_max) and the exact values of a seeded sample of
slots (uniform + improved ones).

Usage:  python oracle/gen_golden_scale.py [qeqea|c4|ga]...
"""
from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))

import gen_golden as G  # noqa: E402  (imports the reference from /root/reference/pkg/src)
from gen_golden import R_eng, TargetSpec, mutate_slot, stream, target_for  # noqa: E402

from oracle.streams import DOM_MEASURE, DOM_SAMPLE, init_slot  # noqa: E402

OUT = ROOT / "tests" / "golden"
BUCKETS = 256
SAMPLE_UNIFORM = 512
SAMPLE_IMPROVED = 512


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def bucket_sums(x: np.ndarray) -> np.ndarray:
    """Sums over 256 contiguous index ranges (axis 0), ranges [b*N//256, (b+1)*N//256)."""
    n = x.shape[0]
    edges = (np.arange(BUCKETS + 1) * n) // BUCKETS
    c = np.concatenate([np.zeros((1,) + x.shape[1:]), np.cumsum(x, axis=0)])
    return c[edges[1:]] - c[edges[:-1]]


def bank_summary(th, q, sm):
    return (bucket_sums(th), bucket_sums(q.real), bucket_sums(q.imag), bucket_sums(sm))


class ScaleQeqea(G.PhiloxQeqeaEngine):
    """gen_golden.PhiloxQeqeaEngine measuring only the touched rotation slots."""

    def __init__(self, cfg, spec, seed):
        super().__init__(cfg, spec, seed)
        Q, Qt = cfg.qubit_count, cfg.qutrit_count
        th = np.empty(Q)
        q = np.empty((Qt, 3), dtype=np.complex128)
        for s in range(Q):
            t, qq = init_slot(seed, s, s < Qt)
            th[s] = t
            if qq is not None:
                q[s] = qq
        self.pop = R_eng.PopulationState(thetas=th, qutrits=q)

    def step(self):
        cfg = self.cfg
        g = self.generation
        blueprints = [R_eng.sample_circuit(cfg, stream(self.seed, DOM_SAMPLE, g, c))
                      for c in range(cfg.size_of_population)]
        bps = np.stack(blueprints)
        axes = np.full(cfg.qutrit_count, -1, dtype=np.int64)
        for s in np.unique(bps[bps < cfg.qutrit_count]):
            s = int(s)
            one = R_eng.PopulationState(thetas=np.zeros(1), qutrits=self.pop.qutrits[s:s + 1])
            axes[s] = int(R_eng.construct_segments(one, cfg, self.templates,
                                                   stream(self.seed, DOM_MEASURE, g, s)).axes[0])
        bank = R_eng.SegmentBank(cfg, self.templates, self.pop.thetas.copy(), axes)
        fitnesses = [R_eng.evaluate_circuit(bp, bank, self.target.matrix) for bp in blueprints]
        improved = set()
        for bp, fit in zip(blueprints, fitnesses):
            improved |= self.table.update(bp, fit)
            if fit > self.best_fitness:
                self.best_fitness = fit
                self.best_gates = [bank.descriptor(int(f)) for f in bp]
        for flat, (theta, qutrit) in self.pending.items():
            if flat not in improved:
                self.pop.thetas[flat] = theta
                if qutrit is not None:
                    self.pop.qutrits[flat] = qutrit
        pending = {}
        for flat in range(cfg.qubit_count):
            snap = mutate_slot(self.pop.thetas, self.pop.qutrits, self.table.slot_max, cfg,
                               self.seed, g, flat)
            if snap is not None:
                pending[flat] = snap
        self.pending = pending
        self.generation += 1
        if self.best_fitness >= cfg.target_fitness:
            self.stop_reason = "target-reached"
        elif self.generation >= cfg.max_generations:
            self.stop_reason = "generation-limit"
        self._last = (bps, np.array(fitnesses), np.array(sorted(improved), dtype=np.int64))
        return max(fitnesses), float(np.mean(fitnesses))


def gen_qeqea_scale(name, n, L, P, target, gens, seed, fit_sample=None, **kw):
    t0 = time.time()
    cfg = R_eng.PopulationConfig(number_of_wires=n, size_of_individual=L, size_of_population=P,
                                 max_generations=gens, **kw)
    eng = ScaleQeqea(cfg, TargetSpec(name, n, target), seed)
    rs = np.random.default_rng(seed + 1000)
    out = dict(n=n, L=L, P=P, seed=seed, gens=gens, target=target,
               p_mut=cfg.probability_of_mutation, mutation_range=cfg.mutation_range,
               n_meas=cfg.n_meas, target_fitness=cfg.target_fitness, buckets=BUCKETS)
    rec, fits, bp_sha, imp_sha, imp_n, collide = [], [], [], [], [], []
    sums = [[], [], [], []]
    s_idx, s_th, s_q, s_sm = [], [], [], []
    while not eng.done:
        gb, gm = eng.step()
        rec.append((gb, gm, eng.best_fitness))
        bps, ft, imp = eng._last
        fits.append(ft)
        bp_sha.append(sha(bps))
        imp_sha.append(sha(imp))
        imp_n.append(imp.size)
        _, counts = np.unique(bps, return_counts=True)
        collide.append(int((counts > 1).sum()))
        th, q, sm = eng.pop.thetas, eng.pop.qutrits, eng.table.slot_max
        for acc, v in zip(sums, bank_summary(th, q, sm)):
            acc.append(v)
        uni = rs.choice(cfg.qubit_count, SAMPLE_UNIFORM, replace=False)
        pick = rs.choice(imp, min(SAMPLE_IMPROVED, imp.size), replace=False) if imp.size else imp
        idx = np.unique(np.concatenate([uni, pick]).astype(np.int64))
        idx = np.concatenate([idx, np.full(SAMPLE_UNIFORM + SAMPLE_IMPROVED - idx.size, -1)])
        s_idx.append(idx)
        ok = idx >= 0
        s_th.append(np.where(ok, th[np.maximum(idx, 0)], 0.0))
        s_sm.append(np.where(ok, sm[np.maximum(idx, 0)], 0.0))
        rot = ok & (idx < cfg.qutrit_count)
        s_q.append(np.where(rot[:, None], q[np.clip(idx, 0, cfg.qutrit_count - 1)], 0.0))
        print(f"  {name} gen {eng.generation}: best {eng.best_fitness:.6f}, improved {imp.size}, "
              f"colliding slots {collide[-1]}, {time.time() - t0:.0f}s", flush=True)
    fits = np.stack(fits)
    if fit_sample is not None and fit_sample < P:
        # large populations: every circuit's fitness enters the records (max,
        # mean); the per-circuit values are kept for a seeded sample
        fidx = np.sort(rs.choice(P, fit_sample, replace=False))
        out.update(fitness_idx=fidx)
        fits = fits[:, fidx]
    out.update(
        records=np.array(rec), fitness=fits, blueprint_sha=np.array(bp_sha),
        improved_sha=np.array(imp_sha), improved_count=np.array(imp_n), colliding_slots=np.array(collide),
        theta_sums=np.stack(sums[0]), qre_sums=np.stack(sums[1]), qim_sums=np.stack(sums[2]),
        slot_max_sums=np.stack(sums[3]), sample_idx=np.stack(s_idx), sample_thetas=np.stack(s_th),
        sample_qutrits=np.stack(s_q), sample_slot_max=np.stack(s_sm),
        best_codes=np.array([G.code_of(g, n) for g in eng.best_gates], dtype=np.uint8),
        best_thetas=np.array([g.theta for g in eng.best_gates]),
        generations_run=eng.generation, stop_reason=str(eng.stop_reason),
    )
    np.savez_compressed(OUT / f"traj_scale_{name}.npz", **out)


def main(which):
    OUT.mkdir(parents=True, exist_ok=True)
    if "qeqea" in which:
        gen_qeqea_scale("n4", 4, 32, 4096, target_for(4, "CCCNOT"), 5, 31)
        gen_qeqea_scale("n5", 5, 64, 1024, target_for(5, "haar"), 5, 32)
    if "c4" in which:  # BASELINE config 4 itself (n=4, L=32, P=2^16, C^3NOT)
        gen_qeqea_scale("c4", 4, 32, 65536, target_for(4, "CCCNOT"), 3, 33, fit_sample=8192)
    if "ga" in which:
        G.gen_ga_traj("p300", 3, 16, 300, target_for(3, "Toffoli"), 12, 41)
        G.gen_ga_traj("p1024", 3, 16, 1024, target_for(3, "Toffoli"), 6, 42)
    print("wrote", sorted(p.name for p in OUT.glob("traj_*.npz")))


if __name__ == "__main__":
    main(sys.argv[1:] or ["qeqea", "ga"])
