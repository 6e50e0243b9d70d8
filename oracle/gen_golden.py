"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

TEST INFRASTRUCTURE ONLY.  Runs in the build container, where the reference
package is importable from /root/reference/pkg/src (it does not exist on the
GPU box, so the outputs are committed as fixtures).  Every value below comes
from the reference's own functions (isingsynth.*), driven with the per-unit
Philox streams of oracle/streams.py wherever the reference would draw from its
sequential Generator:

  fitness.npz     fitness_value(compose_gates(...)) + composed unitaries
  sampling.npz    engine.sample_circuit on Philox streams
  measure.npz     engine.construct_segments per slot stream
  mutate.npz      encoding.mutate_angle / mutate_qutrit per slot stream
  traj_*.npz      PhiloxQeqeaEngine / PhiloxGaEngine trajectories built from
                  reference functions only (init from engine.init_population)

Usage:  python oracle/gen_golden.py   (writes tests/golden/)
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from isingsynth import encoding as R_enc  # noqa: E402
from isingsynth import engine as R_eng  # noqa: E402
from isingsynth import ga as R_ga  # noqa: E402
from isingsynth.fitness import TargetSpec, fitness_value, target_matrix  # noqa: E402
from isingsynth.gates import Axis, GateOp, compose_gates, enumerate_templates  # noqa: E402

from oracle.streams import (  # noqa: E402
    DOM_GA_INIT,
    DOM_GA_MUT,
    DOM_GA_PAIR,
    DOM_GA_SUS,
    DOM_MEASURE,
    DOM_MUTATE,
    DOM_SAMPLE,
    stream,
)


def random_unitary(dim: int, rng: np.random.Generator) -> np.ndarray:
    """pkg/tests/conftest.py:10-14 (QR-Haar)."""
    z = rng.normal(size=(dim, dim)) + 1j * rng.normal(size=(dim, dim))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def gate_of(code: int, theta: float, n: int) -> GateOp:
    return R_ga._with_theta(R_ga.GaConfig(n, 1).gate_choices[int(code)], float(theta))


def code_of(g: GateOp, n: int) -> int:
    for i, c in enumerate(R_ga.GaConfig(n, 1).gate_choices):
        if c.kind == g.kind and c.wire == g.wire and c.axis == g.axis and c.pair == g.pair:
            return i
    raise ValueError(g)


def haar_target(n: int) -> np.ndarray:
    return random_unitary(2 ** n, np.random.default_rng(12345))


def target_for(n: int, name: str) -> np.ndarray:
    if name == "haar":
        return haar_target(n)
    if name == "identity":
        return np.eye(2 ** n, dtype=np.complex128)
    if name == "Fredkin":
        m = np.eye(8, dtype=np.complex128)
        m[[5, 6], [5, 6]] = 0.0
        m[5, 6] = m[6, 5] = 1.0
        return m
    return target_matrix(name).matrix


# ------------------------------------------------------------------ fitness

def gen_fitness():
    rng = np.random.default_rng(20240607)
    out = {}
    cases = [(2, "CNOT"), (3, "Toffoli"), (3, "Peres"), (3, "Fredkin"), (4, "CCCNOT"),
             (5, "haar"), (5, "identity"), (2, "haar"), (3, "haar"), (4, "haar")]
    for n, tname in cases:
        T = target_for(n, tname)
        nc = 3 * n + n * (n - 1) // 2
        for L in (0, 1, 3, 16, 33, 64):
            count = 24 if L else 2
            codes = rng.integers(0, nc, size=(count, L)).astype(np.uint8)
            thetas = rng.uniform(0.0, 2 * math.pi, size=(count, L))
            # exercise both Rx/Ry factorisations and exact special angles
            if L >= 3:
                thetas[0, :3] = [0.0, math.pi, 2 * math.pi - 1e-300]
                thetas[1, :3] = [math.pi / 2, 3 * math.pi / 2, math.pi - 1e-12]
            fits = np.empty(count)
            unis = np.empty((count, 2 ** n, 2 ** n), dtype=np.complex128)
            for c in range(count):
                gates = [gate_of(k, t, n) for k, t in zip(codes[c], thetas[c])]
                u = compose_gates(gates, n)
                unis[c] = u
                fits[c] = fitness_value(u, T)
            key = f"n{n}_{tname}_L{L}"
            out[key + "_codes"] = codes
            out[key + "_thetas"] = thetas
            out[key + "_fit"] = fits
            out[key + "_target"] = T
            if L in (0, 3, 16):
                out[key + "_unitary"] = unis
    np.savez_compressed(OUT / "fitness.npz", **out)


# ----------------------------------------------------------------- sampling

def gen_sampling():
    out = {}
    cfgs = [(2, 3, 4), (3, 16, 5), (4, 32, 1), (5, 64, 1024), (3, 7, 3), (4, 37, 6)]
    for n, L, P in cfgs:
        cfg = R_eng.PopulationConfig(number_of_wires=n, size_of_individual=L, size_of_population=P)
        for seed in (0, 7):
            for gen in (0, 3):
                bps = np.stack([R_eng.sample_circuit(cfg, stream(seed, DOM_SAMPLE, gen, c))
                                for c in range(min(P, 64))])
                out[f"n{n}_L{L}_P{P}_s{seed}_g{gen}"] = bps
    np.savez_compressed(OUT / "sampling.npz", **out)


# -------------------------------------------------------------- measurement

def construct_axis_per_slot(qutrits: np.ndarray, cfg, seed: int, gen: int) -> np.ndarray:
    """engine.construct_segments applied row by row, each on its slot stream."""
    tpl = enumerate_templates(cfg.number_of_wires)
    axes = np.empty(qutrits.shape[0], dtype=np.int64)
    for s in range(qutrits.shape[0]):
        pop = R_eng.PopulationState(thetas=np.zeros(1), qutrits=qutrits[s:s + 1])
        bank = R_eng.construct_segments(pop, cfg, tpl, stream(seed, DOM_MEASURE, gen, s))
        axes[s] = int(bank.axes[0])
    return axes


def gen_measure():
    out = {}
    rng = np.random.default_rng(5)
    for n_meas in (1, 3, 11, 61, 100, 1000):
        cfg = R_eng.PopulationConfig(number_of_wires=3, size_of_individual=8, size_of_population=25,
                                     n_meas=n_meas)
        pop = R_eng.init_population(cfg, rng)
        q = pop.qutrits
        q[0] = [1, 0, 0]
        q[1] = [0, 1j, 0]
        q[2] = [0, 0, -1]
        q[3] = np.array([1, 1, 1]) / math.sqrt(3)
        out[f"nm{n_meas}_qutrits"] = q
        for gen in (0, 9):
            out[f"nm{n_meas}_g{gen}_axes"] = construct_axis_per_slot(q, cfg, 11, gen)
    np.savez_compressed(OUT / "measure.npz", **out)


# ----------------------------------------------------------------- mutation

def mutate_slot(thetas, qutrits, slot_max, cfg, seed, gen, flat):
    """mutate_population's per-slot body (engine.py:244-262) on the slot stream."""
    st = stream(seed, DOM_MUTATE, gen, flat)
    masked = st.random() < cfg.probability_of_mutation
    coin = st.random() < 0.5
    if not masked:
        return None
    f = float(slot_max[flat])
    if f >= 1.0:
        return None
    has_q = flat < cfg.qutrit_count
    snap = (float(thetas[flat]), qutrits[flat].copy() if has_q else None)
    if coin and has_q:
        qutrits[flat] = R_enc.mutate_qutrit(qutrits[flat], f, st)
    else:
        thetas[flat] = R_enc.mutate_angle(thetas[flat], f, cfg.mutation_range, st)
    return snap


def gen_mutate():
    out = {}
    rng = np.random.default_rng(77)
    cfg = R_eng.PopulationConfig(number_of_wires=3, size_of_individual=16, size_of_population=8,
                                 probability_of_mutation=0.5)
    pop = R_eng.init_population(cfg, rng)
    slot_max = rng.uniform(0.0, 1.0, size=cfg.qubit_count)
    slot_max[::17] = 0.0
    slot_max[5::23] = 1.0
    th, q = pop.thetas.copy(), pop.qutrits.copy()
    for gen in (0, 4):
        th2, q2 = th.copy(), q.copy()
        mutated = np.zeros(cfg.qubit_count, dtype=bool)
        for flat in range(cfg.qubit_count):
            mutated[flat] = mutate_slot(th2, q2, slot_max, cfg, 3, gen, flat) is not None
        out[f"g{gen}_thetas"] = th2
        out[f"g{gen}_qutrits"] = q2
        out[f"g{gen}_mutated"] = mutated
    out["thetas0"] = th
    out["qutrits0"] = q
    out["slot_max"] = slot_max
    np.savez_compressed(OUT / "mutate.npz", **out)


# ------------------------------------------------------------ trajectories

class PhiloxQeqeaEngine(R_eng.QeqeaEngine):
    """Reference QeqeaEngine whose every RNG consumption is re-routed to the
    per-unit Philox streams; all arithmetic is the reference's."""

    def step(self):
        cfg = self.cfg
        g = self.generation
        axes = construct_axis_per_slot(self.pop.qutrits, cfg, self.seed, g)
        bank = R_eng.SegmentBank(cfg, self.templates, self.pop.thetas.copy(), axes)
        blueprints = [R_eng.sample_circuit(cfg, stream(self.seed, DOM_SAMPLE, g, c))
                      for c in range(cfg.size_of_population)]
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
        self._last = (np.stack(blueprints), axes, np.array(fitnesses),
                      np.array(sorted(improved), dtype=np.int64))
        return max(fitnesses), float(np.mean(fitnesses))


def gen_qeqea_traj(name, n, L, P, target, gens, seed, **kw):
    cfg = R_eng.PopulationConfig(number_of_wires=n, size_of_individual=L, size_of_population=P,
                                 max_generations=gens, **kw)
    spec = TargetSpec(name, n, target)
    eng = PhiloxQeqeaEngine(cfg, spec, seed)
    init_th, init_q = eng.pop.thetas.copy(), eng.pop.qutrits.copy()
    rec = []
    bps, fits, imp_flat, imp_ptr = [], [], [], [0]
    axes0 = None
    best_trace = []
    while not eng.done:
        gb, gm = eng.step()
        rec.append((gb, gm, eng.best_fitness))
        bp, ax, ft, imp = eng._last
        if axes0 is None:
            axes0 = ax
        bps.append(bp)
        fits.append(ft)
        imp_flat.extend(imp.tolist())
        imp_ptr.append(len(imp_flat))
        best_trace.append(eng.best_fitness)
    best_codes = np.array([code_of(g, n) for g in eng.best_gates], dtype=np.uint8)
    best_thetas = np.array([g.theta for g in eng.best_gates])
    np.savez_compressed(
        OUT / f"traj_qeqea_{name}.npz",
        n=n, L=L, P=P, seed=seed, gens=gens, target=target,
        p_mut=cfg.probability_of_mutation, mutation_range=cfg.mutation_range,
        n_meas=cfg.n_meas, target_fitness=cfg.target_fitness,
        init_thetas=init_th, init_qutrits=init_q,
        records=np.array(rec), blueprints=np.stack(bps), fitness=np.stack(fits),
        axes0=axes0, improved=np.array(imp_flat, dtype=np.int64),
        improved_ptr=np.array(imp_ptr, dtype=np.int64),
        final_thetas=eng.pop.thetas, final_qutrits=eng.pop.qutrits,
        final_slot_max=eng.table.slot_max, best_codes=best_codes, best_thetas=best_thetas,
        generations_run=eng.generation, stop_reason=str(eng.stop_reason),
    )


class PhiloxGaEngine(R_ga.GaEngine):
    """Reference GaEngine on per-unit Philox streams (reference operators)."""

    def __init__(self, cfg, target, seed):
        super().__init__(cfg, target, seed)
        one = R_ga.GaConfig(cfg.number_of_wires, 1)
        self.genomes = [
            tuple(R_ga.random_genome(one, stream(seed, DOM_GA_INIT, 0, i, j))[0]
                  for j in range(cfg.size_of_individual))
            for i in range(cfg.population)
        ]

    def step(self):
        cfg = self.cfg
        g = self.generation
        fitnesses = [fitness_value(R_ga.decode_genome(x, cfg.number_of_wires), self.target.matrix)
                     for x in self.genomes]
        elite = int(np.argmax(fitnesses))
        if fitnesses[elite] > self.best_fitness:
            self.best_fitness = fitnesses[elite]
            self.best_gates = list(self.genomes[elite])
        parents = R_ga.sus_select(fitnesses, cfg.population, stream(self.seed, DOM_GA_SUS, g))
        nxt = [self.genomes[elite]]
        pair_at = 0
        k = 0
        while len(nxt) < cfg.population:
            pa = self.genomes[parents[pair_at % len(parents)]]
            pb = self.genomes[parents[(pair_at + 1) % len(parents)]]
            pair_at += 2
            ca, cb = R_ga.two_point_crossover(pa, pb, stream(self.seed, DOM_GA_PAIR, g, k))
            k += 1
            for child in (ca, cb):
                if len(nxt) >= cfg.population:
                    break
                i = len(nxt)
                nxt.append(tuple(
                    R_ga.ga_mutate((gene,), cfg, stream(self.seed, DOM_GA_MUT, g, i, j))[0]
                    for j, gene in enumerate(child)))
        self.genomes = nxt
        self._parents = parents
        self._fits = fitnesses
        self.generation += 1
        if self.best_fitness >= cfg.target_fitness:
            self.stop_reason = "target-reached"
        elif self.generation >= cfg.max_generations:
            self.stop_reason = "generation-limit"
        return max(fitnesses), float(np.mean(fitnesses))


def genome_arrays(genomes, n):
    codes = np.array([[code_of(x, n) for x in gnm] for gnm in genomes], dtype=np.uint8)
    thetas = np.array([[x.theta for x in gnm] for gnm in genomes])
    return codes, thetas


def gen_ga_traj(name, n, L, P, target, gens, seed, **kw):
    cfg = R_ga.GaConfig(number_of_wires=n, size_of_individual=L, population=P,
                        max_generations=gens, **kw)
    eng = PhiloxGaEngine(cfg, TargetSpec(name, n, target), seed)
    c0, t0 = genome_arrays(eng.genomes, n)
    rec, fits, parents = [], [], []
    while not eng.done:
        gb, gm = eng.step()
        rec.append((gb, gm, eng.best_fitness))
        fits.append(eng._fits)
        parents.append(eng._parents)
    cf, tf = genome_arrays(eng.genomes, n)
    bc = np.array([code_of(x, n) for x in eng.best_gates], dtype=np.uint8)
    bt = np.array([x.theta for x in eng.best_gates])
    np.savez_compressed(
        OUT / f"traj_ga_{name}.npz",
        n=n, L=L, P=P, seed=seed, gens=gens, target=target,
        rate=cfg.mutation_rate, mrange=cfg.mutation_range, structural=cfg.structural_rate,
        target_fitness=cfg.target_fitness,
        init_codes=c0, init_thetas=t0, records=np.array(rec), fitness=np.array(fits),
        parents=np.array(parents), final_codes=cf, final_thetas=tf,
        best_codes=bc, best_thetas=bt, generations_run=eng.generation,
        stop_reason=str(eng.stop_reason),
    )


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    gen_fitness()
    gen_sampling()
    gen_measure()
    gen_mutate()
    gen_qeqea_traj("cnot", 2, 3, 4, target_for(2, "CNOT"), 60, 9)
    gen_qeqea_traj("toffoli_c1", 3, 16, 5, target_for(3, "Toffoli"), 80, 1)
    gen_qeqea_traj("fredkin_c3", 3, 16, 5, target_for(3, "Fredkin"), 40, 2, n_meas=3)
    gen_qeqea_traj("cccnot", 4, 8, 6, target_for(4, "CCCNOT"), 25, 3, probability_of_mutation=0.9)
    gen_qeqea_traj("haar5", 5, 6, 3, target_for(5, "haar"), 12, 4)
    gen_qeqea_traj("identity_conv", 2, 1, 4, target_for(2, "identity"), 4000, 5)
    gen_ga_traj("cnot", 2, 5, 10, target_for(2, "CNOT"), 40, 8)
    gen_ga_traj("toffoli_c2", 3, 16, 50, target_for(3, "Toffoli"), 30, 1)
    gen_ga_traj("odd13", 3, 7, 13, target_for(3, "Peres"), 20, 6, structural_rate=0.4, mutation_rate=0.5)
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
