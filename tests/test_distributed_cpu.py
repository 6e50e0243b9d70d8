"""Population sharding host logic (paper_1809_11134_b200.distributed) on CPU.

World sizes 2 and 3 over gloo.  Each rank drives the same ShardedRunner /
Routing / Comm code the device path uses, with an oracle replica standing in
for the kernels: it samples only its own circuits, routes their touches to
the owning ranks (all-to-all), answers with the gate codes / live angles of
the touches it owns (all-to-all back), scores its circuits from what it
received, and all-gathers fitness + elite records.  The sharded trajectory
must equal the single-process one exactly, and the best gates taken from the
gathered elites must equal the oracle's best circuit."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ga as OG
from oracle import qeqea as O

STOP_CODE = {None: 0, "target-reached": 1, "generation-limit": 2}
REC = np.dtype([("gen_best", "f8"), ("gen_mean", "f8"), ("best_fitness", "f8"), ("reserved", "f8")])
NO_SLOT = -1

QEQEA_CASE = dict(n=3, L=8, P=5, gens=25, seed=7)
GA_CASE = dict(n=2, L=5, P=11, gens=25, seed=5)


def _toffoli_like():
    return np.eye(8)[[0, 1, 2, 3, 4, 5, 7, 6]].astype(complex)


class _OpsBase:
    max_batch = 7

    def begin_batch(self):
        self.recs = []

    def read_batch(self):
        return np.array(self.recs, dtype=REC), STOP_CODE[self.o.stop_reason]


class OracleQeqeaOps(_OpsBase):
    """The QEQEA split-phase protocol (include/isq.h) over an oracle replica."""

    def __init__(self, oracle, lay, rank, world):
        from paper_1809_11134_b200.distributed import Routing

        self.o, self.lay, self.rank, self.world = oracle, lay, rank, world
        self.S = -(-lay.P // world)
        self.c0 = rank * self.S
        self.routing = Routing(lay.L, self.S, world, rank)
        self.E = 2 + 2 * lay.L
        self.fitness = torch.zeros(world * self.S, dtype=torch.float64)
        self.elite = torch.zeros(world * self.E, dtype=torch.float64)

    def generation(self, comm):
        o, lay, r = self.o, self.lay, self.routing
        if o.done:
            return
        o.begin_generation()  # this generation's blueprints, axes and bank angles
        # prepare: own circuits only, padding circuits send NO_SLOT
        flats = np.full((self.S, lay.L), NO_SLOT, dtype=np.int64)
        for i in range(self.S):
            if self.c0 + i < lay.P:
                flats[i] = O.sample_blueprint(lay, o.seed, o.generation, self.c0 + i)
        recv = torch.empty(self.world * self.S * r.Lr, dtype=torch.int64)
        comm.all_to_all(recv, torch.from_numpy(r.route(flats)), r.from_circuits, r.to_owners)
        # values: the owner answers for its positions only
        owned = recv.numpy()
        lo, hi = r.bounds[self.rank], r.bounds[self.rank + 1]
        codes = np.zeros(owned.size, dtype=np.uint8)
        thetas = np.zeros(owned.size)
        for t, f in enumerate(owned):
            if f == NO_SLOT:
                continue
            assert lo <= f % lay.L < hi, "touch routed to a rank that does not own its position"
            axis = o._axes[f] if f < lay.Qt else 0
            codes[t] = O.gate_code(lay, f, axis)
            thetas[t] = o._bank_thetas[f]
        rc = torch.empty(self.S * lay.L, dtype=torch.uint8)
        rt = torch.empty(self.S * lay.L, dtype=torch.float64)
        comm.all_to_all(rc, torch.from_numpy(codes), r.to_owners, r.from_circuits)
        comm.all_to_all(rt, torch.from_numpy(thetas), r.to_owners, r.from_circuits)
        gc, gt = r.unroute(rc.numpy()), r.unroute(rt.numpy())
        # score + elite of the shard
        self.fitness.zero_()
        best, arg = -1.0, -1
        for i in range(self.S):
            c = self.c0 + i
            if c >= lay.P:
                break
            assert list(gc[i]) == list(o._codes[c]), "routed gate codes differ"
            f = O.circuit_fitness(gc[i], gt[i], o.target, lay.n)
            self.fitness[c] = f
            if f > best:
                best, arg = f, c
        e = self.elite[self.rank * self.E:(self.rank + 1) * self.E]
        e.zero_()
        e[0], e[1] = best, arg
        if arg >= 0:
            e[2:2 + lay.L] = torch.from_numpy(gt[arg - self.c0])
            e[2 + lay.L:] = torch.from_numpy(gc[arg - self.c0].astype(np.float64))
        comm.all_gather(self.fitness, self.S)
        comm.all_gather(self.elite, self.E)
        # finish on the gathered vector; best gates from the owning rank's elite
        prev = o.best_fitness
        gb, gm = o.finish_generation(self.fitness[: lay.P].numpy().copy())
        if o.best_fitness > prev:
            fit = self.fitness[: lay.P].numpy()
            c = int(np.argmax(fit))
            ee = self.elite[(c // self.S) * self.E:(c // self.S + 1) * self.E].numpy()
            assert int(ee[1]) == c and ee[0] == fit[c]
            assert [int(x) for x in ee[2 + lay.L:]] == o.best_codes
            assert list(ee[2:2 + lay.L]) == o.best_thetas
        self.recs.append((gb, gm, o.best_fitness, 0.0))


class OracleGaOps(_OpsBase):
    """The GA protocol: score the genome shard, all-gather, breed on every rank."""

    def __init__(self, oracle, P, rank, world):
        self.o, self.P, self.rank = oracle, P, rank
        self.S = -(-P // world)
        self.fitness = torch.zeros(self.S * world, dtype=torch.float64)

    def generation(self, comm):
        if self.o.done:
            return
        c0 = self.rank * self.S
        c1 = min(self.P, c0 + self.S)
        self.fitness.zero_()
        if c1 > c0:
            self.fitness[c0:c1] = torch.from_numpy(self.o.evaluate(c0, c1))
        comm.all_gather(self.fitness, self.S)
        gb, gm = self.o.finish_generation(self.fitness[: self.P].numpy().copy())
        self.recs.append((gb, gm, self.o.best_fitness, 0.0))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_11134_b200.distributed import ShardedRunner

    if kind == "qeqea":
        k = QEQEA_CASE
        lay = O.Layout(k["n"], k["L"], k["P"], max_generations=k["gens"])
        oracle = O.OracleQeqea(lay, _toffoli_like(), k["seed"])
        ops = OracleQeqeaOps(oracle, lay, rank, world)
    else:
        k = GA_CASE
        cfg = OG.GaLayout(k["n"], k["L"], k["P"], max_generations=k["gens"])
        oracle = OG.OracleGa(cfg, np.eye(4)[[0, 1, 3, 2]].astype(complex), k["seed"])
        ops = OracleGaOps(oracle, cfg.P, rank, world)
    r = ShardedRunner(ops)
    rec = r.steps(k["gens"])
    q.put((rank, rec["gen_best"].tolist(), rec["gen_mean"].tolist(), r.generation, r.stop_reason,
           oracle.thetas.tolist() if kind == "qeqea" else oracle.codes.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("qeqea", 2), ("qeqea", 3), ("ga", 2)])
def test_sharded_runner_matches_single_process(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get() for _ in range(world)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if kind == "qeqea":
        k = QEQEA_CASE
        ref = O.OracleQeqea(O.Layout(k["n"], k["L"], k["P"], max_generations=k["gens"]), _toffoli_like(),
                            k["seed"])
        state = lambda o: o.thetas.tolist()
    else:
        k = GA_CASE
        ref = OG.OracleGa(OG.GaLayout(k["n"], k["L"], k["P"], max_generations=k["gens"]),
                          np.eye(4)[[0, 1, 3, 2]].astype(complex), k["seed"])
        state = lambda o: o.codes.tolist()
    trace = [ref.step() for _ in range(k["gens"])]
    for rank, gb, gm, gen, stop, st in res:
        assert gb == [t[0] for t in trace]
        assert gm == [t[1] for t in trace]
        assert gen == k["gens"] and stop == "generation-limit"
        assert st == state(ref)


@pytest.mark.parametrize("L,world", [(8, 2), (8, 3), (64, 8), (5, 5)])
def test_routing_round_trip(L, world):
    """route / unroute are inverse and every position lands at its owner."""
    from paper_1809_11134_b200.distributed import Routing

    S = 3
    owners = [Routing(L, S, world, r) for r in range(world)]
    rng = np.random.default_rng(L * 31 + world)
    circ = rng.integers(0, 10**6, size=(S, L))
    r0 = owners[0]
    grouped = r0.route(circ)
    assert grouped.size == S * L and sum(r0.to_owners) == S * L
    assert np.array_equal(r0.unroute(grouped), circ)
    off = 0
    for o, ro in enumerate(owners):
        block = grouped[off:off + r0.to_owners[o]].reshape(S, ro.Lr)
        assert np.array_equal(block, circ[:, ro.bounds[o]:ro.bounds[o + 1]])
        assert ro.from_circuits == [S * ro.Lr] * world
        off += r0.to_owners[o]
    assert sum(ro.Lr for ro in owners) == L
    assert all(math.isclose(ro.Lr, L / world, abs_tol=1) for ro in owners)
