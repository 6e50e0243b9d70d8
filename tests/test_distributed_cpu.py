"""Population sharding host logic (paper_1809_11134_b200.distributed) on CPU:
world_size 2 over gloo, each rank an oracle replica scoring its shard; the
sharded trajectory must equal the single-process one exactly."""
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


class OracleOps:
    """ShardedRunner ops over an oracle replica (QEQEA or GA)."""

    def __init__(self, oracle, P, rank, world, qeqea: bool):
        self.o, self.P, self.rank, self.world, self.qeqea = oracle, P, rank, world, qeqea
        self.shard_len = -(-P // world)
        self.fitness_full = torch.zeros(self.shard_len * world, dtype=torch.float64)
        self.max_batch = 7

    def begin_batch(self):
        self.recs = []

    def eval(self):
        if self.qeqea:
            self.o.begin_generation()
        c0 = self.rank * self.shard_len
        c1 = min(self.P, c0 + self.shard_len)
        self.fitness_full.zero_()
        if c1 > c0:
            self.fitness_full[c0:c1] = torch.from_numpy(self.o.evaluate(c0, c1))

    def finish(self):
        if self.o.done:
            return
        gb, gm = self.o.finish_generation(self.fitness_full[: self.P].numpy().copy())
        self.recs.append((gb, gm, self.o.best_fitness, 0.0))

    def read_batch(self):
        return np.array(self.recs, dtype=REC), STOP_CODE[self.o.stop_reason]


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
        lay = O.Layout(3, 8, 5, max_generations=25)
        T = np.eye(8)[[0, 1, 2, 3, 4, 5, 7, 6]].astype(complex)
        oracle = O.OracleQeqea(lay, T, 7)
        ops = OracleOps(oracle, lay.P, rank, world, True)
    else:
        cfg = OG.GaLayout(2, 5, 11, max_generations=25)
        T = np.eye(4)[[0, 1, 3, 2]].astype(complex)
        oracle = OG.OracleGa(cfg, T, 5)
        ops = OracleOps(oracle, cfg.P, rank, world, False)
    r = ShardedRunner(ops)
    rec = r.steps(25)
    q.put((rank, rec["gen_best"].tolist(), rec["gen_mean"].tolist(), r.generation, r.stop_reason,
           oracle.thetas.tolist() if kind == "qeqea" else oracle.codes.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["qeqea", "ga"])
def test_sharded_runner_matches_single_process(kind):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get() for _ in range(2)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if kind == "qeqea":
        ref = O.OracleQeqea(O.Layout(3, 8, 5, max_generations=25),
                            np.eye(8)[[0, 1, 2, 3, 4, 5, 7, 6]].astype(complex), 7)
        state = lambda o: o.thetas.tolist()
    else:
        ref = OG.OracleGa(OG.GaLayout(2, 5, 11, max_generations=25),
                          np.eye(4)[[0, 1, 3, 2]].astype(complex), 5)
        state = lambda o: o.codes.tolist()
    trace = [ref.step() for _ in range(25)]
    for rank, gb, gm, gen, stop, st in res:
        assert gb == [t[0] for t in trace]
        assert gm == [t[1] for t in trace]
        assert gen == 25 and stop == "generation-limit"
        assert st == state(ref)
