"""Sharded QEQEA on one GPU: `world` ranks' handles in one process, each
driven by its own ShardedRunner thread, with the collectives emulated by
device-to-device copies between the handles' exchange buffers (no kernel
ever waits on another rank's).  The sharded run must reproduce the
single-rank trajectory bit for bit (records, fitness, stop), the union of the
ranks' owned bank slots must equal the single-rank bank, and every rank must
hold the same best circuit."""
import threading

import numpy as np
import pytest

from conftest import random_unitary

pytestmark = pytest.mark.gpu


class LockstepComm:
    """all_to_all / all_gather among in-process ranks (one thread per rank)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def rank_view(self, rank):
        outer = self

        class _View:
            world = outer.world

            def __init__(self):
                self.rank = rank

            def all_to_all(self, out, inp, out_splits, in_splits):
                outer.slots[rank] = (inp, list(in_splits))
                outer.barrier.wait()
                pos = 0
                for j in range(outer.world):
                    src, splits = outer.slots[j]
                    off = sum(splits[:rank])
                    n = splits[rank]
                    assert n == out_splits[j]
                    out[pos:pos + n].copy_(src[off:off + n])
                    pos += n
                outer.barrier.wait()

            def barrier(self):
                import torch

                torch.cuda.synchronize()
                outer.barrier.wait()

            def connect_peers(self, ops):
                outer.slots[rank] = ops.peer_buffers()
                outer.barrier.wait()
                ops.set_peer_pointers(list(outer.slots))
                outer.barrier.wait()

            def all_gather(self, full, chunk):
                outer.slots[rank] = full
                outer.barrier.wait()
                for j in range(outer.world):
                    if j != rank:
                        full[j * chunk:(j + 1) * chunk].copy_(outer.slots[j][j * chunk:(j + 1) * chunk])
                outer.barrier.wait()

        return _View()


def _run_sharded(cfg, target, seed, world, gens, transport="nccl"):
    import torch

    from paper_1809_11134_b200.distributed import DeviceQeqeaOps, ShardedRunner
    from paper_1809_11134_b200.engine import QeqeaEngine

    comm = LockstepComm(world)
    engines = [QeqeaEngine(cfg, target, seed, rank=r, world=world, max_batch=8) for r in range(world)]
    out = [None] * world

    def worker(r):
        ops = DeviceQeqeaOps(engines[r], transport)
        runner = ShardedRunner(ops, comm=comm.rank_view(r))
        rec = runner.steps(gens)
        torch.cuda.synchronize()
        out[r] = (rec, runner.stop_reason, runner.generation)

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return engines, out


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("n,L,P,gens,world", [(3, 16, 64, 30, 2), (3, 16, 61, 30, 3), (5, 64, 256, 8, 2),
                                              (4, 32, 100, 12, 4)])
def test_sharded_matches_single_rank(n, L, P, gens, world, transport):
    """transport="nccl": collectives between the phases (emulated by copies);
    "p2p": the kernels store into the other ranks' buffers themselves."""
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    T = random_unitary(2 ** n, np.random.default_rng(n * 100 + P))
    cfg = PopulationConfig(number_of_wires=n, size_of_individual=L, size_of_population=P,
                           max_generations=gens, target_fitness=1.0)
    spec = TargetSpec("haar", n, T)
    ref = QeqeaEngine(cfg, spec, seed=3)
    rrec = ref.steps(gens)
    engines, out = _run_sharded(cfg, spec, 3, world, gens, transport)
    for r, (rec, stop, generation) in enumerate(out):
        assert generation == gens and stop == "generation-limit"
        assert np.array_equal(rec["gen_best"], rrec["gen_best"]), r
        assert np.array_equal(rec["gen_mean"], rrec["gen_mean"]), r
        assert np.array_equal(rec["best_fitness"], rrec["best_fitness"]), r
        assert [g.to_dict() for g in engines[r].best_gates] == [g.to_dict() for g in ref.best_gates]
    # the owners' slots reassemble the single-rank bank exactly
    _, full = ref.owned_population()
    seen = np.zeros(cfg.qubit_count, dtype=bool)
    for e in engines:
        slots, pop = e.owned_population()
        assert np.array_equal(pop.thetas, full.thetas[slots])
        rot = slots[slots < cfg.qutrit_count]
        assert np.array_equal(pop.qutrits, full.qutrits[rot])
        seen[slots] = True
    assert seen.all()


def _ipc_worker(rank, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_1809_11134_b200.distributed import sharded_qeqea
    from paper_1809_11134_b200.engine import PopulationConfig
    from paper_1809_11134_b200.fitness import TargetSpec

    T = random_unitary(16, np.random.default_rng(77))
    cfg = PopulationConfig(number_of_wires=4, size_of_individual=16, size_of_population=40,
                           max_generations=20, target_fitness=1.0)
    run = sharded_qeqea(cfg, TargetSpec("haar", 4, T), 5, transport="p2p")
    rec = run.steps(20)
    q.put((rank, rec["gen_best"].tolist(), rec["gen_mean"].tolist(), run.stop_reason))
    run.engine.close()
    dist.destroy_process_group()


def test_p2p_transport_over_cuda_ipc_two_processes():
    """Two processes on the one GPU map each other's exchange buffers with
    CUDA IPC (isq_qeqea_ipc_export / _ipc_open) and run the peer transport,
    ordered by host barriers (gloo): the trajectory equals one rank's."""
    import socket

    import torch.multiprocessing as mp

    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get() for _ in range(2)])
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    T = random_unitary(16, np.random.default_rng(77))
    cfg = PopulationConfig(number_of_wires=4, size_of_individual=16, size_of_population=40,
                           max_generations=20, target_fitness=1.0)
    ref = QeqeaEngine(cfg, TargetSpec("haar", 4, T), 5).steps(20)
    for rank, gb, gm, stop in res:
        assert gb == list(ref["gen_best"]) and gm == list(ref["gen_mean"]), rank
        assert stop == "generation-limit"


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ga_matches_single_rank(world):
    """GA sharding (replicated genomes, genome shards scored per rank, fitness
    all-gathered) reproduces the single-rank GA bit for bit."""
    import torch

    from paper_1809_11134_b200.distributed import DeviceGaOps, ShardedRunner
    from paper_1809_11134_b200.fitness import target_matrix
    from paper_1809_11134_b200.ga import GaConfig, GaEngine

    cfg = GaConfig(number_of_wires=3, size_of_individual=16, population=61, max_generations=25)
    t = target_matrix("Toffoli")
    ref = GaEngine(cfg, t, seed=8)
    rrec = ref.steps(25)
    comm = LockstepComm(world)
    engines = [GaEngine(cfg, t, seed=8, rank=r, world=world, max_batch=8) for r in range(world)]
    out = [None] * world

    def worker(r):
        runner = ShardedRunner(DeviceGaOps(engines[r]), comm=comm.rank_view(r))
        out[r] = runner.steps(25)
        torch.cuda.synchronize()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for r in range(world):
        assert np.array_equal(out[r]["gen_best"], rrec["gen_best"]), r
        assert np.array_equal(out[r]["gen_mean"], rrec["gen_mean"]), r
        c, th_ = engines[r].genome_arrays()
        rc, rt = ref.genome_arrays()
        assert np.array_equal(c, rc) and np.array_equal(th_, rt)


def test_sharded_engines_pickle_and_resume():
    """Checkpoint / resume of a sharded run (engine.py:301-304): each rank
    pickles its own bank shard; the resumed ranks continue bit-identically."""
    import pickle

    import torch

    from paper_1809_11134_b200.distributed import DeviceQeqeaOps, ShardedRunner
    from paper_1809_11134_b200.engine import PopulationConfig, QeqeaEngine
    from paper_1809_11134_b200.fitness import TargetSpec

    T = random_unitary(8, np.random.default_rng(31))
    cfg = PopulationConfig(number_of_wires=3, size_of_individual=16, size_of_population=48,
                           max_generations=40, target_fitness=1.0)
    spec = TargetSpec("haar", 3, T)
    ref = QeqeaEngine(cfg, spec, seed=6).steps(40)

    def drive(engines, gens, comm):
        out = [None] * len(engines)

        def worker(r):
            out[r] = ShardedRunner(DeviceQeqeaOps(engines[r], "p2p"), comm=comm.rank_view(r)).steps(gens)
            torch.cuda.synchronize()

        ths = [threading.Thread(target=worker, args=(r,)) for r in range(len(engines))]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        return out

    engines = [QeqeaEngine(cfg, spec, seed=6, rank=r, world=2, max_batch=8) for r in range(2)]
    first = drive(engines, 15, LockstepComm(2))
    blobs = [pickle.dumps(e) for e in engines]
    for e in engines:
        e.close()
    resumed = [pickle.loads(b) for b in blobs]
    assert all(e.generation == 15 for e in resumed)
    second = drive(resumed, 25, LockstepComm(2))
    for r in range(2):
        gb = np.concatenate([first[r]["gen_best"], second[r]["gen_best"]])
        gm = np.concatenate([first[r]["gen_mean"], second[r]["gen_mean"]])
        assert np.array_equal(gb, ref["gen_best"]) and np.array_equal(gm, ref["gen_mean"]), r
