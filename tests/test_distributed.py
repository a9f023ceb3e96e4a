"""Sharded (multi-rank) Parareal chain logic on CPU: world_size 2 over gloo.

The device engine is swapped for a host engine that implements the same
interface with the CPU oracle's propagators (test infrastructure), so the
send/recv chain, the changed-flag hand-off and the all-reduce of the increment
are exercised without a GPU.  Iterates must be bit-identical to the
single-process oracle run, with the same iteration count.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import chp_oracle as O

KN = O.Knobs(cube="exact")
_SCHEME = {"linear-a": O.LINEAR_A, "linear-b": O.LINEAR_B, "nonlinear-eyre": O.EYRE}


class HostEngine:
    """CPU stand-in for engine.PararealEngine (same attributes / semantics, any batch)."""

    def __init__(self, grid, fine, coarse, L, J, batch=1, device=None):
        self.mesh = O.Mesh(grid.dim, grid.nodes_per_axis)
        self.fine, self.coarse, self.L, self.J, self.B = fine, coarse, L, J, batch
        n = self.mesh.size
        self.U = torch.zeros((batch, L + 1, n), dtype=torch.float64)
        self.G = torch.zeros_like(self.U)
        self.F = torch.zeros_like(self.U)
        self.changed = torch.zeros((batch, L + 1), dtype=torch.uint8)
        self.inc = torch.zeros(batch, dtype=torch.float64)

    def _step(self, spec, v, steps):
        return O.advance(self.mesh, v, _SCHEME[spec.scheme.value], spec.dt, spec.eps, steps, KN)

    def load(self, u0s):
        for i, f in enumerate(u0s):
            self.U[i, 0] = torch.as_tensor(f.values)

    def fine_sweep(self, flags):
        for i in range(self.B):
            if flags[i, 0] & 2:
                continue
            for n in range(self.L):
                if flags[i, n] & 1:
                    self.F[i, n] = torch.as_tensor(self._step(self.fine, self.U[i, n].numpy(),
                                                              self.J))

    def coarse_range(self, mode, n0, n1):
        for i in range(self.B):
            U, G, F, ch = self.U[i].numpy(), self.G[i].numpy(), self.F[i].numpy(), self.changed[i]
            if mode == 1 and ch[0] & 2:
                continue
            for n in range(n0, n1):
                if mode == 0:
                    U[n + 1] = self._step(self.coarse, U[n], 1)
                    G[n] = U[n + 1]
                    continue
                g = self._step(self.coarse, U[n], 1) if ch[n] & 1 else G[n].copy()
                new = (g + F[n]) - G[n]
                ch[n + 1] = (ch[n + 1] & 2) | int(not np.array_equal(new.view(np.int64),
                                                                     U[n + 1].view(np.int64)))
                self.inc[i] = max(float(self.inc[i]), float(np.max(np.abs(new - U[n + 1]))))
                U[n + 1] = new
                G[n] = g

    def check_status(self):
        pass

    def iterates_host(self, i):
        return self.U[i].numpy().copy()


def _worker(rank, world, port, var, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.distributed import ShardedParareal
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    g = SpatialGrid(1, 17)
    part = P.TimePartition(0.05, 4, 4)
    f, c = P.propagator_pair(P.AlgorithmVariant(var), part, 0.1)
    sh = ShardedParareal(g, f, c, 4, 4, rank=rank, world=world, engine_factory=HostEngine)
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, 15)
    sh.load(Field(g, u0))
    k = sh.run()
    out_q.put((rank, k, sh.increments, sh.local_iterates()))
    dist.destroy_process_group()


@pytest.mark.parametrize("var", ["pa3", "npa1"])
def test_two_rank_chain_bit_identical(var):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, var, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, 15)
    ref = O.parareal(O.Mesh(1, 17), u0, var, 0.05, 4, 4, 0.1, KN)
    assert res[0][1] == res[1][1] == ref.k
    assert np.array_equal(np.array(res[0][2]), np.array(ref.increments))
    U = np.concatenate([res[0][3], res[1][3]])
    assert np.array_equal(U, ref.iterates)


def test_shard_bounds():
    from paper_2304_14074_b200.distributed import shard
    assert shard(512, 8, 3) == (192, 256)
    with pytest.raises(ValueError):
        shard(10, 4, 0)


def _worker_defer(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.distributed import ShardedParareal
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    g = SpatialGrid(1, 17)
    part = P.TimePartition(0.05, 4, 4)
    f, c = P.propagator_pair(P.AlgorithmVariant("pa3"), part, 0.1)
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, 15)
    res = []
    for mode in ("sync", "defer", "chunked"):
        sh = ShardedParareal(g, f, c, 4, 4, rank=rank, world=world, engine_factory=HostEngine)
        sh.load(Field(g, u0))
        sh.coarse_init()
        seen = []
        for _ in range(3):
            if mode == "chunked":     # the e2e step's slice-chunked fine and coarse sweeps
                sh.iterate(force_all=True, defer=True, fine_chunks=[(0, 1, None), (1, 2, None)],
                           coarse_chunks=[(0, 1), (1, 2)],
                           on_coarse_chunk=lambda n0, n1: seen.append((n0, n1)))
            else:
                sh.iterate(force_all=True, defer=(mode == "defer"))
        sh.flush()
        if mode == "chunked":
            assert seen == [(0, 1), (1, 2)] * 3
        res.append((sh.k, list(sh.increments), sh.local_iterates()))
    out_q.put((rank, res))
    dist.destroy_process_group()


def test_two_rank_deferred_increments_match():
    """iterate(defer=True) (the bench's pipelined step) and the e2e step's
    slice-chunked sweeps compute exactly what the synchronous iteration computes:
    same iterates bit for bit, same increments."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker_defer, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (sync, deferred, chunked) in out:
        for other in (deferred, chunked):
            assert sync[0] == other[0] == 3
            assert sync[1] == other[1]
            assert np.array_equal(sync[2], other[2])


def _worker_batch(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.distributed import ShardedParareal
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    g = SpatialGrid(1, 17)
    part = P.TimePartition(0.05, 4, 4)
    f, c = P.propagator_pair(P.AlgorithmVariant("npa1"), part, 0.1)
    u0s = [np.random.default_rng(s).uniform(-0.5, 0.5, 15) for s in (3, 4, 5)]
    res = []
    for pipelined in (False, True):
        sh = ShardedParareal(g, f, c, 4, 4, rank=rank, world=world, engine_factory=HostEngine,
                             batch=3)
        sh.load([Field(g, u) for u in u0s])
        conv = sh.run(pipelined=pipelined)
        res.append((list(conv), [x.tolist() for x in sh.incs],
                    [sh.local_iterates(i) for i in range(3)]))
    out_q.put((rank, res))
    dist.destroy_process_group()


def test_two_rank_batched_ics_and_pipelined_run():
    """Sharded Parareal with 3 ICs per rank (config-2 style): per-IC
    increment stop, converged ICs frozen on every rank, boundary hand-off of all ICs;
    the pipelined run() (next fine sweep issued before the increment test) stops at the
    same k with the same iterates as the synchronous loop and as the oracle per IC."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker_batch, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u0s = [np.random.default_rng(s).uniform(-0.5, 0.5, 15) for s in (3, 4, 5)]
    refs = [O.parareal(O.Mesh(1, 17), u, "npa1", 0.05, 4, 4, 0.1, KN) for u in u0s]
    for mode in range(2):
        conv = out[0][1][mode][0]
        assert conv == out[1][1][mode][0] == [r.k for r in refs]
        for i, r in enumerate(refs):
            U = np.concatenate([out[0][1][mode][2][i], out[1][1][mode][2][i]])
            assert np.array_equal(U, r.iterates), (mode, i)
            incs = [x[i] for x in out[0][1][mode][1]][:r.k]
            assert np.array_equal(np.array(incs), np.array(r.increments)), (mode, i)


@pytest.mark.parametrize("world", [2, 4])
def test_simulated_ranks_host_engine(world):
    """SimulatedRanks (one process, loopback hand-off) with the host engine: the same
    k and iterates as the single-process oracle."""
    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.distributed import SimulatedRanks
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    g = SpatialGrid(1, 17)
    part = P.TimePartition(0.1, 8, 4)
    f, c = P.propagator_pair(P.AlgorithmVariant("pa3"), part, 0.1)
    u0 = np.random.default_rng(3).uniform(-0.5, 0.5, 15)
    sim = SimulatedRanks(g, f, c, 8, 4, world, engine_factory=HostEngine)
    sim.load(Field(g, u0))
    k = sim.run()
    ref = O.parareal(O.Mesh(1, 17), u0, "pa3", 0.1, 8, 4, 0.1, KN)
    assert k == ref.k
    assert np.array_equal(np.array(sim.increments), np.array(ref.increments))
    assert np.array_equal(sim.iterates(), ref.iterates)
