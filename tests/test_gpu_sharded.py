"""Multi-rank sharding on ONE B200 (SURVEY.md 4.5 "simulated ranks"):
SimulatedRanks runs the real device engine as 2 and 4 contiguous slice shards in one
process, the boundary hand-off as device-to-device copies, the coarse chain shard after
shard (no kernel waits on another).  The iterates, increments and stopping iteration must
be bit-identical to the single-engine run -- the chain adds no arithmetic."""

import numpy as np
import pytest

from oracle import chp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_14074_b200 import distributed, grid, parareal
    return parareal, grid, distributed


def _single(P, G, g, var, part, eps, u0s, max_iter):
    from paper_2304_14074_b200.engine import PararealEngine
    f, c = P.propagator_pair(P.AlgorithmVariant(var), part, eps)
    eng = PararealEngine(g, f, c, part.num_slices, part.fine_steps, batch=len(u0s))
    eng.load([G.Field(g, u) for u in u0s])
    eng.run(max_iter=max_iter)
    return eng


def _sharded(P, G, D, g, var, part, eps, u0s, world, max_iter, hop=False):
    f, c = P.propagator_pair(P.AlgorithmVariant(var), part, eps)
    sim = D.SimulatedRanks(g, f, c, part.num_slices, part.fine_steps, world, batch=len(u0s),
                           hop=hop)
    sim.load([G.Field(g, u) for u in u0s])
    sim.run(max_iter=max_iter)
    return sim


@pytest.mark.parametrize("case", ["c3_trunc", "c5_trunc", "c2_trunc_batch"])
@pytest.mark.parametrize("world,hop", [(2, False), (4, False), (2, True), (4, True)])
def test_simulated_ranks_bit_identical(M, case, world, hop):
    """hop=True: the boundaries travel by the device-initiated hop of include/chp.h chp_hop
     -- stores fused into the cooperative 2D coarse kernel's last
    correction (c3/c5) or a put kernel after the 1D sweep (c2), flag release, stream wait,
    take and ack -- instead of mailbox copies; still bit-identical."""
    P, G, D = M
    if case == "c3_trunc":        # config 3's grid, eps, dt, dT and u0; first 8 slices
        c = O.CONFIGS[3]
        g = G.SpatialGrid(2, c["nx"])
        dT = c["T"] / c["N"]
        part, eps, var = P.TimePartition(8 * dT, 8, c["J"]), c["eps"], "pa3"
        u0s, max_iter = [O.initial_condition(3)], 4
    elif case == "c5_trunc":      # config 5's grid and parameters; first 4 slices
        c = O.CONFIGS[5]
        g = G.SpatialGrid(2, c["nx"])
        dT = c["T"] / c["N"]
        part, eps, var = P.TimePartition(4 * dT, 4, 16), c["eps"], "pa3"
        u0s, max_iter = [O.initial_condition(5)], 3
    else:                         # config 2's 1D NPA1 with 3 ICs; first 8 slices
        c = O.CONFIGS[2]
        g = G.SpatialGrid(1, c["nx"])
        dT = c["T"] / c["N"]
        part, eps, var = P.TimePartition(8 * dT, 8, c["J"]), c["eps"], "npa1"
        u0s, max_iter = [O.initial_condition(2, b) for b in range(3)], 10
    one = _single(P, G, g, var, part, eps, u0s, max_iter)
    sim = _sharded(P, G, D, g, var, part, eps, u0s, world, max_iter, hop)
    sh0 = sim.shards[0]
    conv = sh0.converged
    assert conv == one.converged_at
    inc_one = np.array(one.increments)
    inc_sim = np.array(sh0.incs)
    assert inc_one.shape == inc_sim.shape
    assert np.array_equal(inc_one, inc_sim)
    for i in range(len(u0s)):
        assert np.array_equal(sim.iterates(i), one.iterates_host(i)), i


@pytest.mark.parametrize("dim", [1, 2])
def test_chunked_sweeps_bit_identical_on_device(M, dim):
    """chunked fine/coarse sweeps (the e2e step's copy pipelining) against one
    sweep on the DEVICE engine (k1d_coarse_sweep / k2d_coarse2): the increment accumulates
    across the chunk launches and the changed flag of the first slice of a chunk survives
    between them, so U, G, changed and the increments must be bit-identical."""
    import torch
    P, G, D = M
    if dim == 1:
        g = G.SpatialGrid(1, 129)
        part, eps = P.TimePartition(0.08, 8, 16), 0.05
        u0 = 0.1 * np.sin(2 * np.pi * np.arange(1, 128) / 128) + \
            np.random.default_rng(3).uniform(-0.01, 0.01, 127)
    else:
        g = G.SpatialGrid(2, 65)
        part, eps = P.TimePartition(0.04, 8, 8), 0.03
        u0 = np.random.default_rng(4).uniform(-0.05, 0.05, g.interior_count)
    f, c = P.propagator_pair(P.AlgorithmVariant.PA3, part, eps)

    def run(chunked):
        sh = D.ShardedParareal(g, f, c, part.num_slices, part.fine_steps)
        sh.load(G.Field(g, u0))
        sh.coarse_init()
        incs = []
        for _ in range(4):
            if chunked:
                incs.append(sh.iterate(fine_chunks=[(0, 3, None), (3, 8, None)],
                                       coarse_chunks=[(0, 2), (2, 5), (5, 8)]))
            else:
                incs.append(sh.iterate())
        torch.cuda.synchronize()
        e = sh.eng
        return (e.U.cpu().numpy().copy(), e.G.cpu().numpy().copy(),
                e.changed.cpu().numpy().copy(), np.array(incs))

    a, b = run(False), run(True)
    for x, y, name in zip(a, b, ("U", "G", "changed", "increments")):
        assert np.array_equal(x, y), name
