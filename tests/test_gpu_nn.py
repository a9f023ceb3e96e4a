"""Neumann-Neumann fine step (Scheme.NN_LINEAR_A, reference ddm.py) on the B200.

The kernel solves the same mixed (u, v) subdomain systems as the reference but
by 2x2 block elimination instead of dense LAPACK LU, so it is compared by
tolerance: the converged field within ATOL of the reference's own output
(tests/golden/nn_small.npz, pinned to the oracle bit for bit by
tests/test_oracle_nn.py), the same interface-sweep count per step, the same
Parareal increments to 1e-9.
"""

import numpy as np
import pytest

from oracle import chp_oracle as O

pytestmark = pytest.mark.gpu

# The interface iteration stops at trace increments <= 1e-10 (cell-weighted
# L2); two runs with different rounding stop within a few of those of the
# fixed point.  Measured: <= 2e-15 (profiles/r01_nn_probe.json); 1e-9 is the bar.
ATOL = 1e-9
CASES = ["c65_s4", "c65_s4_warm", "c65_s2_th40", "c257_s8", "c1025_s8", "c129_s16_warm"]


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_14074_b200 import ddm, grid, parareal, schemes
    return ddm, grid, parareal, schemes


def setup(M, z, name):
    ddm, grid, _, _ = M
    nx, S, th, tol, mi, warm, dt, eps, steps = z[f"{name}/params"]
    g = grid.SpatialGrid(dim=1, nodes_per_axis=int(nx))
    p = ddm.NNParams(n_subdomains=int(S), theta=float(th), tol=float(tol), max_iter=int(mi),
                     warm_start=bool(warm))
    return g, p, float(dt), float(eps), int(steps)


@pytest.mark.parametrize("name", CASES)
def test_nn_propagate_vs_reference(M, golden, name):
    ddm, grid, _, schemes = M
    z = golden("nn_small.npz")
    g, p, dt, eps, steps = setup(M, z, name)
    spec = ddm.nn_propagator(ddm.Decomposition(g, p.n_subdomains), p, dt, eps)
    out = schemes.propagate(grid.Field(g, z[f"{name}/u0"]), spec, steps)
    err = float(np.max(np.abs(out.values - z[f"{name}/out"])))
    assert err < ATOL, err


@pytest.mark.parametrize("name", CASES)
def test_nn_solve_sweeps_and_traces(M, golden, name):
    """Per-step interface sweep counts equal the reference's; final traces agree."""
    ddm, grid, _, _ = M
    z = golden("nn_small.npz")
    g, p, dt, eps, steps = setup(M, z, name)
    dec = ddm.Decomposition(g, p.n_subdomains)
    cur, tr, sweeps = grid.Field(g, z[f"{name}/u0"]), None, []
    for _ in range(steps):
        cur, ftr = ddm._nn_solve(cur, dec, p, dt, eps, traces=tr)
        sweeps.append(ftr.iterations)
        if p.warm_start:
            tr = ddm.InterfaceTraces(g=ftr.g.copy(), h=ftr.h.copy())
    assert sweeps == list(z[f"{name}/sweeps"])
    assert np.max(np.abs(ftr.g - z[f"{name}/g"])) < ATOL
    assert np.max(np.abs(ftr.h - z[f"{name}/h"])) < 1e3 * ATOL   # v = -mu scale
    assert np.max(np.abs(cur.values - z[f"{name}/out"])) < ATOL


@pytest.mark.parametrize("S,nx,nsys,dt", [(4, 65, 37, 2.0 ** -12), (8, 257, 9, 2.0 ** -12),
                                          (2, 33, 70, 2.0 ** -12), (32, 129, 3, 2.0 ** -16)])
def test_nn_batched_with_index_vs_oracle(M, S, nx, nsys, dt):
    """Many systems per launch (warp segments of next_pow2(S) lanes, partial
    warps, a sys_index permutation, in == out) against the oracle per system."""
    import torch
    ddm, grid, _, schemes = M
    g = grid.SpatialGrid(dim=1, nodes_per_axis=nx)
    p = ddm.NNParams(n_subdomains=S, max_iter=400)
    eps, steps = 0.05, 2
    rng = np.random.default_rng(S * 1000 + nsys)
    u0 = rng.uniform(-0.3, 0.3, (nsys, nx - 2))
    buf = torch.as_tensor(u0, device="cuda").contiguous()
    idx = torch.as_tensor(rng.permutation(nsys)[: nsys - 1].astype(np.int32), device="cuda")
    spec = ddm.nn_propagator(ddm.Decomposition(g, S), p, dt, eps)
    info = schemes.propagate_batch(g, spec, steps, buf, buf, sys_index=idx)
    si = schemes.read_sysinfo(info)
    assert np.all(si["status"] == 0)
    got = buf.cpu().numpy()
    mesh = O.Mesh(1, nx)
    on = set(idx.cpu().numpy().tolist())
    nn = O.NNSetup(S, p.theta, p.tol, p.max_iter)
    for s in range(nsys):
        if s not in on:
            assert np.array_equal(got[s], u0[s])      # untouched
            continue
        sw = []
        ref = O.nn_advance(mesh, u0[s], dt, eps, nn, steps, sw)
        assert np.max(np.abs(got[s] - ref)) < ATOL, s
        assert int(si["newton_total"][s]) == sum(sw)
        assert int(si["newton_max"][s]) == max(sw)


def test_nn_budget_error(M, golden):
    ddm, grid, _, _ = M
    z = golden("nn_small.npz")
    g, p, dt, eps, _ = setup(M, z, "c65_s4")
    p = ddm.NNParams(n_subdomains=4, max_iter=3)
    with pytest.raises(ddm.NNConvergenceError) as e:
        ddm.nn_time_step(grid.Field(g, z["c65_s4/u0"]), ddm.Decomposition(g, 4), p, dt, eps)
    it, gi, hi = z["fail/info"]
    assert e.value.iterations == int(it)
    assert abs(e.value.g_increment - gi) < 1e-6 * gi
    assert abs(e.value.h_increment - hi) < 1e-6 * hi


def test_nn_divergence_raises_like_reference(M):
    """32 subdomains of 4 cells at dt = 2^-12: the reference's relaxed iteration
    blows up (increments overflow to inf) and raises NNConvergenceError after
    max_iter sweeps; so must the device path."""
    ddm, grid, _, _ = M
    g = grid.SpatialGrid(dim=1, nodes_per_axis=129)
    u = grid.Field(g, np.random.default_rng(1).uniform(-0.3, 0.3, 127))
    with pytest.raises(ddm.NNConvergenceError) as e:
        ddm.nn_time_step(u, ddm.Decomposition(g, 32), ddm.NNParams(32, max_iter=400),
                         2.0 ** -12, 0.05)
    assert e.value.iterations == 400 and not e.value.g_increment <= 1e-10


def test_nn_validation(M):
    ddm, grid, _, schemes = M
    g = grid.SpatialGrid(dim=1, nodes_per_axis=65)
    with pytest.raises(ValueError, match="split evenly"):
        ddm.Decomposition(g, 5)
    with pytest.raises(ValueError, match="at least 2 mesh cells"):
        ddm.Decomposition(grid.SpatialGrid(dim=1, nodes_per_axis=9), 8)
    with pytest.raises(ValueError, match="1D only"):
        ddm.Decomposition(grid.SpatialGrid(dim=2, nodes_per_axis=9), 2)
    with pytest.raises(ValueError, match="theta"):
        ddm.NNParams(theta=1.0)
    # beyond one warp: the C ABI refuses (reference has no such limit)
    p = ddm.NNParams(n_subdomains=64)
    spec = ddm.nn_propagator(ddm.Decomposition(grid.SpatialGrid(1, 129), 64), p, 1e-4, 0.05)
    with pytest.raises(Exception, match="32 subdomains"):
        schemes.propagate(grid.Field(grid.SpatialGrid(1, 129), np.zeros(127)), spec, 1)


def test_nn_fixed_point_is_linear_a(M):
    """ddm.py:1-27: the converged NN step is the monodomain LINEAR_A step."""
    ddm, grid, _, schemes = M
    g = grid.SpatialGrid(dim=1, nodes_per_axis=257)
    u = grid.Field(g, np.random.default_rng(3).uniform(-0.5, 0.5, 255))
    dt, eps = 2.0 ** -12, 0.05
    a = schemes.step_linear_a(u, schemes.PropagatorSpec(schemes.Scheme.LINEAR_A, dt, eps))
    b = ddm.nn_time_step(u, ddm.Decomposition(g, 8), ddm.NNParams(), dt, eps)
    assert np.max(np.abs(a.values - b.values)) < 1e-9


def test_nn_parareal_vs_reference(M, golden):
    """Parareal whose fine propagator is NN_LINEAR_A (parareal.py:111-125)."""
    ddm, grid, parareal, _ = M
    z = golden("nn_small.npz")
    nx, S, eps, T, N, J = z["pr/params"]
    g = grid.SpatialGrid(dim=1, nodes_per_axis=int(nx))
    nn = ddm.NNParams(n_subdomains=int(S))
    part = parareal.TimePartition(float(T), int(N), int(J))
    var = parareal.AlgorithmVariant.PA1
    init = parareal.coarse_init(grid.Field(g, z["pr/u0"]), var, part, float(eps))
    st = parareal.PararealState(iterates=init, coarse_values=init[1:], fine_reference=[], k=0)
    incs = []
    while st.k < int(N) + 2:
        st = parareal.parareal_iteration(st, var, part, float(eps), nn=nn)
        incs.append(parareal.iterate_increment(st))
        if incs[-1] < 1e-10:
            break
    ref = z["pr/incs"]
    assert len(incs) == len(ref)
    assert np.max(np.abs(np.array(incs) - ref)) < ATOL
    U = np.array([f.values for f in st.iterates])
    assert np.max(np.abs(U - z["pr/U"])) < ATOL


def test_nn_parareal_config2_grid_vs_oracle(M):
    """NPA1-style run at config 2's grid (1D m = 1023, eps = 0.03) with the NN
    fine propagator (8 subdomains): truncated Parareal (N = 4 slices, J = 8)
    against the oracle's dense-LU restatement -- same increments to 1e-9 and
    the same iteration at which the 1e-10 increment test fires."""
    ddm, grid, parareal, _ = M
    nx, eps, T, N, J = 1025, 0.03, 2.0 ** -9, 4, 8
    g = grid.SpatialGrid(1, nx)
    u0 = np.random.default_rng(11).uniform(-0.05, 0.05, nx - 2)
    nn = ddm.NNParams(n_subdomains=8)
    part = parareal.TimePartition(T, N, J)
    var = parareal.AlgorithmVariant.PA1
    init = parareal.coarse_init(grid.Field(g, u0), var, part, eps)
    st = parareal.PararealState(iterates=init, coarse_values=init[1:], fine_reference=[], k=0)
    incs = []
    while st.k < N + 2:
        st = parareal.parareal_iteration(st, var, part, eps, nn=nn)
        incs.append(parareal.iterate_increment(st))
        if incs[-1] < 1e-10:
            break
    ref = O.parareal(O.Mesh(1, nx), u0, "pa1", T, N, J, eps, O.Knobs(nn=O.NNSetup(8)))
    assert len(incs) == len(ref.increments) and ref.k == len(incs)
    assert np.max(np.abs(np.array(incs) - np.array(ref.increments))) < ATOL
    U = np.array([f.values for f in st.iterates])
    assert np.max(np.abs(U - ref.iterates)) < ATOL


def test_spec_acceptance_9_nn_matches_linear_a(M):
    """SPEC.md acceptance 9 (first half): nn_time_step matches the monodomain
    step_linear_a to 1e-8 on 20 random states (N0 = 8, theta = 1/4, nn_tol =
    1e-10), at the paper's section-4.6 mesh h = 1/128 and fine step 1/4000."""
    ddm, grid, _, schemes = M
    g = grid.SpatialGrid(1, 129)
    dt, eps = 1.0 / 4000.0, 0.0725
    dec, p = ddm.Decomposition(g, 8), ddm.NNParams(8, 0.25, 1e-10)
    spec = schemes.PropagatorSpec(schemes.Scheme.LINEAR_A, dt, eps)
    rng = np.random.default_rng(2024)
    for _ in range(20):
        u = grid.Field(g, rng.uniform(-1.0, 1.0, 127))
        a = schemes.step_linear_a(u, spec)
        b = ddm.nn_time_step(u, dec, p, dt, eps)
        assert np.max(np.abs(a.values - b.values)) < 1e-8


def test_spec_acceptance_9_pa1_with_nn_fine(M):
    """SPEC.md acceptance 9 (second half): PA-I with the NN fine solver at the
    section-4.6 configuration (T = 1, N = 20, J = 200, h = 1/128, eps = 0.0725,
    N0 = 8, theta = 1/4) converges to tol 1e-6 against its own serial fine
    reference with an iteration count within +-1 of plain PA-I."""
    ddm, grid, parareal, _ = M
    g = grid.SpatialGrid(1, 129)
    u0 = grid.Field(g, np.random.default_rng(46).uniform(-0.05, 0.05, 127))
    part = parareal.TimePartition(1.0, 20, 200)
    var = parareal.AlgorithmVariant.PA1
    plain = parareal.run(u0, var, part, 0.0725)
    nn = parareal.run(u0, var, part, 0.0725, nn=ddm.NNParams(8, 0.25, 1e-10))
    assert plain.converged_at is not None and nn.converged_at is not None
    assert abs(plain.converged_at - nn.converged_at) <= 1, (plain.converged_at, nn.converged_at)
