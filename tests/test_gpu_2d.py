"""2D parity on the B200 (configs 3-5).

The reference solves the 2D systems with SuperLU (COLAMD), whose rounding no
other solver reproduces; the GPU uses the exact DST-I diagonalisation for
LINEAR_B and DST-preconditioned CG for the variable-coefficient solves.
Tolerances (tier T2): per propagation <= 1e-12 relative
max-norm against the CPU-DST oracle (the reference engine with the spectral
solver injected), and <= 1e-10 against the unmodified reference (SuperLU)
over short propagations.
"""

import numpy as np
import pytest

from oracle import chp_oracle as O

pytestmark = pytest.mark.gpu

SPECTRAL = O.Knobs(cube="numpy", spectral=True)
FAITHFUL = O.Knobs(cube="numpy")


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_14074_b200 import grid, parareal, schemes
    return grid, schemes, parareal


@pytest.mark.parametrize("nx,eps,dt,steps", [(9, 0.1, 1e-3, 3), (17, 0.05, 2.0 ** -10, 8),
                                             (33, 0.05, 2.0 ** -9, 8), (65, 0.03, 2.0 ** -12, 16),
                                             (129, 0.02, 2.0 ** -13, 4),
                                             (257, 0.02, 2.0 ** -14, 8)])
def test_linear_b_vs_spectral_oracle(M, nx, eps, dt, steps):
    G, S, _ = M
    g = G.SpatialGrid(2, nx)
    v = np.random.default_rng(nx).uniform(-0.9, 0.9, g.interior_count)
    got = S.propagate(G.Field(g, v), S.PropagatorSpec(S.Scheme.LINEAR_B, dt, eps), steps).values
    mesh = O.Mesh(2, nx)
    want = O.advance(mesh, v, O.LINEAR_B, dt, eps, steps, SPECTRAL)
    assert rel(got, want) < 1e-12
    if nx <= 65:
        ref = O.advance(mesh, v, O.LINEAR_B, dt, eps, steps, FAITHFUL)
        assert rel(got, ref) < 1e-10


def test_linear_b_golden_reference_steps(M, golden):
    G, S, _ = M
    z = golden("steps.npz")
    ci = 0
    while f"in_{ci}" in z:
        dim, nx, eps, dt = z[f"meta_{ci}"]
        if int(dim) == 2:
            g = G.SpatialGrid(2, int(nx))
            for steps in (1, 8):
                got = S.propagate(G.Field(g, z[f"in_{ci}"]),
                                  S.PropagatorSpec(S.Scheme.LINEAR_B, dt, eps), steps).values
                assert rel(got, z[f"b{steps}_{ci}"]) < 1e-11, (ci, steps)
        ci += 1


def test_linear_b_batched_index_and_zero(M):
    import torch
    G, S, _ = M
    g = G.SpatialGrid(2, 33)
    rng = np.random.default_rng(1)
    flat = rng.uniform(-0.5, 0.5, (5, g.interior_count))
    src = torch.stack([G.to_device_layout(g, torch.tensor(f, device="cuda")) for f in flat])
    src[3].zero_()
    out = torch.full_like(src, 7.0)
    idx = torch.tensor([3, 1, 4], dtype=torch.int32, device="cuda")
    spec = S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-3, 0.05)
    S.propagate_batch(g, spec, 5, src, out, sys_index=idx)
    mesh = O.Mesh(2, 33)
    for k in (1, 4):
        got = G.from_device_layout(g, out[k]).cpu().numpy()
        assert rel(got, O.advance(mesh, flat[k], O.LINEAR_B, 1e-3, 0.05, 5, SPECTRAL)) < 1e-12
        assert float(out[k][:, 0].abs().max()) == 0.0       # pad column written as 0
    assert float(out[3].abs().max()) == 0.0                 # zero is a fixed point
    assert float(out[0].min()) == 7.0 and float(out[2].min()) == 7.0


def test_linear_b_nonfinite(M):
    G, S, _ = M
    g = G.SpatialGrid(2, 17)
    v = np.full(g.interior_count, 1e150)
    with pytest.raises(ValueError, match="non-finite"):
        S.propagate(G.Field(g, v), S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-3, 0.1), 4)


def test_linear_b_config5_grid_short(M):
    """Config 5 grid (1023^2), eps, dt: 4 fine steps vs the CPU-DST oracle."""
    G, S, _ = M
    g = G.SpatialGrid(2, 1025)
    v = O.initial_condition(5)
    dt = 2.0 / 512 / 256
    got = S.propagate(G.Field(g, v), S.PropagatorSpec(S.Scheme.LINEAR_B, dt, 0.01), 4).values
    want = O.advance(O.Mesh(2, 1025), v, O.LINEAR_B, dt, 0.01, 4, SPECTRAL)
    assert rel(got, want) < 1e-12


@pytest.mark.parametrize("nx,eps,dt", [(9, 0.1, 1e-3), (17, 0.05, 2.0 ** -10), (33, 0.02, 2.0 ** -7),
                                       (65, 0.015, 2.0 ** -8), (257, 0.02, 2.0 ** -7)])
def test_linear_a_pcg_vs_reference(M, nx, eps, dt):
    """2D LINEAR_A: matrix-free DST-preconditioned CG vs the reference's SuperLU."""
    G, S, _ = M
    g = G.SpatialGrid(2, nx)
    v = np.random.default_rng(nx + 1).uniform(-1.0, 1.0, g.interior_count)
    got = S.propagate(G.Field(g, v), S.PropagatorSpec(S.Scheme.LINEAR_A, dt, eps), 2).values
    want = O.advance(O.Mesh(2, nx), v, O.LINEAR_A, dt, eps, 2, FAITHFUL)
    assert rel(got, want) < 1e-11


@pytest.mark.parametrize("nx,eps,dt", [(17, 0.05, 2.0 ** -12), (33, 0.05, 2.0 ** -12),
                                       (65, 0.015, 2.0 ** -15), (257, 0.015, 2.0 ** -15)])
def test_newton_2d_vs_reference(M, nx, eps, dt):
    """3 Newton steps (steps 2 and 3 warm-start the batched PCG from the previous
    solve) vs the reference's SuperLU: same Newton counts, <= 1e-10."""
    G, S, _ = M
    g = G.SpatialGrid(2, nx)
    v = np.random.default_rng(nx + 2).uniform(-0.9, 0.9, g.interior_count)
    stats = S.NewtonStats()
    got = S.propagate(G.Field(g, v), S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, dt, eps), 3,
                      stats).values
    cnt = O.NewtonCounter()
    want = O.advance(O.Mesh(2, nx), v, O.EYRE, dt, eps, 3, FAITHFUL, cnt)
    assert rel(got, want) < 1e-10
    assert stats.steps == 3 and stats.total_iterations == cnt.total


def test_golden_2d_steps_a_and_newton(M, golden):
    G, S, _ = M
    z = golden("steps.npz")
    ci = 0
    while f"in_{ci}" in z:
        dim, nx, eps, dt = z[f"meta_{ci}"]
        if int(dim) == 2:
            g = G.SpatialGrid(2, int(nx))
            u = G.Field(g, z[f"in_{ci}"])
            got = S.propagate(u, S.PropagatorSpec(S.Scheme.LINEAR_A, dt, eps), 8).values
            assert rel(got, z[f"a8_{ci}"]) < 1e-10, ci
            if f"n8_{ci}" in z:
                got = S.propagate(u, S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, dt, eps), 8).values
                assert rel(got, z[f"n8_{ci}"]) < 1e-9, ci
        ci += 1


@pytest.mark.parametrize("var", ["pa3", "npa1"])
def test_twod_small_parareal_vs_reference(M, golden, var):
    G, S, P = M
    z = golden("twod_small.npz")
    g = G.SpatialGrid(2, 33)
    T, Nsl, J = (0.05, 4, 16) if var == "pa3" else (0.02, 4, 8)
    tr = P.run(G.Field(g, z["u0"]), P.AlgorithmVariant(var), P.TimePartition(T, Nsl, J), 0.05,
               stop="increment")
    assert tr.converged_at == int(z[f"{var}_k"][0])
    from paper_2304_14074_b200.engine import PararealEngine
    f, c = P.propagator_pair(P.AlgorithmVariant(var), P.TimePartition(T, Nsl, J), 0.05)
    eng = PararealEngine(g, f, c, Nsl, J)
    eng.load([G.Field(g, z["u0"])])
    eng.run()
    assert eng.converged_at[0] == int(z[f"{var}_k"][0])
    assert rel(eng.iterates_host(), z[f"{var}_U"]) < 1e-10


def test_config3_truncated_pa3(M):
    """Config 3 grid/eps/dt/IC, first 4 slices: same k as the CPU-DST oracle
    (spectral LINEAR_B, SuperLU LINEAR_A), iterates within 1e-10."""
    G, S, P = M
    g = G.SpatialGrid(2, 257)
    u0 = O.initial_condition(3)
    dT = 0.5 / 64
    part = P.TimePartition(4 * dT, 4, 128)
    from paper_2304_14074_b200.engine import PararealEngine
    f, c = P.propagator_pair(P.AlgorithmVariant.PA3, part, 0.02)
    eng = PararealEngine(g, f, c, 4, 128)
    eng.load([G.Field(g, u0)])
    eng.run()
    ref = O.parareal(O.Mesh(2, 257), u0, "pa3", part.total_time, 4, 128, 0.02, SPECTRAL)
    assert eng.converged_at[0] == ref.k
    assert rel(eng.iterates_host(), ref.iterates) < 1e-10


def test_config4_truncated_npa1(M, golden):
    """Config 4 grid (511^2), eps, fine/coarse steps and seeded u0, first 4 slices
    (NPA1: Newton fine steps to 1e-10 with the batched PCG, LINEAR_A coarse sweep
    in the cooperative kernel) against the CPU-DST/PCG oracle
    (tools/oracle_c4_trunc.py): same k, final iterates within 1e-10, Newton totals
    equal up to borderline flips."""
    G, S, P = M
    z = golden("config4_trunc.npz")
    g = G.SpatialGrid(2, 513)
    u0 = O.initial_condition(4)
    dT = 0.5 / 128
    part = P.TimePartition(4 * dT, 4, 128)
    from paper_2304_14074_b200.engine import PararealEngine
    f, c = P.propagator_pair(P.AlgorithmVariant.NPA1, part, 0.015)
    eng = PararealEngine(g, f, c, 4, 128)
    eng.load([G.Field(g, u0)])
    eng.run()
    assert eng.converged_at[0] == int(z["k"][0])
    assert rel(eng.iterates_host()[-1], z["U_end"]) < 1e-10
    nt = int(z["newton_total"][0])
    assert abs(eng.newton.total_iterations - nt) <= max(2, nt // 200)


def test_config5_truncated_pa3(M, golden):
    """Config 5 grid (1023^2), eps, fine/coarse steps and seeded u0, first 4 slices
    (PA3: LINEAR_B passes, LINEAR_A coarse sweep in the cooperative kernel at
    N = 1024) against the CPU-DST/PCG oracle (tools/oracle_c5_trunc.py): same k,
    increments within 1e-9, final iterate (every 8th point) within 1e-9.  The
    final iterate is the serial fine solution after 1024 LINEAR_B steps: the GPU
    sits 3.2e-10 from the DST oracle (5.7e-14 per step), while the reference's
    own SuperLU arithmetic sits 6.0e-8 from it (E_env, tools/env_c5_trunc.py) --
    SURVEY.md 8(c) T3 bound max(1e-10, E_env)."""
    G, S, P = M
    z = golden("config5_trunc.npz")
    g = G.SpatialGrid(2, 1025)
    u0 = O.initial_condition(5)
    dT = 2.0 / 512
    part = P.TimePartition(4 * dT, 4, 256)
    from paper_2304_14074_b200.engine import PararealEngine
    f, c = P.propagator_pair(P.AlgorithmVariant.PA3, part, 0.01)
    eng = PararealEngine(g, f, c, 4, 256)
    eng.load([G.Field(g, u0)])
    eng.run()
    assert eng.converged_at[0] == int(z["k"][0])
    inc = np.array([x[0] for x in eng.increments])
    assert np.max(np.abs(inc - z["increments"]) / np.maximum(np.abs(z["increments"]), 1e-300)
                  * (z["increments"] > 0)) < 1e-9
    err = rel(eng.iterates_host()[-1][::8], z["U_end_sub"])
    assert err < 1e-9
    assert err < max(1e-10, float(z["E_env_superlu_vs_dst"][0]))


def test_config5_accuracy_vs_long_double_truth(M, golden):
    """SURVEY.md 8(c) tier T3 at the config-5 grid: 256 and 1024 LINEAR_B steps of config
    5's seeded u0 (1024 steps = the converged truncated config-5 iterate above) against
    an x87 long-double truth (tools/linb_truth.py -> tests/golden/config5_truth.npz).
    The GPU must be no less accurate than the fp64 CPU-DST oracle and far more accurate
    than the reference's own SuperLU arithmetic: no fp64 path meets 1e-10 against the
    truth over 1024 spinodal steps (the oracle itself is ~5e-10 away), which is why the
    truncated test above cannot ask 1e-10 of the GPU-vs-oracle difference."""
    import os
    G, S, P = M
    if not os.path.exists(os.path.join(os.path.dirname(__file__), "golden", "config5_truth.npz")):
        pytest.skip("truth fixture not generated")
    z = golden("config5_truth.npz")
    g = G.SpatialGrid(2, 1025)
    u0 = O.initial_condition(5)
    spec = S.PropagatorSpec(S.Scheme.LINEAR_B, 2.0 / 512 / 256, 0.01)
    v = G.Field(g, u0)
    v256 = S.propagate(v, spec, 256)
    v1024 = S.propagate(v256, spec, 768).values
    for k, got in ((256, v256.values), (1024, v1024)):
        truth = z[f"truth{k}_sub8"]
        err = rel(got[::8], truth)
        assert err <= float(z[f"oracle_dst_{k}_sub8"][0]), (k, err)
        assert err * 10 <= float(z[f"reference_superlu_{k}_sub8"][0]), (k, err)
    assert rel(v1024[::8], z["truth1024_sub8"]) < 1e-9


def test_coarse_sweep_rejects_misaligned_fields(M):
    """The 2D sweep moves fields as 16-byte words: a field buffer that is only 8-byte
    aligned is refused with CHP_ERR_ARG (ValueError), not read through misaligned loads."""
    import torch
    grid, schemes, parareal = M
    from paper_2304_14074_b200.engine import PararealEngine
    g = grid.SpatialGrid(2, 33)
    part = parareal.TimePartition(0.02, 4, 2)
    f, c = parareal.propagator_pair(parareal.AlgorithmVariant.PA3, part, 0.05)
    eng = PararealEngine(g, f, c, 4, 2)
    eng.load([grid.Field(g, np.random.default_rng(0).uniform(-0.05, 0.05, g.interior_count))])
    good = eng.U
    buf = torch.zeros(good.numel() + 1, dtype=good.dtype, device=good.device)
    eng.U = buf[1:].view(good.shape)
    eng.U.copy_(good)
    assert eng.U.data_ptr() % 16 == 8
    with pytest.raises(ValueError, match="16-byte aligned"):
        eng.coarse_init()
    eng.U = good
    eng.coarse_init()                      # the aligned buffer still works
    assert bool(torch.isfinite(eng.U).all())
