"""Property tests from the reference spec on the B200."""

import numpy as np
import pytest

from oracle import chp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_14074_b200 import grid, parareal, schemes
    return grid, schemes, parareal


@pytest.mark.parametrize("dim,nx", [(1, 65), (2, 33)])
@pytest.mark.parametrize("dt", [1e-3, 1e-2, 1e-1, 1.0])
def test_gradient_stability(M, dim, nx, dt):
    """SPEC.md:478 (acceptance 4): 50 steps of every scheme never increase the
    discrete Ginzburg-Landau energy (relative slack 1e-12)."""
    G, S, _ = M
    g = G.SpatialGrid(dim, nx)
    v = np.random.default_rng(11).uniform(-0.1, 0.1, g.interior_count)
    for sch in (S.Scheme.LINEAR_A, S.Scheme.LINEAR_B, S.Scheme.NONLINEAR_EYRE):
        spec = S.PropagatorSpec(sch, dt, 0.1)
        u = G.Field(g, v)
        e_prev = G.energy(u, 0.1)
        for _ in range(50):
            u = S.propagate(u, spec, 1)
            e = G.energy(u, 0.1)
            assert e <= e_prev + 1e-12 * abs(e_prev), (sch, dt)
            e_prev = e


def test_newton_contract(M):
    """every Newton step converges to <= 1e-10 in <= 20 iterations
    (config-2 grid and step)."""
    G, S, _ = M
    g = G.SpatialGrid(1, 1025)
    stats = S.NewtonStats()
    u = G.Field(g, O.initial_condition(2, 3))
    S.propagate(u, S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, 2.0 / 64 / 512, 0.03), 64, stats)
    assert stats.steps == 64
    assert stats.max_residual <= 1e-10 and stats.max_iterations <= 20


def test_linear_b_cached_factor(M):
    """the cached constant-coefficient factor gives the same result
    as a fresh solve (here: repeated calls are bit-identical)."""
    G, S, _ = M
    g = G.SpatialGrid(1, 129)
    v = np.random.default_rng(2).uniform(-0.5, 0.5, 127)
    spec = S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-3, 0.07)
    a = S.propagate(G.Field(g, v), spec, 3).values
    b = S.propagate(G.Field(g, v), spec, 3).values
    assert np.array_equal(a, b)


@pytest.mark.parametrize("var", ["pa3", "npa1"])
def test_determinism_and_pinning(M, var):
    """repeated runs are bit-identical (fixed-order
    reductions, no FP atomics) and U_0^k stays pinned to u0."""
    G, S, P = M
    g = G.SpatialGrid(2, 33)
    u0 = np.random.default_rng(4).uniform(-0.05, 0.05, g.interior_count)
    part = P.TimePartition(0.02, 4, 8)
    outs = []
    for _ in range(2):
        tr = P.run(G.Field(g, u0), P.AlgorithmVariant(var), part, 0.05, stop="increment")
        outs.append((tr.converged_at, tr.increments, tr.records[-1].iterate_norms))
    assert outs[0] == outs[1]
    st = P.initial_state(G.Field(g, u0), P.AlgorithmVariant(var), part, 0.05)
    for _ in range(2):
        st = P.parareal_iteration(st, P.AlgorithmVariant(var), part, 0.05)
        assert np.array_equal(st.iterates[0].values, u0)


def test_fixed_point(M):
    """if U^k is the fine reference, U^{k+1} = U^k."""
    G, S, P = M
    g = G.SpatialGrid(1, 33)
    u0 = np.random.default_rng(6).uniform(-0.3, 0.3, 31)
    part = P.TimePartition(0.05, 4, 8)
    var = P.AlgorithmVariant.PA3
    ref = P.serial_fine_reference(G.Field(g, u0), var, part, 0.05)
    f, c = P.propagator_pair(var, part, 0.05)
    coarse = [S.propagate(ref[n], c, 1) for n in range(4)]
    st = P.PararealState(iterates=ref, coarse_values=coarse, fine_reference=ref, k=0)
    nxt = P.parareal_iteration(st, var, part, 0.05)
    for a, b in zip(nxt.iterates, ref):
        assert np.max(np.abs(a.values - b.values)) <= 1e-14 * (1 + np.max(np.abs(b.values)))


def test_device_field_roundtrip(M):
    import torch
    G, S, _ = M
    g = G.SpatialGrid(2, 17)
    v = torch.rand(g.interior_count, dtype=torch.float64, device="cuda")
    f = G.Field(g, v)
    assert np.array_equal(f.values, v.cpu().numpy())
    out = S.propagate(f, S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-3, 0.1), 2)
    assert out.values.shape == (g.interior_count,)
    with pytest.raises(ValueError, match="non-finite"):
        G.Field(g, torch.full((g.interior_count,), float("nan"), device="cuda"))
