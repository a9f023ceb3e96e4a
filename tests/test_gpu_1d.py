"""1D parity on the B200 (configs 1 and 2).

The 1D kernels reproduce the reference's arithmetic operation by operation
(LAPACK dpbtf2/dpbtrs and dgbtf2/dgbtrs in OpenBLAS's FMA order, scipy CSR
mat-vec order), with the cube computed by a fixed exact-two-product sequence.
So the bar is: bit-identical to the oracle in cube="exact" mode, and within
1e-10 relative max-norm of the unmodified reference (golden vectors), with the
same Parareal iteration counts.
"""

import numpy as np
import pytest

from oracle import chp_oracle as O

pytestmark = pytest.mark.gpu

EXACT = O.Knobs(cube="exact")


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_14074_b200 import parareal, schemes, grid
    return parareal, schemes, grid


def _steps_cases(z, dim=1):
    ci = 0
    while f"in_{ci}" in z:
        d, nx, eps, dt = z[f"meta_{ci}"]
        if int(d) == dim:
            yield ci, int(nx), float(eps), float(dt)
        ci += 1


def test_single_steps_bitwise_vs_oracle(P, golden):
    _, S, G = P
    z = golden("steps.npz")
    for ci, nx, eps, dt in _steps_cases(z):
        g = G.SpatialGrid(1, nx)
        mesh = O.Mesh(1, nx)
        v = z[f"in_{ci}"]
        for s, sch, och in (("a", S.Scheme.LINEAR_A, O.LINEAR_A), ("b", S.Scheme.LINEAR_B, O.LINEAR_B),
                            ("n", S.Scheme.NONLINEAR_EYRE, O.EYRE)):
            spec = S.PropagatorSpec(sch, dt, eps)
            for steps in (1, 8):
                try:
                    want = O.advance(mesh, v, och, dt, eps, steps, EXACT)
                except O.NewtonFailure as exc:
                    with pytest.raises(S.NewtonDivergenceError) as ei:
                        S.propagate(G.Field(g, v), spec, steps)
                    assert ei.value.iterations == exc.iterations
                    continue
                got = S.propagate(G.Field(g, v), spec, steps).values
                assert np.array_equal(got, want), (ci, s, steps, rel(got, want))
                if f"{s}{steps}_{ci}" in z:   # unmodified reference (numpy cube)
                    # only the host's numpy v**3 (1-ulp, SVML) differs; Newton amplifies it
                    tol = 1e-12 if s != "n" else 1e-10
                    assert rel(got, z[f"{s}{steps}_{ci}"]) < tol, (ci, s, steps)


def test_batched_propagate_with_index(P):
    import torch
    _, S, G = P
    g = G.SpatialGrid(1, 129)
    rng = np.random.default_rng(3)
    V = rng.uniform(-0.8, 0.8, (6, g.interior_count))
    src = torch.tensor(V, device="cuda")
    out = torch.zeros_like(src)
    idx = torch.tensor([5, 0, 3], dtype=torch.int32, device="cuda")
    spec = S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, 1e-4, 0.05)
    info = S.propagate_batch(g, spec, 4, src, out, sys_index=idx)
    si = S.read_sysinfo(info)
    mesh = O.Mesh(1, 129)
    for k in range(6):
        if k in (5, 0, 3):
            cnt = O.NewtonCounter()
            want = O.advance(mesh, V[k], O.EYRE, 1e-4, 0.05, 4, EXACT, cnt)
            assert np.array_equal(out[k].cpu().numpy(), want)
            assert si["newton_steps"][k] == 4 and si["newton_total"][k] == cnt.total
        else:
            assert float(out[k].abs().max()) == 0.0 and si["newton_steps"][k] == 0


def test_zero_is_fixed_point(P):
    _, S, G = P
    g = G.SpatialGrid(1, 65)
    for sch in (S.Scheme.LINEAR_A, S.Scheme.LINEAR_B, S.Scheme.NONLINEAR_EYRE):
        out = S.propagate(G.Field(g, np.zeros(63)), S.PropagatorSpec(sch, 1e-3, 0.1), 5)
        assert np.all(out.values == 0.0)


def test_nonfinite_raises(P):
    _, S, G = P
    g = G.SpatialGrid(1, 33)
    v = np.full(31, 1e120)
    with pytest.raises(ValueError, match="non-finite"):
        S.propagate(G.Field(g, v), S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-3, 0.1), 3)


def test_newton_budget_raises(P):
    _, S, G = P
    g = G.SpatialGrid(1, 65)
    v = np.random.default_rng(0).uniform(-0.9, 0.9, 63)
    spec = S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, 1e-2, 0.05, newton_tol=1e-30,
                            newton_max_iter=3)
    with pytest.raises(S.NewtonDivergenceError) as ei:
        S.propagate(G.Field(g, v), spec, 1)
    assert ei.value.iterations == 3


@pytest.mark.parametrize("var", ["pa1", "pa2", "pa3", "npa1", "npa2"])
def test_spec_small_parareal(P, golden, var):
    PP, S, G = P
    z = golden("spec_small.npz")
    g = G.SpatialGrid(1, 10)
    u0 = z["u0"]
    tr = PP.run(G.Field(g, u0), PP.AlgorithmVariant(var), PP.TimePartition(0.5, 4, 4), 0.1,
                stop="increment")
    ref = O.parareal(O.Mesh(1, 10), u0, var, 0.5, 4, 4, 0.1, EXACT)
    assert tr.converged_at == ref.k == int(z[f"{var}_k"][0])
    assert np.array_equal(np.array(tr.increments), np.array(ref.increments))
    # after N iterations the error vs the serial fine reference
    nrm = tr.reference_norm
    assert tr.records[4].error <= 1e-12 * (1 + nrm)


def test_parareal_iteration_api_matches_engine(P, golden):
    PP, S, G = P
    z = golden("spec_small.npz")
    g = G.SpatialGrid(1, 10)
    var, part = PP.AlgorithmVariant.PA3, PP.TimePartition(0.5, 4, 4)
    st = PP.initial_state(G.Field(g, z["u0"]), var, part, 0.1)
    hist, states = [], []
    for _ in range(3):
        st = PP.parareal_iteration(st, var, part, 0.1)
        states.append(st)
        hist.append(np.array([f.values for f in st.iterates]))
        assert PP.iterate_increment(st) >= 0.0
    ref = O.parareal(O.Mesh(1, 10), z["u0"], "pa3", 0.5, 4, 4, 0.1, EXACT, keep_history=True,
                     max_iter=3, inc_tol=0.0)
    for k in range(3):
        assert np.array_equal(hist[k], ref.history[k])
    # U_0 pinned; previous is the frozen U^k of the iteration (parareal.py:258)
    assert np.array_equal(st.iterates[0].values, z["u0"])
    assert np.array_equal(np.array([f.values for f in st.previous]), hist[1])
    assert PP.iterate_increment(st) == float(np.max(np.abs(hist[2] - hist[1])))
    # a state rebuilt from host fields (no device cache: the engine is re-created from
    # iterates + coarse values) iterates to the same bits
    s2 = states[1]
    st2 = PP.PararealState(iterates=[G.Field(g, np.array(f.values)) for f in s2.iterates],
                           coarse_values=[G.Field(g, np.array(f.values)) for f in s2.coarse_values],
                           fine_reference=[], k=2)
    st3 = PP.parareal_iteration(st2, var, part, 0.1)
    assert np.array_equal(np.array([f.values for f in st3.iterates]), hist[2])


def test_config1_pa3_full(P, golden):
    """Config 1: same k (17) as the reference, iterates within 1e-10."""
    PP, S, G = P
    z = golden("config1.npz")
    g = G.SpatialGrid(1, 257)
    tr = PP.run(G.Field(g, z["u0"]), PP.AlgorithmVariant.PA3, PP.TimePartition(1.0, 16, 256),
                0.05, stop="increment")
    assert tr.converged_at == int(z["pa3_k"][0]) == 17
    ref = O.parareal(O.Mesh(1, 257), z["u0"], "pa3", 1.0, 16, 256, 0.05, EXACT)
    assert np.array_equal(np.array(tr.increments), np.array(ref.increments))
    assert tr.fine_point_steps == 136 * 256 * 255
    from paper_2304_14074_b200.parareal import _engine_for  # noqa: F401


def test_config1_iterates_vs_reference(P, golden):
    PP, S, G = P
    z = golden("config1.npz")
    g = G.SpatialGrid(1, 257)
    f, c = PP.propagator_pair(PP.AlgorithmVariant.PA3, PP.TimePartition(1.0, 16, 256), 0.05)
    from paper_2304_14074_b200.engine import PararealEngine
    eng = PararealEngine(g, f, c, 16, 256)
    eng.load([G.Field(g, z["u0"])])
    eng.coarse_init()
    ref = O.parareal(O.Mesh(1, 257), z["u0"], "pa3", 1.0, 16, 256, 0.05, EXACT,
                     keep_history=True)
    for k in range(1, 18):
        eng.iterate()
        assert np.array_equal(eng.iterates_host(), ref.history[k - 1])   # bit-identical
        # Intermediate iterates pass through the kappa~1e7 coarse solve, which
        # amplifies the reference host's 1-ulp v**3 differences (SURVEY.md 8(c),
        # T2 note); converged iterates are insensitive.
        if k == 1:
            assert rel(eng.iterates_host(), z["pa3_U1"]) < 1e-10
        if k == 8:
            assert rel(eng.iterates_host(), z["pa3_U8"]) < 1e-8
    U = eng.iterates_host()
    assert rel(U, z["pa3_U"]) < 1e-10
    assert eng.converged_at[0] == 17


def test_config1_size_npa1(P, golden):
    PP, S, G = P
    z = golden("config1.npz")
    g = G.SpatialGrid(1, 257)
    tr = PP.run(G.Field(g, z["u0"]), PP.AlgorithmVariant.NPA1, PP.TimePartition(0.25, 4, 64),
                0.05, stop="increment")
    ref = O.parareal(O.Mesh(1, 257), z["u0"], "npa1", 0.25, 4, 64, 0.05, EXACT)
    assert tr.converged_at == ref.k == int(z["npa1_k"][0])
    assert np.array_equal(np.array(tr.increments), np.array(ref.increments))


def test_config2_truncated_npa1(P, golden):
    """Config 2 parameters, IC 0, first 4 slices (J=512, Newton tol 1e-10)."""
    PP, S, G = P
    z = golden("config2_trunc.npz")
    g = G.SpatialGrid(1, 1025)
    part = PP.TimePartition(4 * 2.0 / 64, 4, 512)
    from paper_2304_14074_b200.engine import PararealEngine
    f, c = PP.propagator_pair(PP.AlgorithmVariant.NPA1, part, 0.03)
    eng = PararealEngine(g, f, c, 4, 512)
    eng.load([G.Field(g, z["u0"])])
    conv = eng.run()
    assert conv[0] == int(z["npa1_k"][0])
    U = eng.iterates_host()
    ref = O.parareal(O.Mesh(1, 1025), z["u0"], "npa1", part.total_time, 4, 512, 0.03, EXACT)
    assert ref.k == conv[0]
    assert np.array_equal(U, ref.iterates)
    # vs the unmodified reference: only the numpy-vs-exact cube ulps differ
    assert rel(U, z["npa1_U"]) < 1e-8
    assert eng.newton.steps > 0


def test_run_batch_matches_single_runs(P):
    PP, S, G = P
    g = G.SpatialGrid(1, 129)
    part = PP.TimePartition(0.01, 4, 16)
    u0s = [G.Field(g, np.random.default_rng(b).uniform(-0.05, 0.05, 127)) for b in range(3)]
    res = PP.run_batch(u0s, PP.AlgorithmVariant.NPA1, part, 0.05)
    for b in range(3):
        ref = O.parareal(O.Mesh(1, 129), u0s[b].values, "npa1", 0.01, 4, 16, 0.05, EXACT)
        assert res.converged_at[b] == ref.k
        assert np.array_equal(res.engine.iterates_host(b), ref.iterates)


@pytest.mark.parametrize("name", ["d1", "d1b", "d2"])
def test_step_nonlinear_residual_history(P, golden, name):
    """StepReport.residual_history (schemes.py:285-290) recorded on the device
    (chp_propagate_hist) vs the reference's own step_nonlinear: same length
    (iteration count), every pre-convergence residual to 1e-8 relative plus
    1e-14 of the initial residual (2D solves are CG to 1e-14, not SuperLU), the
    accepted one below newton_tol."""
    _, schemes, grid = P
    z = golden("newton_hist.npz")
    dim, nx, dt, eps = z[f"{name}/params"]
    g = grid.SpatialGrid(int(dim), int(nx))
    spec = schemes.PropagatorSpec(schemes.Scheme.NONLINEAR_EYRE, float(dt), float(eps))
    out, rep = schemes.step_nonlinear(grid.Field(g, z[f"{name}/u0"]), spec)
    ref = z[f"{name}/hist"]
    h = np.array(rep.residual_history)
    assert len(h) == len(ref) == rep.newton_iterations + 1
    assert np.all(np.abs(h[:-1] - ref[:-1]) <= 1e-8 * ref[:-1] + 1e-14 * ref[0])
    assert h[-1] <= spec.newton_tol and h[-1] == rep.residual_norm
    assert rel(out.values, z[f"{name}/out"]) < 1e-10
