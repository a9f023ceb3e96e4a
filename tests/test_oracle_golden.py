"""Pin the CPU oracle (oracle/chp_oracle.py) to golden vectors produced by the
UNMODIFIED reference (tests/golden/make_golden.py).  With cube="numpy" and the
reference's LAPACK/SuperLU solvers the oracle must be bit-identical."""

import numpy as np
import pytest

from oracle import chp_oracle as O


def test_operators_match_reference(golden):
    z = golden("operators.npz")
    for dim, nx in ((1, 4), (1, 10), (1, 17), (2, 4), (2, 6)):
        ops = O.operators(O.Mesh(dim, nx))
        assert np.array_equal(ops.L.toarray(), z[f"L_{dim}_{nx}"])
        assert np.array_equal(ops.L2.toarray(), z[f"L2_{dim}_{nx}"])
    for nx in (4, 10, 257, 1025):
        assert np.array_equal(O.axis_eigenvalues(nx), z[f"eig_{nx}"])
    # SPEC.md:48-59 known answers
    assert np.array_equal(z["L_1_4"], 9.0 * np.array([[-2.0, 1.0], [1.0, -2.0]]))
    assert np.all(np.diag(z["L_2_4"]) == -36.0)
    assert abs(z["eig_4"][0] + 9.0) < 1e-12


def test_single_steps_bitwise(golden):
    z = golden("steps.npz")
    ci = 0
    while f"in_{ci}" in z:
        dim, nx, eps, dt = z[f"meta_{ci}"]
        mesh = O.Mesh(int(dim), int(nx))
        v = z[f"in_{ci}"]
        kn = O.Knobs(cube="numpy")
        for s, sch in (("a", O.LINEAR_A), ("b", O.LINEAR_B), ("n", O.EYRE)):
            cnt = O.NewtonCounter()
            if f"{s}8_{ci}" not in z:          # reference raised NewtonDivergenceError
                assert s == "n" and f"nerr_{ci}" in z
                steps = 1 if f"{s}1_{ci}" not in z else 8
                if steps == 8:
                    assert np.array_equal(O.advance(mesh, v, sch, dt, eps, 1, kn),
                                          z[f"{s}1_{ci}"])
                with pytest.raises(O.NewtonFailure) as ei:
                    O.advance(mesh, v, sch, dt, eps, steps, kn)
                assert ei.value.iterations == int(z[f"nerr_{ci}"][0])
                assert ei.value.residual == z[f"nerr_{ci}"][1]
                continue
            out1 = O.advance(mesh, v, sch, dt, eps, 1, kn, cnt)
            out8 = O.advance(mesh, v, sch, dt, eps, 8, kn, cnt)
            assert np.array_equal(out1, z[f"{s}1_{ci}"]), (ci, s)
            assert np.array_equal(out8, z[f"{s}8_{ci}"]), (ci, s)
            if s == "n":
                st = z[f"nstat_{ci}"]
                assert (cnt.steps, cnt.total, cnt.max_iter) == tuple(int(x) for x in st[:3])
                assert cnt.max_residual == st[3]
        ci += 1


def test_spec_small_all_variants(golden):
    z = golden("spec_small.npz")
    mesh = O.Mesh(1, 10)
    for var in ("pa1", "pa2", "pa3", "npa1", "npa2"):
        r = O.parareal(mesh, z["u0"], var, 0.5, 4, 4, 0.1, O.Knobs(cube="numpy"),
                       keep_history=True, with_serial=True)
        assert r.k == int(z[f"{var}_k"][0])
        assert np.array_equal(np.array(r.increments), z[f"{var}_inc"])
        assert np.array_equal(r.iterates, z[f"{var}_U"])
        assert np.array_equal(r.history[0], z[f"{var}_U1"])
        assert np.array_equal(r.serial, z[f"{var}_serial"])
        # SPEC.md:475 acceptance 1 -- finite-step convergence after N iterations
        nrm = max(O.l2(mesh, f) for f in r.serial)
        assert r.errors[3] <= 1e-12 * (1 + nrm)


def test_config1_pa3_full_bitwise(golden):
    z = golden("config1.npz")
    mesh = O.Mesh(1, 257)
    assert np.array_equal(z["u0"], O.initial_condition(1))
    r = O.parareal(mesh, z["u0"], "pa3", 1.0, 16, 256, 0.05, O.Knobs(cube="numpy"),
                   keep_history=True)
    assert r.k == int(z["pa3_k"][0]) == 17
    assert np.array_equal(np.array(r.increments), z["pa3_inc"])
    assert np.array_equal(r.iterates, z["pa3_U"])
    assert np.array_equal(r.history[7], z["pa3_U8"])
    # skip-stable-slices: half the fine work, same bits
    assert r.fine_props == 136


def test_config1_size_npa1_bitwise(golden):
    z = golden("config1.npz")
    mesh = O.Mesh(1, 257)
    r = O.parareal(mesh, z["u0"], "npa1", 0.25, 4, 64, 0.05, O.Knobs(cube="numpy"))
    assert r.k == int(z["npa1_k"][0])
    assert np.array_equal(r.iterates, z["npa1_U"])


def test_twod_small_bitwise(golden):
    z = golden("twod_small.npz")
    mesh = O.Mesh(2, 33)
    r = O.parareal(mesh, z["u0"], "pa3", 0.05, 4, 16, 0.05, O.Knobs(cube="numpy"))
    assert r.k == int(z["pa3_k"][0])
    assert np.array_equal(r.iterates, z["pa3_U"])
    r = O.parareal(mesh, z["u0"], "npa1", 0.02, 4, 8, 0.05, O.Knobs(cube="numpy"))
    assert r.k == int(z["npa1_k"][0])
    assert np.array_equal(r.iterates, z["npa1_U"])


def test_exact_cube_is_deterministic_and_accurate():
    from fractions import Fraction
    rng = np.random.default_rng(5)
    v = np.concatenate([rng.uniform(-1.5, 1.5, 4000), [0.0, -0.0, 1.0, -1.0, 1e-3]])
    c = O.exact_cube(v)
    exact = np.array([float(Fraction(x) ** 3) for x in v])
    assert np.mean(c == exact) > 0.999
    assert np.max(np.abs(c - exact) / np.maximum(np.abs(exact), 1e-300)) <= 2.3e-16


def test_oracle_pcg_knob_matches_superlu():
    """The oracle's 2D DST-PCG solve (Knobs(pcg=True), used for truncated config-4
    runs) agrees with the reference's SuperLU solve to ~1e-13."""
    mesh = O.Mesh(2, 65)
    ops = O.operators(mesh)
    rng = np.random.default_rng(0)
    v = rng.uniform(-0.9, 0.9, mesh.size)
    rhs = rng.uniform(-1.0, 1.0, mesh.size)
    for a, b in ((2.0 ** -8, 0.02 ** 2 * 2.0 ** -8), (3 * 2.0 ** -15, 0.015 ** 2 * 2.0 ** -15)):
        x1 = O.variable_solve(ops, a, b, v * v, rhs)
        x2 = O.variable_solve(ops, a, b, v * v, rhs, pcg=True)
        assert np.max(np.abs(x1 - x2)) / np.max(np.abs(x1)) < 1e-12


RUN_TAGS = ("spec_pa1", "spec_pa2", "spec_pa3", "spec_npa1", "spec_npa2", "c1", "c1n", "d2", "d2n")


def _run_case(z, tag):
    nx, T, N, J, eps = z[f"{tag}_meta"]
    dim = 2 if tag.startswith("d2") else 1
    variant = {"spec_pa1": "pa1", "spec_pa2": "pa2", "spec_pa3": "pa3", "spec_npa1": "npa1",
               "spec_npa2": "npa2", "c1": "pa3", "c1n": "npa1", "d2": "pa3", "d2n": "npa1"}[tag]
    return O.Mesh(dim, int(nx)), variant, float(T), int(N), int(J), float(eps)


@pytest.mark.parametrize("tag", RUN_TAGS)
def test_oracle_serial_and_run_errors(golden, tag):
    """a18/a19 pins: the oracle's serial fine reference equals the reference's
    serial_fine_reference bit for bit, and its per-iteration L_inf(0,T;L2) errors
    equal the reference run()'s records (parareal.py:145-164, 262-374)."""
    z = golden("run_traces.npz")
    mesh, var, T, N, J, eps = _run_case(z, tag)
    u0 = z[f"{tag}_u0"]
    kn = O.Knobs(cube="numpy")
    ser = O.serial_fine(mesh, u0, var, T, N, J, eps, kn)
    assert np.array_equal(ser, z[f"{tag}_serial"])
    conv = int(z[f"{tag}_converged"][0])
    r = O.parareal(mesh, u0, var, T, N, J, eps, kn, with_serial=True, inc_tol=0.0,
                   max_iter=conv)
    errs = np.array(r.errors)
    want = z[f"{tag}_error"][1:]
    assert errs.shape == want.shape
    assert np.allclose(errs, want, rtol=1e-12, atol=1e-15), (errs, want)
    assert errs[-1] <= 1e-6 < errs[-2]


def test_package_configs_match_oracle_inputs():
    """The package's seeded generators (bench / time to tolerance) produce exactly the
    oracle's inputs, so every parity golden applies to the benchmarked workloads."""
    from paper_2304_14074_b200 import configs as C
    for c in range(1, 6):
        assert C.CONFIGS[c] == O.CONFIGS[c]
        for ic in (0, 1, 63):
            assert np.array_equal(C.initial_condition(c, ic), O.initial_condition(c, ic))
