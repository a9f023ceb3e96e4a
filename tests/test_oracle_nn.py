"""Pin the oracle's Neumann-Neumann restatement (oracle/chp_oracle.py, ddm.py
section) to the reference's own outputs (tests/golden/make_golden_nn.py):
the same dense LAPACK LU calls in the same order, so bit-identical."""

import numpy as np
import pytest

from oracle import chp_oracle as O

CASES = ["c65_s4", "c65_s4_warm", "c65_s2_th40", "c257_s8", "c1025_s8", "c129_s16_warm"]


def nn_case(z, name):
    nx, S, th, tol, mi, warm, dt, eps, steps = z[f"{name}/params"]
    nn = O.NNSetup(int(S), float(th), float(tol), int(mi), bool(warm))
    return O.Mesh(1, int(nx)), nn, float(dt), float(eps), int(steps)


@pytest.mark.parametrize("name", CASES)
def test_nn_oracle_bitwise(golden, name):
    z = golden("nn_small.npz")
    mesh, nn, dt, eps, steps = nn_case(z, name)
    sweeps = []
    out = O.nn_advance(mesh, z[f"{name}/u0"], dt, eps, nn, steps, sweeps)
    assert np.array_equal(out, z[f"{name}/out"])
    assert sweeps == list(z[f"{name}/sweeps"])


def test_nn_oracle_budget_error(golden):
    z = golden("nn_small.npz")
    mesh, nn, dt, eps, _ = nn_case(z, "c65_s4")
    nn = O.NNSetup(4, 0.25, 1e-10, 3)
    with pytest.raises(O.NNFailure) as e:
        O.nn_step(mesh, z["c65_s4/u0"], dt, eps, nn)
    it, gi, hi = z["fail/info"]
    assert e.value.sweeps == int(it) and e.value.g_inc == gi and e.value.h_inc == hi


def test_nn_fixed_point_is_linear_a(golden):
    """ddm.py:1-27: the interface iteration's fixed point is the monodomain
    LINEAR_A step; the converged NN step must agree with it to the trace tol."""
    z = golden("nn_small.npz")
    mesh, nn, dt, eps, _ = nn_case(z, "c257_s8")
    u0 = z["c257_s8/u0"]
    a = O.step_a(mesh, u0, dt, eps, O.Knobs())
    b, *_ = O.nn_step(mesh, u0, dt, eps, nn)
    assert np.max(np.abs(a - b)) < 1e-9


def test_nn_parareal_oracle(golden):
    z = golden("nn_small.npz")
    nx, S, eps, T, N, J = z["pr/params"]
    r = O.parareal(O.Mesh(1, int(nx)), z["pr/u0"], "pa1", float(T), int(N), int(J), float(eps),
                   O.Knobs(nn=O.NNSetup(int(S))), skip_stable=False)
    assert np.array_equal(np.array(r.increments), z["pr/incs"])
    assert np.array_equal(r.iterates, z["pr/U"])
