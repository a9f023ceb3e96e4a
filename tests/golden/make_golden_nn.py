"""Golden vectors of the reference's Neumann-Neumann fine step (ddm.py).

Run in the build container only (imports /root/reference):

    python tests/golden/make_golden_nn.py

Writes tests/golden/nn_small.npz: per case the input field, the reference's
output after ``steps`` NN steps (ddm.nn_propagate), the per-step sweep counts
(ddm._nn_solve's InterfaceTraces.iterations), the final traces, one
NNConvergenceError case, and a small Parareal run whose fine propagator is
NN_LINEAR_A (parareal.propagator_pair(..., nn=...)).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

# (name, nx, n_sub, theta, tol, max_iter, warm, dt, eps, steps, seed)
CASES = [
    ("c65_s4", 65, 4, 0.25, 1e-10, 100, False, 2.0 ** -12, 0.05, 3, 1),
    ("c65_s4_warm", 65, 4, 0.25, 1e-10, 100, True, 2.0 ** -12, 0.05, 3, 1),
    ("c65_s2_th40", 65, 2, 0.4, 1e-11, 200, False, 2.0 ** -10, 0.05, 2, 2),
    ("c257_s8", 257, 8, 0.25, 1e-10, 200, False, 2.0 ** -12, 0.05, 2, 3),
    ("c1025_s8", 1025, 8, 0.25, 1e-10, 300, False, 2.0 ** -14, 0.03, 1, 4),
    ("c129_s16_warm", 129, 16, 0.25, 1e-10, 400, True, 2.0 ** -12, 0.05, 3, 5),
]


def main():
    sys.path.insert(0, REF)
    from chparareal import ddm, grid, parareal, schemes

    out = {}
    for name, nx, S, th, tol, mi, warm, dt, eps, steps, seed in CASES:
        g = grid.SpatialGrid(dim=1, nodes_per_axis=nx)
        rng = np.random.default_rng(seed)
        x = np.arange(1, nx - 1) / (nx - 1)
        u0 = 0.2 * np.sin(2 * np.pi * x) + rng.uniform(-0.05, 0.05, nx - 2)
        p = ddm.NNParams(n_subdomains=S, theta=th, tol=tol, max_iter=mi, warm_start=warm)
        dec = ddm.Decomposition(g, S)
        spec = ddm.nn_propagator(dec, p, dt, eps)
        res = ddm.nn_propagate(grid.Field(g, u0), spec, steps)
        # sweep counts and traces per step, replaying nn_propagate's loop
        cur, tr, sweeps = grid.Field(g, u0), None, []
        for _ in range(steps):
            cur, ftr = ddm._nn_solve(cur, dec, p, dt, eps, traces=tr)
            sweeps.append(ftr.iterations)
            if warm:
                tr = ddm.InterfaceTraces(g=ftr.g.copy(), h=ftr.h.copy())
        assert np.array_equal(cur.values, res.values)
        out[f"{name}/params"] = np.array([nx, S, th, tol, mi, int(warm), dt, eps, steps])
        out[f"{name}/u0"] = u0
        out[f"{name}/out"] = res.values
        out[f"{name}/sweeps"] = np.array(sweeps)
        out[f"{name}/g"] = ftr.g
        out[f"{name}/h"] = ftr.h

    # budget exhausted -> NNConvergenceError(iterations, g_inc, h_inc)
    g = grid.SpatialGrid(dim=1, nodes_per_axis=65)
    u0 = out["c65_s4/u0"]
    p = ddm.NNParams(n_subdomains=4, theta=0.25, tol=1e-10, max_iter=3)
    try:
        ddm.nn_time_step(grid.Field(g, u0), ddm.Decomposition(g, 4), p, 2.0 ** -12, 0.05)
        raise SystemExit("expected NNConvergenceError")
    except ddm.NNConvergenceError as e:
        out["fail/info"] = np.array([e.iterations, e.g_increment, e.h_increment])

    # Parareal with the NN fine propagator: coarse_init + iterations to increment 1e-10
    nx, S, eps, T, N, J = 65, 4, 0.05, 0.0625, 4, 8
    g = grid.SpatialGrid(dim=1, nodes_per_axis=nx)
    x = np.arange(1, nx - 1) / (nx - 1)
    u0 = 0.2 * np.sin(2 * np.pi * x) + np.random.default_rng(7).uniform(-0.05, 0.05, nx - 2)
    nn = ddm.NNParams(n_subdomains=S)
    part = parareal.TimePartition(total_time=T, num_slices=N, fine_steps=J)
    var = parareal.AlgorithmVariant.PA1
    init = parareal.coarse_init(grid.Field(g, u0), var, part, eps)
    st = parareal.PararealState(iterates=init, coarse_values=init[1:], fine_reference=[], k=0)
    incs = []
    while st.k < N + 2:
        st = parareal.parareal_iteration(st, var, part, eps, nn=nn)
        incs.append(max(float(np.max(np.abs(a.values - b.values)))
                        for a, b in zip(st.iterates, st.previous)))
        if incs[-1] < 1e-10:
            break
    out["pr/params"] = np.array([nx, S, eps, T, N, J])
    out["pr/u0"] = u0
    out["pr/U"] = np.array([f.values for f in st.iterates])
    out["pr/incs"] = np.array(incs)
    np.savez_compressed(os.path.join(OUT, "nn_small.npz"), **out)
    for k in sorted(out):
        if k.endswith("sweeps") or k.startswith("fail") or k.endswith("incs"):
            print(k, out[k])


if __name__ == "__main__":
    main()
