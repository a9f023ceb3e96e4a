"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

The reference ships no tests or fixtures, so these files
are the pins for the CPU oracle (oracle/chp_oracle.py): tests/test_oracle_golden.py
checks the oracle against them bit for bit.  Inputs are seeded and small.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def ref_modules():
    sys.path.insert(0, REF)
    from chparareal import grid, parareal, schemes  # noqa: E402
    return grid, schemes, parareal


def increment_driver(parareal, grid, u0, variant, part, eps, max_iter=None, tol=1e-10,
                     keep=None):
    """coarse_init + parareal_iteration until max|U^{k+1}-U^k| < tol
    (the reference's own functions)."""
    init = parareal.coarse_init(u0, variant, part, eps)
    st = parareal.PararealState(iterates=init, coarse_values=init[1:],
                                fine_reference=[], k=0)
    stats = parareal.NewtonStats() if hasattr(parareal, "NewtonStats") else None
    from chparareal.schemes import NewtonStats
    stats = NewtonStats()
    if max_iter is None:
        max_iter = part.num_slices + 2
    incs, snaps = [], {}
    k_done = None
    while st.k < max_iter:
        st = parareal.parareal_iteration(st, variant, part, eps, stats=stats)
        inc = max(float(np.max(np.abs(a.values - b.values)))
                  for a, b in zip(st.iterates, st.previous))
        incs.append(inc)
        if keep is not None and st.k in keep:
            snaps[st.k] = np.array([f.values for f in st.iterates])
        if inc < tol:
            k_done = st.k
            break
    U = np.array([f.values for f in st.iterates])
    return k_done, np.array(incs), U, snaps, stats


def main():
    grid, schemes, parareal = ref_modules()
    t0 = time.time()

    # 1. operators and eigenvalues (SPEC.md:48-59 examples)
    ops = {}
    for dim, nx in ((1, 4), (1, 10), (1, 17), (2, 4), (2, 6)):
        g = grid.SpatialGrid(dim, nx)
        op = grid.build_laplacian(g)
        ops[f"L_{dim}_{nx}"] = op.matrix.toarray()
        ops[f"L2_{dim}_{nx}"] = op.squared.toarray()
    for nx in (4, 10, 257, 1025):
        ops[f"eig_{nx}"] = grid.laplacian_eigenvalues(grid.SpatialGrid(1, nx))
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **ops)

    # 2. single steps and short propagations on seeded inputs
    steps = {}
    cases = [(1, 17, 0.1, 1e-3), (1, 257, 0.05, 2.0 ** -12), (1, 257, 0.05, 2.0 ** -4),
             (1, 1025, 0.03, 2.0 ** -15), (2, 9, 0.1, 1e-3), (2, 17, 0.05, 2.0 ** -10),
             (2, 33, 0.02, 2.0 ** -9)]
    for ci, (dim, nx, eps, dt) in enumerate(cases):
        g = grid.SpatialGrid(dim, nx)
        rng = np.random.default_rng(100 + ci)
        v = rng.uniform(-0.9, 0.9, g.interior_count)
        steps[f"in_{ci}"] = v
        steps[f"meta_{ci}"] = np.array([dim, nx, eps, dt])
        u = grid.Field(g, v)
        for sname, sch in (("a", schemes.Scheme.LINEAR_A), ("b", schemes.Scheme.LINEAR_B),
                           ("n", schemes.Scheme.NONLINEAR_EYRE)):
            spec = schemes.PropagatorSpec(sch, dt, eps)
            st = schemes.NewtonStats()
            try:
                steps[f"{sname}1_{ci}"] = schemes.propagate(u, spec, 1, st).values
                steps[f"{sname}8_{ci}"] = schemes.propagate(u, spec, 8, st).values
            except schemes.NewtonDivergenceError as exc:   # edge case: recorded
                steps[f"nerr_{ci}"] = np.array([exc.iterations, exc.residual])
            if sname == "n":
                steps[f"nstat_{ci}"] = np.array([st.steps, st.total_iterations,
                                                 st.max_iterations, st.max_residual])
    np.savez_compressed(os.path.join(OUT, "steps.npz"), **steps)

    # 3. SPEC.md acceptance 1 config (1D, N_x=10, T=0.5, N=4, J=4, eps=0.1), all variants
    spec_runs = {}
    g = grid.SpatialGrid(1, 10)
    u0 = grid.Field(g, 0.1 * np.sin(np.pi * g.interior_coordinates())
                    + np.random.default_rng(7).uniform(-0.1, 0.1, g.interior_count))
    spec_runs["u0"] = u0.values
    part = parareal.TimePartition(0.5, 4, 4)
    for var in parareal.AlgorithmVariant:
        k, incs, U, snaps, st = increment_driver(parareal, grid, u0, var, part, 0.1,
                                                 keep={1, 2})
        ser = parareal.serial_fine_reference(u0, var, part, 0.1)
        spec_runs[f"{var.value}_k"] = np.array([-1 if k is None else k])
        spec_runs[f"{var.value}_inc"] = incs
        spec_runs[f"{var.value}_U"] = U
        spec_runs[f"{var.value}_U1"] = snaps[1]
        spec_runs[f"{var.value}_serial"] = np.array([f.values for f in ser])
    np.savez_compressed(os.path.join(OUT, "spec_small.npz"), **spec_runs)

    # 4. config 1 in full (PA3) and a config-1-size NPA1 run
    sys.path.insert(0, os.path.join(OUT, "..", ".."))
    from oracle.chp_oracle import initial_condition  # seeded generator only
    c1 = {}
    g = grid.SpatialGrid(1, 257)
    u0 = grid.Field(g, initial_condition(1))
    part = parareal.TimePartition(1.0, 16, 256)
    t1 = time.time()
    k, incs, U, snaps, _ = increment_driver(parareal, grid, u0, parareal.AlgorithmVariant.PA3,
                                            part, 0.05, keep={1, 8})
    c1["pa3_seconds"] = np.array([time.time() - t1])
    c1["u0"] = u0.values
    c1["pa3_k"] = np.array([k])
    c1["pa3_inc"] = incs
    c1["pa3_U"] = U
    c1["pa3_U1"] = snaps[1]
    c1["pa3_U8"] = snaps[8]
    c1["pa3_serial"] = np.array([f.values for f in parareal.serial_fine_reference(
        u0, parareal.AlgorithmVariant.PA3, part, 0.05)])
    part = parareal.TimePartition(0.25, 4, 64)
    k, incs, U, snaps, st = increment_driver(parareal, grid, u0, parareal.AlgorithmVariant.NPA1,
                                             part, 0.05, keep={1})
    c1["npa1_k"] = np.array([k])
    c1["npa1_inc"] = incs
    c1["npa1_U"] = U
    c1["npa1_U1"] = snaps[1]
    c1["npa1_newton"] = np.array([st.steps, st.total_iterations, st.max_iterations,
                                  st.max_residual])
    np.savez_compressed(os.path.join(OUT, "config1.npz"), **c1)

    # 5. config 2 truncated: IC 0, 4 slices of the config-2 coarse step, J=512
    c2 = {}
    g = grid.SpatialGrid(1, 1025)
    u0 = grid.Field(g, initial_condition(2, 0))
    part = parareal.TimePartition(4 * 2.0 / 64, 4, 512)
    k, incs, U, snaps, st = increment_driver(parareal, grid, u0, parareal.AlgorithmVariant.NPA1,
                                             part, 0.03, keep={1})
    c2["u0"] = u0.values
    c2["npa1_k"] = np.array([k])
    c2["npa1_inc"] = incs
    c2["npa1_U"] = U
    c2["npa1_U1"] = snaps[1]
    c2["npa1_newton"] = np.array([st.steps, st.total_iterations, st.max_iterations,
                                  st.max_residual])
    np.savez_compressed(os.path.join(OUT, "config2_trunc.npz"), **c2)

    # 6. small 2D runs (PA3 and NPA1), grids small enough for SuperLU in seconds
    d2 = {}
    g = grid.SpatialGrid(2, 33)
    v = np.random.default_rng(0).uniform(-0.05, 0.05, g.interior_count)
    u0 = grid.Field(g, v - v.mean())
    d2["u0"] = u0.values
    part = parareal.TimePartition(0.05, 4, 16)
    k, incs, U, snaps, _ = increment_driver(parareal, grid, u0, parareal.AlgorithmVariant.PA3,
                                            part, 0.05, keep={1})
    d2["pa3_k"] = np.array([k]); d2["pa3_inc"] = incs; d2["pa3_U"] = U; d2["pa3_U1"] = snaps[1]
    part = parareal.TimePartition(0.02, 4, 8)
    k, incs, U, snaps, st = increment_driver(parareal, grid, u0, parareal.AlgorithmVariant.NPA1,
                                             part, 0.05, keep={1})
    d2["npa1_k"] = np.array([k]); d2["npa1_inc"] = incs; d2["npa1_U"] = U
    d2["npa1_U1"] = snaps[1]
    d2["npa1_newton"] = np.array([st.steps, st.total_iterations, st.max_iterations,
                                  st.max_residual])
    np.savez_compressed(os.path.join(OUT, "twod_small.npz"), **d2)
    print(f"golden vectors written in {time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
