"""Golden traces of the UNMODIFIED reference's own ``run()`` and ``serial_fine_reference``
(reference parareal.py:145-164, 262-374), for the a18/a19 parity tests
(tests/test_gpu_run.py).  Build container only (imports /root/reference):

    python tests/golden/make_golden_run.py

Cases (seeded, small enough for the reference to finish in seconds):
* ``spec_<variant>``: SPEC.md acceptance-1 config (1D, N_x = 10, T = 0.5, N = 4, J = 4,
  eps = 0.1), every variant, run(tol=1e-6) -- converged_at, every record's error /
  energy_end / mass_end / iterate norms, the serial reference, the Newton totals;
* ``c1``: BASELINE config 1 (1D m = 255, PA3, N = 16, J = 256, eps = 0.05) run(tol=1e-6);
* ``c1n``: config-1 grid with NPA1 (N = 8, J = 32, T = 0.25), run(tol=1e-6);
* ``d2`` / ``d2n``: 2D 15^2 interior grid, PA3 / NPA1, N = 4 (SuperLU in the reference).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from chparareal import grid, parareal  # noqa: E402

    out = {}

    def record(tag, g, u0, variant, part, eps):
        tr = parareal.run(grid.Field(g, u0), variant, part, eps, tol=1e-6)
        ref = parareal.serial_fine_reference(grid.Field(g, u0), variant, part, eps)
        out[f"{tag}_u0"] = u0
        out[f"{tag}_meta"] = np.array([g.nodes_per_axis, part.total_time, part.num_slices,
                                       part.fine_steps, eps])
        out[f"{tag}_converged"] = np.array([-1 if tr.converged_at is None else tr.converged_at])
        out[f"{tag}_k"] = np.array([r.k for r in tr.records])
        out[f"{tag}_error"] = np.array([r.error for r in tr.records])
        out[f"{tag}_energy"] = np.array([r.energy_end for r in tr.records])
        out[f"{tag}_mass"] = np.array([r.mass_end for r in tr.records])
        out[f"{tag}_norms"] = np.array([r.iterate_norms for r in tr.records])
        out[f"{tag}_refnorm"] = np.array([tr.reference_norm])
        out[f"{tag}_newton"] = np.array([tr.newton.steps, tr.newton.total_iterations,
                                         tr.newton.max_iterations])
        out[f"{tag}_serial"] = np.array([f.values for f in ref])
        print(tag, tr.converged_at, [f"{e:.3e}" for e in tr.errors], flush=True)

    g = grid.SpatialGrid(1, 10)
    u0 = np.random.default_rng(7).uniform(-0.1, 0.1, g.interior_count)
    for v in ("pa1", "pa2", "pa3", "npa1", "npa2"):
        record(f"spec_{v}", g, u0, parareal.AlgorithmVariant(v), parareal.TimePartition(0.5, 4, 4),
               0.1)

    g = grid.SpatialGrid(1, 257)
    x = g.interior_coordinates()
    u0 = 0.1 * np.sin(2 * np.pi * x) + np.random.default_rng(0).uniform(-0.01, 0.01, x.size)
    record("c1", g, u0, parareal.AlgorithmVariant.PA3, parareal.TimePartition(1.0, 16, 256), 0.05)
    record("c1n", g, u0, parareal.AlgorithmVariant.NPA1, parareal.TimePartition(0.25, 8, 32),
           0.05)
    g = grid.SpatialGrid(2, 17)
    u0 = np.random.default_rng(5).uniform(-0.3, 0.3, g.interior_count)
    record("d2", g, u0, parareal.AlgorithmVariant.PA3, parareal.TimePartition(0.02, 4, 8), 0.05)
    record("d2n", g, u0, parareal.AlgorithmVariant.NPA1, parareal.TimePartition(0.01, 4, 4),
           0.05)
    np.savez_compressed(os.path.join(OUT, "run_traces.npz"), **out)


if __name__ == "__main__":
    main()
