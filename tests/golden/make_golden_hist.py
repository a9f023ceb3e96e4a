"""Golden StepReport.residual_history of the reference's step_nonlinear
(schemes.py:270-305).  Build container only (imports /root/reference):

    python tests/golden/make_golden_hist.py   -> tests/golden/newton_hist.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from chparareal import grid, schemes  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [("d1", 1, 129, 2.0 ** -10, 0.05, 1), ("d1b", 1, 257, 2.0 ** -8, 0.03, 2),
         ("d2", 2, 33, 2.0 ** -10, 0.05, 3)]
out = {}
for name, dim, nx, dt, eps, seed in CASES:
    g = grid.SpatialGrid(dim=dim, nodes_per_axis=nx)
    u0 = np.random.default_rng(seed).uniform(-0.6, 0.6, g.interior_count)
    spec = schemes.PropagatorSpec(schemes.Scheme.NONLINEAR_EYRE, dt, eps)
    f, rep = schemes.step_nonlinear(grid.Field(g, u0), spec)
    out[f"{name}/params"] = np.array([dim, nx, dt, eps])
    out[f"{name}/u0"] = u0
    out[f"{name}/out"] = f.values
    out[f"{name}/hist"] = np.array(rep.residual_history)
    print(name, rep.newton_iterations, rep.residual_history)
np.savez_compressed(os.path.join(OUT, "newton_hist.npz"), **out)
