"""NN_LINEAR_A (ddm.py) on the GPU: parity margins against the reference's
golden outputs and throughput of a config-2-shaped batch.

    python tools/nn_probe.py > profiles/r01_nn_probe.json

Config-2 shape: 4096 systems (64 ICs x 64 slices) of the 1D m = 1023 grid,
8 subdomains, dt = 2^-14 (config 2's fine step), eps = 0.03.  The CPU line is
the oracle (the reference's dense-LU arithmetic) on one system.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import chp_oracle as O  # noqa: E402
from paper_2304_14074_b200 import ddm, grid, schemes  # noqa: E402

z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "nn_small.npz"))
margins = {}
for name in ["c65_s4", "c65_s4_warm", "c65_s2_th40", "c257_s8", "c1025_s8", "c129_s16_warm"]:
    nx, S, th, tol, mi, warm, dt, eps, steps = z[f"{name}/params"]
    g = grid.SpatialGrid(1, int(nx))
    p = ddm.NNParams(int(S), float(th), float(tol), int(mi), bool(warm))
    spec = ddm.nn_propagator(ddm.Decomposition(g, int(S)), p, float(dt), float(eps))
    out = schemes.propagate(grid.Field(g, z[f"{name}/u0"]), spec, int(steps))
    margins[name] = float(np.max(np.abs(out.values - z[f"{name}/out"])))

nsys, nx, S, dt, eps, steps = 4096, 1025, 8, 2.0 ** -14, 0.03, 8
g = grid.SpatialGrid(1, nx)
p = ddm.NNParams(S)
spec = ddm.nn_propagator(ddm.Decomposition(g, S), p, dt, eps)
u0 = torch.as_tensor(np.random.default_rng(0).uniform(-0.05, 0.05, (nsys, nx - 2)), device="cuda")
out = torch.empty_like(u0)
for _ in range(2):
    info = schemes.propagate_batch(g, spec, steps, u0, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    info = schemes.propagate_batch(g, spec, steps, u0, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
si = schemes.read_sysinfo(info)
assert np.all(si["status"] == 0)
sweeps = float(si["newton_total"].sum()) / (nsys * steps)

mesh = O.Mesh(1, nx)
v = u0[0].cpu().numpy()
t0 = time.perf_counter()
O.nn_advance(mesh, v, dt, eps, O.NNSetup(S), 2)
cpu_s = (time.perf_counter() - t0) / 2
gpu_out = out[0].cpu().numpy()
print(json.dumps({
    "what": "NN_LINEAR_A fine step (chp_nn_propagate), config-2 shape",
    "golden_max_abs_diff": margins,
    "batch": {"systems": nsys, "nx": nx, "n_subdomains": S, "dt": dt, "eps": eps,
              "steps": steps},
    "gpu_ms_per_launch": ms,
    "gpu_system_steps_per_s": nsys * steps / (ms * 1e-3),
    "gpu_grid_point_steps_per_s": nsys * steps * (nx - 2) / (ms * 1e-3),
    "mean_sweeps_per_step": sweeps,
    "cpu_oracle_s_per_system_step": cpu_s,
    "cpu_grid_point_steps_per_s": (nx - 2) / cpu_s,
}))
