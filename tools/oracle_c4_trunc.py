"""CPU-DST/PCG oracle run of config 4 truncated to its first 4 slices (full
511^2 grid, eps, fine/coarse steps and seeded u0 of config 4; NPA1: Newton fine
steps to 1e-10, LINEAR_A coarse), SURVEY.md 8(c) "truncated parity plan".
Writes tests/golden/config4_trunc.npz for tests/test_gpu_2d.py (~10 min of CPU)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import chp_oracle as O  # noqa: E402

c = O.CONFIGS[4]
mesh = O.Mesh(2, c["nx"])
u0 = O.initial_condition(4)
dT = c["T"] / c["N"]
N = 4
t0 = time.time()


def cb(k, inc, U):
    print(json.dumps({"k": k, "inc": inc, "t": time.time() - t0}), flush=True)


kn = O.Knobs(cube="numpy", spectral=True, pcg=True)
r = O.parareal(mesh, u0, "npa1", N * dT, N, c["J"], c["eps"], kn, on_iteration=cb)
np.savez_compressed("tests/golden/config4_trunc.npz", k=np.array([-1 if r.k is None else r.k]),
                    increments=np.array(r.increments), U_end=r.iterates[-1],
                    newton_total=np.array([r.newton.total]),
                    newton_steps=np.array([r.newton.steps]), seconds=np.array([r.seconds]))
print("done", r.k, r.increments, r.newton.total, r.seconds, flush=True)
