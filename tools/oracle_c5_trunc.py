"""CPU-DST/PCG oracle run of config 5 truncated to its first 4 slices (full
1023^2 grid, eps, fine/coarse steps and seeded u0 of config 5; PA3: spectral LINEAR_B fine
steps, LINEAR_A coarse by DST-PCG), SURVEY.md 8(c) "truncated parity plan".
Writes tests/golden/config5_trunc.npz for tests/test_gpu_2d.py (~20 min of CPU)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import chp_oracle as O  # noqa: E402

c = O.CONFIGS[5]
mesh = O.Mesh(2, c["nx"])
u0 = O.initial_condition(5)
dT = c["T"] / c["N"]
N = 4
t0 = time.time()


def cb(k, inc, U):
    print(json.dumps({"k": k, "inc": inc, "t": time.time() - t0}), flush=True)


kn = O.Knobs(cube="numpy", spectral=True, pcg=True)
r = O.parareal(mesh, u0, "pa3", N * dT, N, c["J"], c["eps"], kn, on_iteration=cb)
U = r.iterates[-1]   # every 8th point kept (the full field is 8 MB)
np.savez_compressed("tests/golden/config5_trunc.npz", k=np.array([-1 if r.k is None else r.k]),
                    increments=np.array(r.increments), U_end_sub=U[::8].copy(),
                    U_end_maxabs=np.array([np.max(np.abs(U))]),
                    U_end_l2=np.array([np.sqrt(np.sum(U * U))]), seconds=np.array([r.seconds]))
print("done", r.k, r.increments, r.newton.total, r.seconds, flush=True)
