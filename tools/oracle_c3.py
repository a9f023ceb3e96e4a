"""CPU oracle run of config 3 in full (PA3 at 255^2, eps 0.02, T 0.5, N 64, J 128): the
CPU-DST oracle of SURVEY.md 8(c) -- spectral LINEAR_B fine steps, LINEAR_A coarse solves
by DST-preconditioned CG to 1e-14 (pcg=True, the solve the GPU runs) -- iterated to the
increment stop.  Writes tests/golden/config3_full.npz (k, every increment, final and middle
iterates) for tests/test_gpu_parity_full.py.  ~30-60 min of CPU."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import chp_oracle as O  # noqa: E402

c = O.CONFIGS[3]
mesh = O.Mesh(2, c["nx"])
u0 = O.initial_condition(3)
t0 = time.time()


def cb(k, inc, U):
    print(json.dumps({"k": k, "inc": inc, "t": round(time.time() - t0, 1)}), flush=True)


r = O.parareal(mesh, u0, "pa3", c["T"], c["N"], c["J"], c["eps"],
               O.Knobs(cube="numpy", spectral=True, pcg=True), on_iteration=cb)
np.savez_compressed("tests/golden/config3_full.npz", k=np.array([-1 if r.k is None else r.k]),
                    increments=np.array(r.increments), U_end=r.iterates[-1],
                    U_mid=r.iterates[32], seconds=np.array([r.seconds]),
                    fine_props=np.array([r.fine_props]))
print("done", r.k, r.seconds, flush=True)
