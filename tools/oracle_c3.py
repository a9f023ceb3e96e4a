"""CPU oracle run of config 3 in full (PA3, spectral LINEAR_B as the CPU-DST
oracle, SuperLU LINEAR_A as the reference) -- long (hours); writes
tests/golden/config3_oracle.npz for the GPU parity test of the full config."""
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
    print(json.dumps({"k": k, "inc": inc, "t": time.time() - t0}), flush=True)
    np.savez_compressed("tests/golden/config3_oracle_partial.npz", k=k, U_last=U[-1])


r = O.parareal(mesh, u0, "pa3", c["T"], c["N"], c["J"], c["eps"],
               O.Knobs(cube="numpy", spectral=True), on_iteration=cb)
np.savez_compressed("tests/golden/config3_oracle.npz", k=np.array([-1 if r.k is None else r.k]),
                    increments=np.array(r.increments), U_end=r.iterates[-1],
                    U_mid=r.iterates[32], seconds=np.array([r.seconds]))
print("done", r.k, r.seconds, flush=True)
