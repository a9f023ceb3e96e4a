"""Envelope between the unmodified reference's arithmetic (SuperLU LINEAR_B, numpy
cube) and the CPU-DST oracle over the serial fine propagation that the converged
truncated config-5 run equals (4 slices x 256 steps at 1023^2): SURVEY.md 8(c)
tier T3, E_env.  ~20 min of CPU; prints one JSON line."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import chp_oracle as O  # noqa: E402

z = np.load("tests/golden/config5_trunc.npz")
mesh = O.Mesh(2, 1025)
u0 = O.initial_condition(5)
dt = 2.0 / 512 / 256
t0 = time.time()
v = O.advance(mesh, u0, O.LINEAR_B, dt, 0.01, 1024, O.Knobs(cube="numpy", spectral=False))
sub = v[::8]
env = float(np.max(np.abs(sub - z["U_end_sub"])) / np.max(np.abs(z["U_end_sub"])))
print(json.dumps({"E_env_superlu_vs_dst": env, "steps": 1024, "seconds": time.time() - t0}),
      flush=True)
