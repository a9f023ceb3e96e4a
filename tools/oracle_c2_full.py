"""CPU oracle run of config 2 in full for one initial condition (NPA1, 1D m = 1023,
eps 0.03, T = 2, N = 64, J = 512, Newton tol 1e-10), SURVEY.md 8(c) parity plan.

Runs the oracle with cube="exact" (the 1D device kernels are bit-identical to it) to the
increment stop and writes tests/golden/config2_ic{IC}.npz: k, every increment, the Newton
totals, the final iterate U_N and a SHA-256 of all N+1 final iterates (the GPU test
asserts bit identity through the digest).  ~15-25 min of one CPU core per IC.

usage: python tools/oracle_c2_full.py IC
"""
import hashlib
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import chp_oracle as O  # noqa: E402

ic = int(sys.argv[1])
c = O.CONFIGS[2]
mesh = O.Mesh(1, c["nx"])
u0 = O.initial_condition(2, ic)
t0 = time.time()


def cb(k, inc, U):
    print(json.dumps({"ic": ic, "k": k, "inc": inc, "t": round(time.time() - t0, 1)}), flush=True)


r = O.parareal(mesh, u0, c["variant"], c["T"], c["N"], c["J"], c["eps"],
               O.Knobs(cube="exact"), on_iteration=cb)
U = np.ascontiguousarray(r.iterates)
np.savez_compressed(f"tests/golden/config2_ic{ic}.npz",
                    k=np.array([-1 if r.k is None else r.k]), increments=np.array(r.increments),
                    U_end=U[-1].copy(), U_mid=U[32].copy(),
                    sha256=np.frombuffer(hashlib.sha256(U.tobytes()).digest(), np.uint8),
                    newton=np.array([r.newton.steps, r.newton.total, r.newton.max_iter]),
                    fine_props=np.array([r.fine_props]), seconds=np.array([r.seconds]))
print("done", ic, r.k, r.newton.total, r.seconds, flush=True)
