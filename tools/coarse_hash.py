"""Hashes of the engine state after a coarse init and two Parareal iterations (kernel-variant
bit-identity check: run once per CHP_LIB and compare).  Usage: python tools/coarse_hash.py [nx]"""
import hashlib
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200.engine import PararealEngine  # noqa: E402
from paper_2304_14074_b200.grid import Field, SpatialGrid  # noqa: E402

out = {}
for nx in ([int(sys.argv[1])] if len(sys.argv) > 1 else [1025, 513, 257, 65]):
    g = SpatialGrid(2, nx)
    nsl = 4
    part = P.TimePartition(2.0 / 512 * nsl, nsl, 2)
    f, c = P.propagator_pair(P.AlgorithmVariant.PA3, part, 0.01)
    eng = PararealEngine(g, f, c, nsl, 2)
    eng.load([Field(g, 0.1 + np.random.default_rng(0).uniform(-0.05, 0.05, g.interior_count))])
    eng.coarse_init()
    incs = [float(eng.iterate()[0]) for _ in range(2)]
    h = hashlib.sha256(eng.U.cpu().numpy().tobytes() + eng.G.cpu().numpy().tobytes()).hexdigest()
    out[nx] = {"hash": h[:16], "inc": incs}
print(json.dumps(out))
