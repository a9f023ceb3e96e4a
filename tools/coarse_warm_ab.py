"""A/B of the 2D coarse-sweep warm start (chp_coarse_warm_start) on config 5:
coarse init + K Parareal iterations with cold and warm CG starts; per-iteration
coarse-sweep seconds, CG iterations, and the max difference of the iterates.

    python tools/coarse_warm_ab.py [K]

Needs the (rejected, reverted) warm-start patch: PararealEngine(coarse_warm=...)
and chp_coarse_warm_start are not in the tree; kept as the record of the A/B.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import chp_oracle as O  # noqa: E402
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200.engine import PararealEngine  # noqa: E402
from paper_2304_14074_b200.grid import Field, SpatialGrid  # noqa: E402
from paper_2304_14074_b200.schemes import read_sysinfo  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = O.CONFIGS[5]
g = SpatialGrid(2, cfg["nx"])
part = P.TimePartition(cfg["T"], cfg["N"], cfg["J"])
fine, coarse = P.propagator_pair(P.AlgorithmVariant.PA3, part, cfg["eps"])
u0 = O.initial_condition(5)
res = {}
finals = {}
for warm in (False, True):
    eng = PararealEngine(g, fine, coarse, cfg["N"], cfg["J"], timing=True, coarse_warm=warm)
    eng.load([Field(g, u0)])
    eng.coarse_init()
    rows = []
    for k in range(K):
        c0 = eng.stats.coarse_seconds
        eng.info_coarse.zero_()
        inc = eng.iterate()
        si = read_sysinfo(eng.info_coarse)
        rows.append({"k": k + 1, "coarse_s": eng.stats.coarse_seconds - c0,
                     "cg_total": int(si["cg_total"][0]), "cg_max": int(si["cg_max"][0]),
                     "inc": float(np.max(inc))})
    finals[warm] = eng.U.clone().cpu()
    res["warm" if warm else "cold"] = rows
    del eng
    torch.cuda.empty_cache()
res["max_abs_diff_final_iterates"] = float((finals[True] - finals[False]).abs().max())
print(json.dumps(res))
