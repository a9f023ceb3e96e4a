"""A/B of the e2e step's copy pipelining on config 5 (one GPU):
python tools/e2e_ab.py -> one JSON line per (chunks, coarse_chunked)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import chp_oracle as O  # noqa: E402
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200.distributed import ShardedParareal  # noqa: E402
from paper_2304_14074_b200.grid import Field, SpatialGrid  # noqa: E402

cfg = O.CONFIGS[5]
g = SpatialGrid(2, cfg["nx"])
part = P.TimePartition(cfg["T"], cfg["N"], cfg["J"])
fine, coarse = P.propagator_pair(P.AlgorithmVariant.PA3, part, cfg["eps"])
eng = ShardedParareal(g, fine, coarse, cfg["N"], cfg["J"])
eng.load(Field(g, O.initial_condition(5)))
eng.coarse_init()
for ch, cc in [(2, True), (3, True), (4, True), (2, True), (4, True)]:
    r = eng.e2e_step_rate(2, chunks=ch, coarse_chunked=cc)
    print(json.dumps({"chunks": ch, "coarse_chunked": cc, "ms": r["ms_per_step"],
                      "value": r["value"]}), flush=True)
