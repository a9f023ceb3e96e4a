"""Time split of a truncated time-to-tolerance run (host wall, synchronised per phase)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from oracle.chp_oracle import CONFIGS, initial_condition  # seeded inputs only  # noqa: E402
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200.engine import PararealEngine  # noqa: E402
from paper_2304_14074_b200.grid import Field, SpatialGrid  # noqa: E402

cfg, iters = int(sys.argv[1]), int(sys.argv[2])
c = CONFIGS[cfg]
g = SpatialGrid(c["dim"], c["nx"])
part = P.TimePartition(c["T"], c["N"], c["J"])
f, co = P.propagator_pair(P.AlgorithmVariant(c["variant"]), part, c["eps"])
eng = PararealEngine(g, f, co, c["N"], c["J"], timing=True)
eng.load([Field(g, initial_condition(cfg, 0))])
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.run(max_iter=iters)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
s = eng.stats
print(json.dumps({"config": cfg, "iterations": eng.k, "wall": wall, "fine_s": s.fine_seconds,
                  "coarse_s": s.coarse_seconds, "other_s": wall - s.fine_seconds - s.coarse_seconds,
                  "fine_systems": s.fine_systems}))
