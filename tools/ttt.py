"""Parareal time-to-tolerance on one B200 for BASELINE configs 1-5
(increment stop max|U^{k+1}-U^k| < 1e-10).  Usage: python tools/ttt.py 1 2 3"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_14074_b200.configs import CONFIGS, initial_condition  # noqa: E402
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200.engine import PararealEngine  # noqa: E402
from paper_2304_14074_b200.grid import Field, SpatialGrid  # noqa: E402


def run(cfg: int, max_iter=None, n_ic=None):
    c = CONFIGS[cfg]
    g = SpatialGrid(c["dim"], c["nx"])
    B = n_ic or c.get("batch", 1)
    part = P.TimePartition(c["T"], c["N"], c["J"])
    f, co = P.propagator_pair(P.AlgorithmVariant(c["variant"]), part, c["eps"])
    eng = PararealEngine(g, f, co, c["N"], c["J"], batch=B)
    eng.load([Field(g, initial_condition(cfg, b)) for b in range(B)])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    conv = eng.run(max_iter=max_iter)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    incs = np.array(eng.increments)
    return {"config": cfg, "variant": c["variant"], "ics": B, "k": conv,
            "iterations_run": eng.k, "seconds": wall,
            "fine_point_steps": eng.stats.fine_point_steps,
            "fine_slice_propagations": eng.stats.fine_systems,
            "fine_rate": eng.stats.fine_point_steps / wall,
            "newton_steps": eng.newton.steps, "newton_total": eng.newton.total_iterations,
            "last_increments": incs[-4:, 0].tolist() if incs.size else [],
            "increments_ic0": incs[:, 0].tolist() if incs.size else []}


if __name__ == "__main__":
    for a in sys.argv[1:]:
        cfg, _, mi = a.partition(":")
        print(json.dumps(run(int(cfg), int(mi) if mi else None)), flush=True)
