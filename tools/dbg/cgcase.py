import sys, numpy as np
sys.path.insert(0, ".")
from paper_2304_14074_b200 import grid as G, parareal as P, schemes as S
from paper_2304_14074_b200.engine import PararealEngine
g = G.SpatialGrid(2, 33)
u0 = np.random.default_rng(4).uniform(-0.05, 0.05, g.interior_count)
part = P.TimePartition(0.02, 4, 8)
f, c = P.propagator_pair(P.AlgorithmVariant("pa3"), part, 0.05)
eng = PararealEngine(g, f, c, 4, 8)
eng.load([G.Field(g, u0)])
try:
    eng.coarse_init()
except Exception as e:
    print("coarse_init", e)
print("coarse sysinfo", S.read_sysinfo(eng.info_coarse))
try:
    eng.run()
    print("k", eng.converged_at)
except Exception as e:
    print("run", e)
print("coarse sysinfo", S.read_sysinfo(eng.info_coarse))
