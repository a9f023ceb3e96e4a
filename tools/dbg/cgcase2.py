import sys, numpy as np
sys.path.insert(0, ".")
from paper_2304_14074_b200 import grid as G, parareal as P, schemes as S
from paper_2304_14074_b200.engine import PararealEngine
pre = sys.argv[1] if len(sys.argv) > 1 else "none"
g = G.SpatialGrid(2, 33)
if pre != "none":
    v = np.random.default_rng(11).uniform(-0.1, 0.1, g.interior_count)
    schs = {"a": [S.Scheme.LINEAR_A], "b": [S.Scheme.LINEAR_B], "n": [S.Scheme.NONLINEAR_EYRE]}[pre]
    for dt in [1e-3, 1e-2, 1e-1, 1.0]:
        for sch in schs:
            u = G.Field(g, v)
            for _ in range(50):
                u = S.propagate(u, S.PropagatorSpec(sch, dt, 0.1), 1)
u0 = np.random.default_rng(4).uniform(-0.05, 0.05, g.interior_count)
part = P.TimePartition(0.02, 4, 8)
f, c = P.propagator_pair(P.AlgorithmVariant("pa3"), part, 0.05)
eng = PararealEngine(g, f, c, 4, 8)
eng.load([G.Field(g, u0)])
try:
    eng.coarse_init(); print(pre, "coarse ok", S.read_sysinfo(eng.info_coarse))
except Exception as e:
    print(pre, "coarse_init FAIL", e, S.read_sysinfo(eng.info_coarse))
