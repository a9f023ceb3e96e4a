"""Small end-to-end cases for compute-sanitizer (one tool per run)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2304_14074_b200 import parareal as P  # noqa: E402
from paper_2304_14074_b200 import schemes as S  # noqa: E402
from paper_2304_14074_b200.grid import Field, SpatialGrid  # noqa: E402

rng = np.random.default_rng(0)
# 1D: every scheme, batched
g1 = SpatialGrid(1, 33)
for sch in (S.Scheme.LINEAR_A, S.Scheme.LINEAR_B, S.Scheme.NONLINEAR_EYRE):
    S.propagate(Field(g1, rng.uniform(-0.5, 0.5, 31)), S.PropagatorSpec(sch, 1e-3, 0.1), 3)
P.run(Field(g1, rng.uniform(-0.1, 0.1, 31)), P.AlgorithmVariant.NPA1, P.TimePartition(0.02, 4, 4),
      0.1, stop="increment")
# 2D: LINEAR_B passes, host PCG, Newton, cooperative coarse sweep
g2 = SpatialGrid(2, 33)
for sch in (S.Scheme.LINEAR_A, S.Scheme.LINEAR_B, S.Scheme.NONLINEAR_EYRE):
    S.propagate(Field(g2, rng.uniform(-0.5, 0.5, g2.interior_count)), S.PropagatorSpec(sch, 1e-3, 0.05), 2)
P.run(Field(g2, rng.uniform(-0.05, 0.05, g2.interior_count)), P.AlgorithmVariant.PA3,
      P.TimePartition(0.02, 4, 4), 0.05, stop="increment")
g3 = SpatialGrid(2, 129)
S.propagate(Field(g3, rng.uniform(-0.5, 0.5, g3.interior_count)), S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-4, 0.02), 2)
# N = 1024: bulk-copy row fill, TMA tile fill and TMA store of the column pass
g4 = SpatialGrid(2, 1025)
S.propagate(Field(g4, rng.uniform(-0.5, 0.5, g4.interior_count)), S.PropagatorSpec(S.Scheme.LINEAR_B, 1e-5, 0.01), 2)
print("sanitize cases done")
