"""One config-2-shaped 1D Newton launch (4096 systems x 4 steps) for ncu."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_14074_b200 import schemes as S  # noqa: E402
from paper_2304_14074_b200.grid import SpatialGrid  # noqa: E402

g = SpatialGrid(1, 1025)
src = torch.tensor(np.random.default_rng(0).uniform(-0.05, 0.05, (4096, 1023)), device="cuda")
out = torch.empty_like(src)
spec = S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, 2.0 ** -15, 0.03)
S.propagate_batch(g, spec, 4, src, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
S.propagate_batch(g, spec, 4, src, out)
b.record()
torch.cuda.synchronize()
print(json.dumps({"ms_per_step": a.elapsed_time(b) / 4}))
