import sys, time, torch
sys.path.insert(0, '.')
import bench
from paper_2304_14074_b200 import parareal as P
from paper_2304_14074_b200.grid import Field, SpatialGrid
from paper_2304_14074_b200.distributed import ShardedParareal
from oracle.chp_oracle import initial_condition
C = bench.CFG
g = SpatialGrid(C["dim"], C["nx"]); part = P.TimePartition(C["T"], C["N"], C["J"])
fine, coarse = P.propagator_pair(P.AlgorithmVariant.PA3, part, C["eps"])
eng = ShardedParareal(g, fine, coarse, C["N"], C["J"])
eng.load(Field(g, initial_condition(5))); eng.coarse_init(); eng.iterate(force_all=True)
e = eng.eng
hU = torch.empty(e.U.shape, dtype=torch.float64, pin_memory=True); hG = torch.empty(e.G.shape, dtype=torch.float64, pin_memory=True)
hU.copy_(e.U); hG.copy_(e.G); torch.cuda.synchronize()
def T(f, n=2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f(); torch.cuda.synchronize(); a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
print("h2d U", T(lambda: e.U.copy_(hU, non_blocking=True)))
print("h2d G", T(lambda: e.G.copy_(hG, non_blocking=True)))
print("d2h U", T(lambda: hU.copy_(e.U, non_blocking=True)))
print("iterate", T(lambda: eng.iterate(force_all=True)))
print("e2e", eng.e2e_step_rate(2))
