import sys, numpy as np
sys.path.insert(0, '.')
from oracle import chp_oracle as O
from paper_2304_14074_b200 import grid as G, schemes as S
z = np.load('tests/golden/config5_trunc.npz')
g = G.SpatialGrid(2, 1025); u0 = O.initial_condition(5); dt = 2.0 / 512 / 256
spec = S.PropagatorSpec(S.Scheme.LINEAR_B, dt, 0.01)
v = S.propagate(G.Field(g, u0), spec, 1024).values
print("GPU serial 1024 steps vs oracle:", np.max(np.abs(v[::8] - z["U_end_sub"])) / np.max(np.abs(z["U_end_sub"])))
w1 = S.propagate(G.Field(g, u0), spec, 1).values
o1 = O.advance(O.Mesh(2, 1025), u0, O.LINEAR_B, dt, 0.01, 1, O.Knobs(cube="numpy", spectral=True))
print("1 step:", np.max(np.abs(w1 - o1)) / np.max(np.abs(o1)))
