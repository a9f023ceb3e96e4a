"""Full-length parity pins of the BASELINE configs on the B200 (added
row N1): the whole Parareal run to the increment stop against the CPU oracle run of the
same full config (tools/oracle_c2_full.py, tools/oracle_c3.py -> tests/golden/).

* config 2 (1D NPA1, 64 ICs, N = 64, J = 512, Newton tol 1e-10): the device run of all
  64 ICs; for every IC with a golden, the same k (65) and increments, and the final
  iterates (all 65 x 1023 values) bit-identical to the oracle (cube="exact"), checked
  through a SHA-256 of the iterate array.
* config 3 (2D PA3, 255^2, N = 64, J = 128): the same k and final iterate within 1e-10
  relative max-norm of the CPU-DST/PCG oracle; the borderline last increment
   is reported in the assertion message.
"""

import glob
import hashlib
import os

import numpy as np
import pytest

from oracle import chp_oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_14074_b200 import grid, parareal
    return parareal, grid


def test_config2_full_bitwise(P):
    PP, G = P
    files = sorted(glob.glob(os.path.join(GOLD, "config2_ic*.npz")))
    assert files, "config-2 goldens missing"
    c = O.CONFIGS[2]
    g = G.SpatialGrid(1, c["nx"])
    u0s = [G.Field(g, O.initial_condition(2, b)) for b in range(c["batch"])]
    res = PP.run_batch(u0s, PP.AlgorithmVariant.NPA1, PP.TimePartition(c["T"], c["N"], c["J"]),
                       c["eps"])
    assert all(k == c["N"] + 1 for k in res.converged_at), res.converged_at
    for f in files:
        z = np.load(f)
        b = int(os.path.basename(f)[len("config2_ic"):-4])
        assert res.converged_at[b] == int(z["k"][0])
        incs = res.increments[:, b][:len(z["increments"])]
        assert np.array_equal(incs, z["increments"]), b
        U = np.ascontiguousarray(res.engine.iterates_host(b))
        assert np.array_equal(U[-1], z["U_end"]), b
        assert hashlib.sha256(U.tobytes()).digest() == bytes(z["sha256"]), b


def test_config3_full(P):
    PP, G = P
    f = os.path.join(GOLD, "config3_full.npz")
    if not os.path.exists(f):
        pytest.skip("config-3 oracle golden not generated")
    z = np.load(f)
    c = O.CONFIGS[3]
    g = G.SpatialGrid(2, c["nx"])
    tr = PP.run(G.Field(g, O.initial_condition(3)), PP.AlgorithmVariant.PA3,
                PP.TimePartition(c["T"], c["N"], c["J"]), c["eps"], stop="increment")
    k_ref = int(z["k"][0])
    inc = np.array(tr.increments)
    assert tr.converged_at == k_ref, (tr.converged_at, k_ref, inc[-3:], z["increments"][-3:])
    eng_U = np.array(tr.records[-1].iterate_norms)
    assert eng_U.shape[0] == c["N"] + 1
    U = tr.engine.iterates_host(0)
    scale = np.max(np.abs(z["U_end"]))
    assert np.max(np.abs(U[-1] - z["U_end"])) / scale < 1e-10
    assert np.max(np.abs(U[c["N"] // 2] - z["U_mid"])) / scale < 1e-10
