"""Accuracy of the 2D LINEAR_B fine step (schemes.py:249-267) at the config-5 grid against an
extended-precision truth (SURVEY.md 8(c) tier T3).

  python tools/linb_truth.py gpu [tag]  -- on the GPU box: 1 and 64 LINEAR_B steps of config 5's
                                           seeded u0 -> gpurun_out/linb_gpu[_tag].npz
  python tools/linb_truth.py cpu [tag]  -- here: the same steps in x87 long double (scipy.fft
                                           long-double DST-I, long-double stencil, cube and
                                           divisors) and in fp64 by the CPU-DST oracle and the
                                           reference's SuperLU arithmetic; writes the test
                                           fixture tests/golden/config5_truth.npz (~30 min);
                                           prints/writes the relative max-norm errors of each
                                           against the long-double truth.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import chp_oracle as O  # noqa: E402

NX, EPS, DT = 1025, 0.01, 2.0 / 512 / 256
STEPS = (1, 64, 256, 1024)


def gpu(tag):
    from paper_2304_14074_b200 import grid as G, schemes as S
    g = G.SpatialGrid(2, NX)
    u0 = O.initial_condition(5)
    spec = S.PropagatorSpec(S.Scheme.LINEAR_B, DT, EPS)
    out = {f"s{k}": S.propagate(G.Field(g, u0), spec, k).values for k in STEPS}
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed(f"gpurun_out/linb_gpu{tag}.npz", **out)


def ld_step(v, lam2, cdt, dt):
    """One LINEAR_B step in long double: rhs = v + dt L(v^3 - 3v), x = S D S rhs."""
    import scipy.fft as sfft
    m = v.shape[0]
    w = v * v * v - 3 * v
    Lw = -4 * w
    Lw[1:, :] += w[:-1, :]
    Lw[:-1, :] += w[1:, :]
    Lw[:, 1:] += w[:, :-1]
    Lw[:, :-1] += w[:, 1:]
    rhs = v + cdt * Lw
    r = sfft.dstn(rhs, type=1, norm="ortho")
    return sfft.dstn(r / lam2, type=1, norm="ortho").reshape(m, m)


def cpu(tag):
    ld = np.longdouble
    mesh = O.Mesh(2, NX)
    m = mesh.m
    u0 = O.initial_condition(5)
    h = ld(1) / ld(NX - 1)
    p = np.arange(1, NX - 1, dtype=ld)
    lam = -4 / (h * h) * np.sin(p * ld(np.pi) / (2 * (NX - 1))) ** 2
    # pi in long double: np.pi is a double; refine with the long-double arctan identity
    pi_ld = 4 * np.arctan(ld(1))
    lam = -4 / (h * h) * np.sin(p * pi_ld / (2 * (NX - 1))) ** 2
    x = lam[:, None] + lam[None, :]
    dt = ld(DT)
    b64 = ld(EPS ** 2) * dt
    lam2 = (1 - 2 * dt * x) + b64 * x * x
    cdt = dt / (h * h)
    v = u0.reshape(m, m).astype(ld)
    truth = {}
    t0 = time.time()
    for k in range(1, max(STEPS) + 1):
        v = ld_step(v, lam2, cdt, dt)
        if k in STEPS:
            truth[k] = v.reshape(-1).copy()
    t_truth = time.time() - t0
    res = {"grid": "1023^2", "steps": list(STEPS), "truth": "x87 long double (64-bit mantissa)",
           "truth_seconds": round(t_truth, 1)}
    def errs(tag, k, v):
        tr = truth[k].astype(np.float64)
        res[f"{tag}_{k}"] = float(np.max(np.abs(v - tr)) / np.max(np.abs(tr)))
        res[f"{tag}_{k}_sub8"] = float(np.max(np.abs(v[::8] - tr[::8])) / np.max(np.abs(tr[::8])))

    kn = O.Knobs(cube="numpy", spectral=True)
    o = u0
    for k in range(1, max(STEPS) + 1):
        o = O.advance(mesh, o, O.LINEAR_B, DT, EPS, 1, kn)
        if k in STEPS:
            errs("oracle_dst", k, o)
    # the unmodified reference's arithmetic (SuperLU cached factor, numpy cube)
    sl = u0
    for k in range(1, max(STEPS) + 1):
        sl = O.advance(mesh, sl, O.LINEAR_B, DT, EPS, 1, O.Knobs(cube="numpy"))
        if k in STEPS:
            errs("reference_superlu", k, sl)
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed("gpurun_out/linb_truth.npz",
                        **{f"t{k}": truth[k].astype(np.float64) for k in STEPS})
    # test fixture (tests/test_gpu_2d.py): every 8th value of the truth after 256 and
    # 1024 steps, and the fp64 CPU paths' errors against it on the same subsample
    fx = {f"truth{k}_sub8": truth[k].astype(np.float64)[::8].copy() for k in (256, 1024)}
    for k in (256, 1024):
        for tag in ("oracle_dst", "reference_superlu"):
            fx[f"{tag}_{k}_sub8"] = np.array([res[f"{tag}_{k}_sub8"]])
    np.savez_compressed("tests/golden/config5_truth.npz", **fx)
    f = f"gpurun_out/linb_gpu{tag}.npz"
    if os.path.exists(f):
        z = np.load(f)
        for k in STEPS:
            errs("gpu", k, z[f"s{k}"])
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    mode = sys.argv[1]
    tag = sys.argv[2] if len(sys.argv) > 2 else ""
    (gpu if mode == "gpu" else cpu)(tag)
