"""Kernel micro-timings on the GPU (CUDA events): 2D LINEAR_B fine propagator,
2D LINEAR_A PCG coarse step, 1D propagators.  Usage: python tools/kbench.py [what]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2304_14074_b200 import schemes as S  # noqa: E402
from paper_2304_14074_b200.grid import SpatialGrid, to_device_layout  # noqa: E402


def ev_time(fn, reps=3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def fields(g, n, seed=0, base=0.0):
    rng = np.random.default_rng(seed)
    flat = torch.tensor(base + rng.uniform(-0.05, 0.05, (n, g.interior_count)), device="cuda")
    return torch.stack([to_device_layout(g, flat[i]) for i in range(n)])


def linb_2d(nx=1025, nsys=64, steps=16):
    g = SpatialGrid(2, nx)
    src = fields(g, nsys, base=0.1)
    out = torch.empty_like(src)
    spec = S.PropagatorSpec(S.Scheme.LINEAR_B, 2.0 / 512 / 256, 0.01)
    ms = ev_time(lambda: S.propagate_batch(g, spec, steps, src, out))
    pts = nsys * steps * g.interior_count
    return {"what": "2D LINEAR_B", "nx": nx, "nsys": nsys, "steps": steps, "ms": ms,
            "pt_steps_per_s": pts / (ms * 1e-3), "GBps_at_32B": 32 * pts / (ms * 1e-3) / 1e9}


def lina_2d(nx=1025, nsys=1):
    g = SpatialGrid(2, nx)
    src = fields(g, nsys, base=0.1)
    out = torch.empty_like(src)
    spec = S.PropagatorSpec(S.Scheme.LINEAR_A, 2.0 / 512, 0.01)
    info = S.new_sysinfo(nsys, "cuda")
    ms = ev_time(lambda: S.propagate_batch(g, spec, 1, src, out, info=info), reps=3)
    si = S.read_sysinfo(info)
    return {"what": "2D LINEAR_A PCG", "nx": nx, "nsys": nsys, "ms": ms,
            "cg_iters": int(si["cg_total"][0]) / 4}


def one_d(nx, nsys, scheme, dt, eps, steps):
    g = SpatialGrid(1, nx)
    src = torch.tensor(np.random.default_rng(0).uniform(-0.05, 0.05, (nsys, nx - 2)), device="cuda")
    out = torch.empty_like(src)
    spec = S.PropagatorSpec(scheme, dt, eps)
    ms = ev_time(lambda: S.propagate_batch(g, spec, steps, src, out), reps=2)
    pts = nsys * steps * (nx - 2)
    return {"what": f"1D {scheme.value}", "nx": nx, "nsys": nsys, "steps": steps, "ms": ms,
            "pt_steps_per_s": pts / (ms * 1e-3)}


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    res = []
    if what == "linb":                       # short case for ncu
        res.append(linb_2d(1025, 32, 4))
    if what in ("all", "2d"):
        res.append(linb_2d(1025, 64, 16))
        res.append(linb_2d(257, 64, 64))
        res.append(lina_2d(1025, 1))
        res.append(lina_2d(257, 1))
    if what in ("all", "1d"):
        res.append(one_d(257, 16, S.Scheme.LINEAR_B, 2.0 ** -12, 0.05, 256))
        res.append(one_d(1025, 4096, S.Scheme.NONLINEAR_EYRE, 2.0 ** -15, 0.03, 16))
        res.append(one_d(1025, 64, S.Scheme.LINEAR_A, 2.0 ** -5, 0.03, 1))
    for r in res:
        print(json.dumps(r), flush=True)


def coarse_sweep(nx=1025, nsl=8):
    """Device coarse sweep (cooperative LINEAR_A kernel): ms per slice."""
    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.engine import PararealEngine
    from paper_2304_14074_b200.grid import Field
    g = SpatialGrid(2, nx)
    part = P.TimePartition(2.0 / 512 * nsl, nsl, 1)
    f, c = P.propagator_pair(P.AlgorithmVariant.PA3, part, 0.01)
    eng = PararealEngine(g, f, c, nsl, 1)
    eng.load([Field(g, 0.1 + np.random.default_rng(0).uniform(-0.05, 0.05, g.interior_count))])
    ms = ev_time(lambda: eng.coarse_init(), reps=2)
    si = S.read_sysinfo(eng.info_coarse)
    return {"what": "2D coarse sweep (mode 0)", "nx": nx, "slices": nsl, "ms": ms,
            "ms_per_slice": ms / nsl, "cg_total": int(si["cg_total"][0])}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "coarse":
    print(json.dumps(coarse_sweep()), flush=True)
    print(json.dumps(coarse_sweep(1025, 64)), flush=True)


def coarse_trace(nx=1025, nsl=4):
    """Per-phase timeline of the cooperative coarse kernel (CHP_COOP_TRACE=1)."""
    import ctypes
    os.environ["CHP_COOP_TRACE"] = "1"
    from paper_2304_14074_b200 import _native as NN
    r = coarse_sweep(nx, nsl)
    buf = (ctypes.c_ulonglong * 4096)()
    n = NN.lib().chp_debug_trace(buf, 4096)
    ts = np.array(buf[:n], dtype=np.int64)
    ts = ts[ts > 0]
    d = np.diff(ts) / 1e3
    return {"coarse": r, "barriers": int(ts.size), "phase_us": [round(x, 1) for x in d[:80]]}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "trace":
    print(json.dumps(coarse_trace()), flush=True)


def kernel_split(nx=1025, nsys=64, steps=16):
    """Per-kernel average device time (torch profiler) of the LINEAR_B propagation."""
    from torch.profiler import profile, ProfilerActivity
    g = SpatialGrid(2, nx)
    src = fields(g, nsys, base=0.1)
    out = torch.empty_like(src)
    spec = S.PropagatorSpec(S.Scheme.LINEAR_B, 2.0 / 512 / 256, 0.01)
    S.propagate_batch(g, spec, steps, src, out)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        S.propagate_batch(g, spec, steps, src, out)
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            k = e.name[:60]
            t, c = agg.get(k, (0.0, 0))
            agg[k] = (t + e.device_time, c + 1)
    return {k: {"us_avg": round(t / c, 1), "n": c} for k, (t, c) in agg.items()}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "split":
    print(json.dumps(kernel_split()), flush=True)
    print(json.dumps(kernel_split(257, 64, 64)), flush=True)


def coarse_ft(nx=1025, nsl=2):
    """Inside-the-phase clock64 stamps of block 0 / thread 0 (library built with -DCHP_C2_FT)."""
    import ctypes
    os.environ["CHP_COOP_TRACE"] = "1"
    from paper_2304_14074_b200 import _native as NN
    r = coarse_sweep(nx, nsl)
    n = 4096 * 9
    buf = (ctypes.c_ulonglong * n)()
    NN.lib().chp_debug_trace(buf, n)
    a = np.array(buf[:n], dtype=np.int64)
    ft = a[4096:].reshape(4096, 8)
    rows = []
    for g in range(1, 4095):
        if ft[g, 0] == 0 or ft[g + 1, 0] == 0:
            continue
        st = ft[g]
        nxt = ft[g + 1, 0]
        rows.append({"gen": g, "clk": [int(st[k] - st[0]) if st[k] else None for k in range(1, 6)],
                     "next_exit": int(nxt - st[0])})
    lo = int(os.environ.get("FT_LO", "40"))
    return {"coarse": r, "phases": rows[lo:lo + int(os.environ.get("FT_N", "24"))]}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ft":
    print(json.dumps(coarse_ft()), flush=True)
