"""Benchmark: fine grid-point-steps/s (fp64) of the Parareal fine propagator +
coarse sweep on BASELINE.json config 5 (2D 1023^2 PA3, eps=0.01, T=2, N=512
slices, J=256 fine steps), the largest single-GPU configuration.

A step = one full Parareal iteration (parareal.py:216-259) with every slice
active: one batched fine launch sequence over all 512 slices (2J+1 passes) +
the sequential device coarse sweep + correction + increment.  value = fine
grid-point-steps computed / step time.  Inputs (13 GB of iterates) are far
larger than L2, so no explicit flush is needed between steps.

--impl reference times the reference's CPU arithmetic (the oracle port, which
calls the same scipy SuperLU routines as the reference) on a bounded sample.

Also on the line: ``time_to_tolerance`` -- full
Parareal runs of configs 1, 2 (64 ICs) and 3 to the increment stop on the same
GPUs in the same run (``--ttt`` selects configs; 4 and 5 take minutes), with k and
the fine work; ``fp64`` -- a measured DFMA peak and the 1D configs' flop-model
fractions; ``cpu_baselines`` -- the reference's arithmetic per config on this
host's cores (config 1 in full at 1 and all workers, configs 2/3 per-step samples
with the labelled extrapolation of SURVEY.md 8(d)); ``coarse_cg_per_step``.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(dim=2, nx=1025, eps=0.01, T=2.0, N=512, J=256, variant="pa3")
METRIC = "fine grid-point-steps/s (fp64)"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k] == "Active"})
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        pw = [num(r[6]) for r in rows if len(r) > 7 and num(r[6]) is not None]
        pl = [num(r[7]) for r in rows if len(r) > 7 and num(r[7]) is not None]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows),
                "power_w": float(np.median(pw)) if pw else None,
                "power_limit_w": max(pl) if pl else None}


def count_launches(fn):
    """Kernels of libchp.so launched by fn() (torch profiler / CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = {}
    for ev in prof.events():
        nm = ev.name
        if any(s in nm for s in ("k2d_", "k1d_", "k_max_abs_diff")):
            short = nm.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0]
            names[short] = names.get(short, 0) + 1
    return sum(names.values()), names


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


def cpu_sample(seconds_target: float = 15.0, workers: int = 1) -> dict:
    """Reference arithmetic on the host: LINEAR_B fine steps at 1023^2 through
    the oracle port (same scipy SuperLU factor + solve as schemes.py:218-224).
    With workers > 1 it mirrors the reference's own parallelism: a thread pool
    over slices (parareal.py:239-241) sharing the cached factor behind a lock
    (schemes.py:220-224)."""
    import threading
    from concurrent.futures import ThreadPoolExecutor

    from oracle import chp_oracle as O
    mesh = O.Mesh(2, CFG["nx"])
    dt = CFG["T"] / CFG["N"] / CFG["J"]
    kn = O.Knobs(cube="numpy")
    t0 = time.perf_counter()
    O.advance(mesh, O.initial_condition(5), O.LINEAR_B, dt, CFG["eps"], 1, kn)  # factor (cached)
    t_fact = time.perf_counter() - t0
    ops = O.operators(mesh)
    solve = O.constant_solver(ops, dt, CFG["eps"], False)
    lock = threading.Lock()

    def slice_worker(seed):
        v = O.initial_condition(5, seed)
        n = 0
        t_end = time.perf_counter() + seconds_target
        while time.perf_counter() < t_end or n < 2:
            rhs = v + dt * (ops.L @ (v ** 3 - 3.0 * v))          # schemes.py:260
            with lock:                                           # schemes.py:223-224
                v = solve(rhs)
            n += 1
        return n

    t0 = time.perf_counter()
    if workers > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            steps = sum(pool.map(slice_worker, range(workers)))
    else:
        steps = slice_worker(0)
    el = time.perf_counter() - t0
    return {"value": steps * mesh.size / el, "unit": "grid-point-steps/s", "cores": workers,
            "kind": "port",
            "sample": f"{steps} LINEAR_B fine steps of 1023^2 slices over {workers} thread(s) "
                      f"(scipy SuperLU cached factor behind the reference's lock; "
                      f"factorisation {t_fact:.1f} s excluded)",
            "seconds": el}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    samples = []
    workers = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_sample(2.0, workers)
    for _ in range(args.steps):
        samples.append(cpu_sample(args.ref_seconds, workers))
    val = float(np.median([s["value"] for s in samples]))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "grid-point-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.median([s["seconds"] for s in samples]) * 1e3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded config-5 initial condition)",
            "config": {"workload": "config5: 2D 1023^2 PA3 eps=0.01 T=2 N=512 J=256",
                       "sample": "per step: bounded run of LINEAR_B fine steps on one slice"},
            "cpu_baseline": {"value": val, "unit": "grid-point-steps/s", "cores": workers,
                             "kind": "port", "sample": samples[0]["sample"]},
            "e2e": {"value": val, "unit": "grid-point-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    from paper_2304_14074_b200.distributed import ShardedParareal

    g = SpatialGrid(CFG["dim"], CFG["nx"])
    part = P.TimePartition(CFG["T"], CFG["N"], CFG["J"])
    fine, coarse = P.propagator_pair(P.AlgorithmVariant.PA3, part, CFG["eps"])
    from paper_2304_14074_b200.configs import initial_condition
    u0 = initial_condition(5)
    eng = ShardedParareal(g, fine, coarse, CFG["N"], CFG["J"], rank=rank, world=world)
    eng.load(Field(g, u0))
    t0 = time.perf_counter()
    eng.coarse_init()
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0

    def step():
        eng.iterate(force_all=True)

    def step_pipelined():
        eng.iterate(force_all=True, defer=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # per-phase device timing of one step (fine sweep = dominant kernels)
    fine_ms = eng.time_fine_sweep()
    launches, names = count_launches(step)      # every rank steps (collectives inside)
    sampler = ClockSampler(local)
    cg0 = eng.eng.stats.coarse_cg_iterations
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step_pipelined()
    eng.flush()                                   # the increments' all-reduces are inside
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    coarse_cg = (eng.eng.stats.coarse_cg_iterations - cg0) / (args.steps * eng.local_slices)
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pts = CFG["N"] * CFG["J"] * g.interior_count      # whole job, all ranks
    value = pts / (ms * 1e-3)

    # e2e: host-resident iterates through the public engine API
    e2e = eng.e2e_step_rate(args.e2e_steps) if args.e2e_steps > 0 else None
    local_slices = eng.local_slices
    del eng
    torch.cuda.empty_cache()
    ttt = time_to_tolerance([int(c) for c in args.ttt.split(",") if c], rank, world) \
        if args.ttt else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks, src = measured_peaks()
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            traffic = json.load(f)["fine_step_bytes_per_grid_point_step"]
    except (OSError, KeyError, ValueError):
        traffic = None
    local_pts = local_slices * CFG["J"] * g.interior_count
    fine_bytes = 32.0 * local_pts          # algorithmic HBM bytes of the fine sweep
    achieved = fine_bytes / (fine_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "grid-point-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-5 initial condition, SURVEY.md 8(d))",
        "config": {"workload": "config5: 2D 1023^2 PA3 eps=0.01 T=2 N=512 J=256, every slice "
                               "active each step", "parallelism": f"time-slices x{world}",
                   "coarse_chain_hop": ("none (one rank)" if world == 1 else
                                        "device-initiated hop over cudaIpc (CHP_HOP=ipc)"
                                        if os.environ.get("CHP_HOP", "") == "ipc"
                                        else "torch.distributed send/recv (NCCL)"),
                   "l2": "working set 13 GB >> 126 MB L2 (no flush needed)"},
        "fine_phase": {"ms": fine_ms, "grid_point_steps_per_s": local_pts / (fine_ms * 1e-3)},
        "coarse_init_s": init_s,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "peak_source": src,
                     "kernel": "LINEAR_B fine propagator (linb::k2d_rowb + linb::k2d_colt), "
                               "32 B/grid-point-step", "traffic": traffic,
                     "traffic_unit": "DRAM bytes per grid-point-step (ncu, row+column pass)"},
        "coarse_cg_per_step": coarse_cg,
        "time_to_tolerance": ttt,
        "clocks": clocks, "gpu_launches": launches * args.steps if launches else launches,
        "launches_per_step": names,
        "e2e": e2e,
    }
    line["fp64"] = fp64_block()
    line["config4_newton_pcg"] = config4_block(line["roofline"]["peak"])
    if args.cpu_baseline:
        line["cpu_baseline"] = cpu_sample(args.ref_seconds)
        line["cpu_baselines"] = cpu_baselines()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()



# ---------------------------------------------------------------------------
# Time to tolerance, FP64 model, per-config CPU baselines
# ---------------------------------------------------------------------------

def time_to_tolerance(cfgs, rank, world) -> dict:
    """Full Parareal runs (coarse init + iterations to max|U^{k+1}-U^k| < 1e-10, every
    IC) of the given configs over the job's ranks (contiguous slice shards, pipelined
    run), timed between barriers; wall = max over ranks.  Seeded inputs of SURVEY.md
    8(d).  Fine work is the pt-steps actually computed (skip-stable slices)."""
    import torch
    import torch.distributed as dist

    from paper_2304_14074_b200 import parareal as P
    from paper_2304_14074_b200.configs import CONFIGS, initial_condition
    from paper_2304_14074_b200.distributed import ShardedParareal
    from paper_2304_14074_b200.grid import Field, SpatialGrid
    out = {}
    for cfg in cfgs:
        c = CONFIGS[cfg]
        g = SpatialGrid(c["dim"], c["nx"])
        B = c.get("batch", 1)
        part = P.TimePartition(c["T"], c["N"], c["J"])
        f, co = P.propagator_pair(P.AlgorithmVariant(c["variant"]), part, c["eps"])
        sh = ShardedParareal(g, f, co, c["N"], c["J"], rank=rank, world=world, batch=B)
        sh.load([Field(g, initial_condition(cfg, b)) for b in range(B)])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sh.run(pipelined=True)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = sh.eng.stats
        vals = torch.tensor([wall, float(st.fine_point_steps), float(sh.eng.newton.total_iterations),
                             float(sh.eng.newton.steps)], dtype=torch.float64, device="cuda")
        if world > 1:
            t = vals[:1].clone()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            rest = vals[1:].clone()
            dist.all_reduce(rest, op=dist.ReduceOp.SUM)
            vals = torch.cat([t, rest])
        wall, fps, ntot, nsteps = (float(x) for x in vals.cpu())
        ks = [int(k) if k is not None else None for k in sh.converged]
        out[f"config{cfg}"] = {
            "variant": c["variant"], "ics": B, "k": ks[0] if B == 1 else
            {"min": min(k for k in ks if k is not None) if any(k is not None for k in ks) else None,
             "max": max(k for k in ks if k is not None) if any(k is not None for k in ks) else None,
             "all_converged": all(k is not None for k in ks)},
            "seconds": wall, "fine_point_steps": fps,
            "newton_solves_per_step": (ntot / nsteps) if nsteps else None,
            "last_increment": float(sh.incs[-1][0]) if sh.incs else None,
            "ranks": world}
        del sh
        torch.cuda.empty_cache()
    return out


def fp64_block() -> dict:
    """Measured DFMA peak (chp_probe_dfma) and the 1D configs' fine propagators against
    the flop model of BASELINE.md 3 (LINEAR_B ~21 flop/pt-step, Newton ~30 + 62 n_N)."""
    import ctypes

    import torch

    from paper_2304_14074_b200 import _native as N
    from paper_2304_14074_b200 import schemes as S
    from paper_2304_14074_b200.configs import CONFIGS, initial_condition
    from paper_2304_14074_b200.grid import SpatialGrid
    ctx = N.Context.get(torch.cuda.current_device())
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    buf = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = sms * 8, 20000
    best = None
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.check(ctx.L.chp_probe_dfma(ctx.h, blocks, iters, N.ptr(buf), N.stream_ptr()),
                  "chp_probe_dfma")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    peak = 2.0 * 16 * iters * 256 * blocks / (best * 1e-3) / 1e12
    res = {"dfma_peak_tflops": peak, "probe": f"{blocks} x 256 threads x 16 DFMA chains x {iters}"}

    def rate(cfg, scheme, nsys, steps):
        c = CONFIGS[cfg]
        g = SpatialGrid(1, c["nx"])
        src = torch.tensor(np.stack([initial_condition(cfg, b % 64) for b in range(nsys)]),
                           device="cuda")
        out = torch.empty_like(src)
        dt = c["T"] / c["N"] / c["J"]
        spec = S.PropagatorSpec(scheme, dt, c["eps"])
        S.propagate_batch(g, spec, steps, src, out)
        info = S.new_sysinfo(nsys, "cuda")
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        S.propagate_batch(g, spec, steps, src, out, info=info)
        b.record()
        torch.cuda.synchronize()
        si = S.read_sysinfo(info)
        nn = float(si["newton_total"].sum()) / max(1.0, float(si["newton_steps"].sum()))
        return nsys * steps * g.interior_count / (a.elapsed_time(b) * 1e-3), nn
    r1, _ = rate(1, S.Scheme.LINEAR_B, 16, 256)          # one config-1 fine sweep
    r2, nn = rate(2, S.Scheme.NONLINEAR_EYRE, 4096, 16)  # config 2's 64 ICs x 64 slices
    f1, f2 = 21.0, 30.0 + 62.0 * nn
    res["config1_linear_b"] = {"pt_steps_per_s": r1, "flop_per_pt_step": f1,
                               "tflops": r1 * f1 / 1e12, "frac": r1 * f1 / 1e12 / peak,
                               "shape": "16 systems x 256 steps (one config-1 fine sweep)"}
    res["config2_newton"] = {"pt_steps_per_s": r2, "newton_solves_per_step": nn,
                             "flop_per_pt_step": f2, "tflops": r2 * f2 / 1e12,
                             "frac": r2 * f2 / 1e12 / peak,
                             "shape": "4096 systems x 16 steps (config 2's 64 ICs x 64 slices)"}
    return res


def config4_block(peak_gbs: float) -> dict:
    """2D Newton-PCG fine path at config 4's shape (511^2, eps=0.015, 128 slices; VERDICT r1
    item 3): fine grid-point-steps/s of one batched chp_propagate, the device Newton and
    CG counters, and the achieved bytes of SURVEY.md 8(d)'s model -- one LINEAR_B-like
    32 B pass pair for the step itself and one per operator application,
    32 (1 + n_N (1 + n_CG)) B per grid-point-step -- against the HBM peak."""
    import torch

    from paper_2304_14074_b200 import schemes as S
    from paper_2304_14074_b200.configs import CONFIGS, initial_condition
    from paper_2304_14074_b200.grid import SpatialGrid, to_device_layout
    c = CONFIGS[4]
    g = SpatialGrid(2, c["nx"])
    nsys, steps = c["N"], 4
    u0 = torch.tensor(initial_condition(4), device="cuda")
    src = torch.stack([to_device_layout(g, u0)] * nsys)
    # distinct states per slice: slice n starts from n coarse-sized LINEAR_B steps of u0 scaled
    # down to stay cheap -- every system then has its own Newton/CG history
    spec_b = S.PropagatorSpec(S.Scheme.LINEAR_B, c["T"] / c["N"] / c["J"], c["eps"])
    tmp = torch.empty_like(src[:1])
    for n in range(1, nsys):
        S.propagate_batch(g, spec_b, 2, src[n - 1:n], tmp)
        src[n].copy_(tmp[0])
    out = torch.empty_like(src)
    spec = S.PropagatorSpec(S.Scheme.NONLINEAR_EYRE, c["T"] / c["N"] / c["J"], c["eps"])
    S.propagate_batch(g, spec, steps, src, out)
    info = S.new_sysinfo(nsys, "cuda")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    S.propagate_batch(g, spec, steps, src, out, info=info)
    b.record()
    torch.cuda.synchronize()
    si = S.read_sysinfo(info)
    nst = max(1.0, float(si["newton_steps"].sum()))
    n_n = float(si["newton_total"].sum()) / nst
    n_cg = float(si["cg_total"].sum()) / max(1.0, float(si["newton_total"].sum()))
    rate = nsys * steps * g.interior_count / (a.elapsed_time(b) * 1e-3)
    bytes_pt = 32.0 * (1.0 + n_n * (1.0 + n_cg))
    return {"pt_steps_per_s": rate, "ms": a.elapsed_time(b), "newton_solves_per_step": n_n,
            "cg_iterations_per_solve": n_cg, "bytes_per_pt_step_model": bytes_pt,
            "achieved_GBps": rate * bytes_pt / 1e9, "frac_of_hbm": rate * bytes_pt / 1e9 / peak_gbs,
            "shape": f"{nsys} systems x {steps} Newton steps at 511^2 (config 4's slices, "
                     "states = u0 advanced 2 n LINEAR_B steps for slice n)"}


def cpu_baselines() -> dict:
    """The reference's arithmetic per config on this host's cores (oracle port: the same
    numpy / scipy LAPACK / SuperLU calls as the reference)."""
    from oracle import chp_oracle as O
    from paper_2304_14074_b200.configs import CONFIGS, initial_condition
    cores = os.cpu_count() or 1
    out = {"cores": cores, "kind": "port"}
    kn = O.Knobs(cube="numpy")
    c = CONFIGS[1]
    m = O.Mesh(1, c["nx"])
    u0 = initial_condition(1)
    t0 = time.perf_counter()
    O.serial_fine(m, u0, "pa3", c["T"], c["N"], c["J"], c["eps"], kn)
    t_ser = time.perf_counter() - t0
    par = {}
    for w in (1, cores):
        t0 = time.perf_counter()
        r = O.parareal(m, u0, "pa3", c["T"], c["N"], c["J"], c["eps"], kn, skip_stable=False,
                       workers=w)
        par[w] = (time.perf_counter() - t0, r.k)
    out["config1"] = {"serial_fine_s": t_ser, "parareal_workers1_s": par[1][0],
                      f"parareal_workers{cores}_s": par[cores][0], "k": par[1][1],
                      "sample": "full run (reference recomputes every slice each iteration)"}
    # config 2: Newton fine steps of one IC; serial fine = N*J steps, Parareal (k = N+1,
    # the reference recomputes all N slices per iteration) extrapolated from the step time
    c = CONFIGS[2]
    m = O.Mesh(1, c["nx"])
    dt = c["T"] / c["N"] / c["J"]
    t0 = time.perf_counter()
    O.advance(m, initial_condition(2), O.EYRE, dt, c["eps"], 512, kn)
    tf = (time.perf_counter() - t0) / 512
    t0 = time.perf_counter()
    O.advance(m, initial_condition(2), O.LINEAR_A, c["T"] / c["N"], c["eps"], 8, kn)
    tg = (time.perf_counter() - t0) / 8
    k = c["N"] + 1
    per_ic = c["N"] * tg + k * (c["N"] * c["J"] * tf + c["N"] * tg)
    out["config2"] = {"fine_step_ms": tf * 1e3, "coarse_step_ms": tg * 1e3,
                      "serial_fine_per_ic_s": c["N"] * c["J"] * tf,
                      "parareal_per_ic_s_extrapolated": per_ic,
                      "parareal_64ics_s_extrapolated": per_ic * c["batch"] / cores,
                      "sample": "512 Newton steps + 8 coarse steps of IC 0; T = N t_G + k (N J t_F "
                                "+ N t_G), k = N+1, 64 ICs over the host cores"}
    # config 3: LINEAR_B steps (cached SuperLU factor) + LINEAR_A SuperLU coarse steps
    c = CONFIGS[3]
    m = O.Mesh(2, c["nx"])
    dt = c["T"] / c["N"] / c["J"]
    u0 = initial_condition(3)
    O.advance(m, u0, O.LINEAR_B, dt, c["eps"], 1, kn)      # factor (cached)
    t0 = time.perf_counter()
    O.advance(m, u0, O.LINEAR_B, dt, c["eps"], 16, kn)
    tf = (time.perf_counter() - t0) / 16
    t0 = time.perf_counter()
    O.advance(m, u0, O.LINEAR_A, c["T"] / c["N"], c["eps"], 1, kn)
    tg = time.perf_counter() - t0
    k = 63
    out["config3"] = {"fine_step_ms": tf * 1e3, "coarse_step_s": tg,
                      "serial_fine_s_extrapolated": c["N"] * c["J"] * tf,
                      "parareal_s_extrapolated": c["N"] * tg + k * (c["N"] * c["J"] * tf +
                                                                   c["N"] * tg),
                      "sample": "16 LINEAR_B steps + 1 SuperLU LINEAR_A step at 255^2; k = 63 "
                                "(the GPU's and the oracle's)"}
    return out

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--ttt", default="1,2,3",
                    help="configs whose full time to tolerance is measured (e.g. 1,2,3,4,5; '' = none)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
