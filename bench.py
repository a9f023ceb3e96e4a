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
              "clocks_event_reasons.sw_power_cap")

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
            if len(parts) == 6:
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
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


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
    from oracle.chp_oracle import initial_condition   # seeded input generator only
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
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    pts = CFG["N"] * CFG["J"] * g.interior_count      # whole job, all ranks
    value = pts / (ms * 1e-3)

    # e2e: host-resident iterates through the public engine API
    e2e = eng.e2e_step_rate(args.e2e_steps) if args.e2e_steps > 0 else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks, src = measured_peaks()
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            traffic = json.load(f)["fine_step_bytes_per_grid_point_step"]
    except (OSError, KeyError, ValueError):
        traffic = None
    local_pts = eng.local_slices * CFG["J"] * g.interior_count
    fine_bytes = 32.0 * local_pts          # algorithmic HBM bytes of the fine sweep
    achieved = fine_bytes / (fine_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "grid-point-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-5 initial condition, SURVEY.md 8(d))",
        "config": {"workload": "config5: 2D 1023^2 PA3 eps=0.01 T=2 N=512 J=256, every slice "
                               "active each step", "parallelism": f"time-slices x{world}",
                   "l2": "working set 13 GB >> 126 MB L2 (no flush needed)"},
        "fine_phase": {"ms": fine_ms, "grid_point_steps_per_s": local_pts / (fine_ms * 1e-3)},
        "coarse_init_s": init_s,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "peak_source": src,
                     "kernel": "LINEAR_B fine propagator (linb::k2d_rowb + linb::k2d_colb), "
                               "32 B/grid-point-step", "traffic": traffic,
                     "traffic_unit": "DRAM bytes per grid-point-step (ncu, row+column pass)"},
        "clocks": clocks, "gpu_launches": launches * args.steps if launches else launches,
        "launches_per_step": names,
        "e2e": e2e,
    }
    if args.cpu_baseline:
        line["cpu_baseline"] = cpu_sample(args.ref_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
