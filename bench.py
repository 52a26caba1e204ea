#!/usr/bin/env python3
"""bench.py -- T_eff of the distributed Fig. 1 heat step on B200 (BASELINE.json).

A "step" is one pass of the whole hot path: one
@hide_communication (16,2,2) { step!(T2,T,Ci,...); update_halo!(T2) } time
step of the paper's 512^3-per-GPU Float64 workload
 followed by the pointer swap.

  python bench.py [--gpus N] [--steps K] [--warmup W]       # our CUDA path
  python bench.py --impl reference ...                        # the CPU oracle
  torchrun --nproc-per-node N ... bench.py --gpus N ...       # weak scaling, dims 2x1x1/2x2x1/2x2x2

value = T_eff summed over all GPUs = N * 24 B * 512^3 / t_step (B:5), t_step =
max over ranks of the CUDA-event time of K steps / K.  Inputs are 3 x 1 GiB
per GPU (> the 126 MB L2), so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "T_eff GB/s per GPU and weak-scaling efficiency at 1/2/4/8 B200"
BYTES_PER_CELL = 24          # T read + Ci read + T2 write, 8 B each (B:5)
DIMS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}   # B:9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64",
                    help="heat workload: f64 (the paper's Float64, default) or the binary32 variant (f4)")
    ap.add_argument("--workload", choices=["heat", "acoustic"], default="heat",
                    help="heat: the north-star Fig. 1 step (default); acoustic: the staggered second workload")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--bw", default="16,2,2")
    ap.add_argument("--path", choices=["nccl", "p2p"], default="p2p")
    ap.add_argument("--init", choices=["paper", "random"], default="paper")
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 generic region kernel (ablation)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-exposed", action="store_true")
    ap.add_argument("--fused", type=int, default=-1, help="1 fused stencil+P2P put kernel, 0 split, -1 auto")
    ap.add_argument("--fused-mode", type=int, default=0, help="ablation build only: binary32 schedule bits")
    ap.add_argument("--kc2", type=int, default=0, help="fused path: tail z-chunk planes (0 auto)")
    ap.add_argument("--ncomm", type=int, default=1, help="fused path: CTAs per receive/forward kernel")
    ap.add_argument("--dims", default="", help="override the process topology, e.g. 1,2,1")
    ap.add_argument("--schedule", type=int, default=0, help="0 concurrent, 1 boundary first (paper order)")
    ap.add_argument("--timeline", action="store_true", help="record the overlap timeline (extra events)")
    ap.add_argument("--xalign", type=int, default=64, help="x boundary-slab alignment in cells (1 = exact bw)")
    ap.add_argument("--periodic", default="0,0,0", help="periodic axes (1-GPU self-wrap experiments)")
    ap.add_argument("--per-step", action="store_true", help="time igg_heat_step calls instead of igg_heat_run")
    ap.add_argument("--skip-comm", action="store_true", help="timing experiment only: no exchange (INVALID results)")
    ap.add_argument("--samples", type=int, default=20, help="paper statistics: samples of nt=100 steps")
    ap.add_argument("--no-stats", action="store_true", help="skip the 20-sample statistics pass")
    ap.add_argument("--fused-f32", action="store_true", help="binary32 through the fused kernel (IGG_OPT_FUSED_F32)")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def dram_traffic_per_launch(name="traffic.json"):
    """ncu dram__bytes_read+write per launch of the dominant kernel, from the
    committed summary of this round's `ncu --set full` capture, else None."""
    p = os.path.join(ROOT, "profiles", name)
    try:
        d = json.load(open(p))
        return d
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,clocks.mem")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons, pw, mem = [], None, set(), [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                if len(f) >= 9:
                    pw.append(float(f[7]))
                    mem.append(float(f[8]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": statistics.median(pw) if pw else None,
                "mem_mhz_median": statistics.median(mem) if mem else None}


def cpu_oracle_baseline(n: int, target_s: float = 12.0, f32: bool = False):
    """The oracle as it stands (plain C, OpenMP) on this host: full n^3 paper
    workload, as many single steps as fit in ~target_s (at least 2)."""
    import numpy as np
    from oracle import heat3d as OH
    OH.build()
    OH.set_threads(len(os.sched_getaffinity(0)))   # all host cores (torchrun sets OMP_NUM_THREADS=1)
    if f32:   # the binary32 oracle: one-step runs (the copy T2 = T inside is part of the sample)
        T = np.full((n, n, n), 1.7, dtype=np.float32)
        Ci = np.full((n, n, n), 0.5, dtype=np.float32)
        d = 1.0 / (n - 1)
        dt = d * d / 0.5 / 6.1
        times = []
        t_end = time.perf_counter() + target_s
        while len(times) < 2 or (time.perf_counter() < t_end and len(times) < 30):
            t0 = time.perf_counter()
            T = OH.heat_run_f32(T, Ci, 1, (0, 0, 0), 1.0, dt, d, d, d)
            times.append(time.perf_counter() - t0)
        t = statistics.median(times)
        return {"value": 12 * n ** 3 / t / 1e9, "unit": "GB/s", "cores": OH.num_threads(), "kind": "oracle",
                "sample": f"{len(times)} binary32 oracle steps (full {n}^3 grid, each with its T2 = copy(T)), "
                          f"median {t:.3f} s/step, T_eff = 12 B x {n}^3 / t"}
    T = np.full((n, n, n), 1.7)
    T2 = T.copy()
    Ci = np.full((n, n, n), 0.5)
    d = 1.0 / (n - 1)
    dt = OH.stable_dt(d, d, d, 1.0, Ci)
    times = []
    t_end = time.perf_counter() + target_s
    while len(times) < 2 or (time.perf_counter() < t_end and len(times) < 50):
        t0 = time.perf_counter()
        OH.heat_step(T, Ci, T2, (0, 0, 0), 1.0, dt, d, d, d, OH.LITERAL)
        times.append(time.perf_counter() - t0)
        T, T2 = T2, T
    t = statistics.median(times)
    return {"value": BYTES_PER_CELL * n ** 3 / t / 1e9, "unit": "GB/s", "cores": OH.num_threads(),
            "kind": "oracle",
            "sample": f"{len(times)} oracle steps (paper-literal, full {n}^3 grid, T=1.7 Ci=0.5), median "
                      f"{t:.3f} s/step, T_eff = 24 B x {n}^3 / t"}


def run_reference(a):
    """--impl reference: the CPU oracle timed as it stands on the host cores.
    Each step = one oracle step (paper-literal C, OpenMP over z) of the SAME workload as our arm's
    line: the full n^3 local grid of the paper setup (T = 1.7, Ci = 0.5)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from oracle import heat3d as OH
    OH.build()
    OH.set_threads(len(os.sched_getaffinity(0)))   # all host cores (torchrun sets OMP_NUM_THREADS=1)
    n = a.n
    T = np.full((n, n, n), 1.7)
    T2 = T.copy()
    Ci = np.full((n, n, n), 0.5)
    d = 1.0 / (n - 1)
    dt = OH.stable_dt(d, d, d, 1.0, Ci)
    for _ in range(a.warmup):
        OH.heat_step(T, Ci, T2, (0, 0, 0), 1.0, dt, d, d, d, OH.LITERAL)
        T, T2 = T2, T
    t0 = time.perf_counter()
    for _ in range(a.steps):
        OH.heat_step(T, Ci, T2, (0, 0, 0), 1.0, dt, d, d, d, OH.LITERAL)
        T, T2 = T2, T
    el = time.perf_counter() - t0
    cells = n ** 3
    val = BYTES_PER_CELL * cells * a.steps / el / 1e9
    sample = f"{a.steps} oracle steps of the full {n}^3 grid (paper-literal C, OpenMP), after {a.warmup} warm-up"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": el / a.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"3-D heat diffusion Float64, local {n}^3, CPU oracle on the host cores",
                   "n_local": n, "sample_cells": cells},
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": OH.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def bpc_(f32: bool) -> int:
    return BYTES_PER_CELL // 2 if f32 else BYTES_PER_CELL


def median_ci95(xs):
    """Median and a distribution-free 95 % confidence interval of the median (order statistics of the
    binomial(n, 1/2): for n = 20 the 6th and 15th smallest, coverage 95.9 %) -- the paper's statistics
    of 20 samples (Fig. 2 caption)."""
    import math
    v = sorted(xs)
    n = len(v)
    if n < 6:
        return statistics.median(v), [v[0], v[-1]]
    # largest k with P(Binom(n, 1/2) < k) <= 2.5 %: [v[k-1], v[n-k]]
    k, acc = 0, 0.0
    while True:
        p = math.comb(n, k) / 2 ** n
        if acc + p > 0.025:
            break
        acc += p
        k += 1
    k = max(k, 1)
    return statistics.median(v), [v[k - 1], v[n - k]]


def main():
    a = parse()
    if a.workload == "acoustic":
        return run_acoustic(a)
    if a.impl == "reference":
        return run_reference(a)

    import torch
    import torch.distributed as dist
    import paper_2211_15716_b200 as P
    from paper_2211_15716_b200 import heat3d as app

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else (DIMS.get(world) or P.dims_create(world))
    bw = tuple(int(x) for x in a.bw.split(","))
    n = a.n
    periods = tuple(int(x) for x in a.periodic.split(","))
    g = P.init_global_grid(n, n, n, dims=dims, periods=periods, path=a.path, device=local)
    if a.kernel:
        g.set_option(P.OPT_STENCIL_KERNEL, a.kernel)
    g.set_option(P.OPT_X_ALIGN, a.xalign)
    if a.fused_f32:
        g.set_option(P.OPT_FUSED_F32, 1)
    g.set_option(P.OPT_SCHEDULE, a.schedule)
    g.set_option(P.OPT_FUSED, a.fused)
    if a.fused_mode:
        g.set_option(8, a.fused_mode)
    g.set_option(9, a.kc2)
    g.set_option(10, a.ncomm)
    if a.skip_comm:
        g.set_option(P.OPT_SKIP_COMM, 1)
    T, T2, Ci = app.alloc_fields(g)
    (app.init_paper if a.init == "paper" else app.init_random)(g, T, T2, Ci)
    d = app.spacing(g)
    dt = app.stable_dt(g, Ci, *d)
    stream = torch.cuda.current_stream()

    f32 = a.dtype == "f32"
    if f32:   # the binary32 variant (igg_heat_step_f32): same fields rounded to float once
        T, T2, Ci = (list(x) for x in app.alloc_fields(g, dtype=torch.float32))
        (app.init_paper if a.init == "paper" else app.init_random)(g, T, T2, Ci)

    def steps(k):   # Fig. 1's time loop through the public API (igg_heat_run; --per-step: igg_heat_step x k)
        nonlocal T, T2
        T, T2 = app.run(g, T, T2, Ci, k, dt, d, app.LAM, bw=bw, per_step=a.per_step)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    steps(max(a.warmup, 3))
    barrier()

    # ---------------- timed region: K steps, CUDA events on the launching stream
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.4)
    l0 = g.kernel_launches()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps(a.steps)
    e1.record(stream)
    barrier()
    launches = g.kernel_launches() - l0
    ms = e0.elapsed_time(e1) / a.steps
    per_rank_ms = [ms]
    if world > 1:
        allms = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(world)]
        dist.all_gather(allms, torch.tensor([ms], dtype=torch.float64, device="cuda"))
        per_rank_ms = [float(t.item()) for t in allms]
    ms = max_over_ranks(ms)
    clk = clocks.stop() if clocks else None
    g.check()

    def sampled(nsamples, nt):
        """The paper's statistics: nsamples samples of nt steps, each
        bracketed by barrier + synchronize, CUDA events on the launching stream, max over ranks."""
        xs = []
        for _ in range(nsamples):
            barrier()
            e0.record(stream)
            steps(nt)
            e1.record(stream)
            barrier()
            xs.append(max_over_ranks(e0.elapsed_time(e1) / nt))
        med, ci = median_ci95(xs)
        return {"samples": nsamples, "nt": nt, "median_ms": med, "ci95_ms": ci, "min_ms": min(xs),
                "max_ms": max(xs)}

    stats = None
    if not a.no_stats:
        sclk = ClockSampler(local) if rank == 0 else None
        if sclk:
            sclk.start()
            time.sleep(0.4)
        stats = sampled(a.samples, 100)
        if sclk:
            stats["clocks"] = sclk.stop()
        stats["t_eff_per_gpu_gbs_median"] = bpc_(f32) * n ** 3 / (stats["median_ms"] * 1e-3) / 1e9
        if a.init == "paper":   # B:8 (ii): the same timing on non-trivial (random) data
            (app.init_random)(g, T, T2, Ci)
            rclk = ClockSampler(local) if rank == 0 else None
            if rclk:
                rclk.start()
                time.sleep(0.4)
            stats["random_init"] = sampled(a.samples, 100)
            if rclk:
                stats["random_init"]["clocks"] = rclk.stop()
            app.init_paper(g, T, T2, Ci)
        g.check()
    # roofline pass (not timed above): CUDA events around the main stencil launches on their stream
    g.set_option(P.OPT_PROFILE, 2 if a.timeline else 1)
    g.profile_stencil()
    prof_steps = min(a.steps, 50)
    steps(prof_steps)
    barrier()
    k_ms, k_n, k_cells = g.profile_stencil()
    timeline = g.profile_timeline() if a.timeline else None
    g.set_option(P.OPT_PROFILE, 0)
    g.check()

    bpc = bpc_(f32)   # binary32: 3 x 4 B per cell
    per_gpu = bpc * n ** 3 / (ms * 1e-3) / 1e9
    value = per_gpu * world

    # ---------------- in-run streaming reference: torch fp64 a+b->c over 1 GiB arrays (2 reads + 1 write)
    stream_ref = None
    if rank == 0:
        x = torch.empty(n ** 3, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        zz = torch.empty_like(x)
        x.fill_(1.0)
        y.fill_(2.0)
        for _ in range(3):
            torch.add(x, y, out=zz)
        e0.record(stream)
        for _ in range(20):
            torch.add(x, y, out=zz)
        e1.record(stream)
        torch.cuda.synchronize()
        stream_ref = 3 * 8 * n ** 3 * 20 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        del x, y, zz
        torch.cuda.empty_cache()

    # ---------------- exposed halo time: same schedule with the exchange skipped (timing only)
    exposed = None
    if (world > 1 or any(periods)) and not a.no_exposed and not a.skip_comm:
        g.set_option(P.OPT_SKIP_COMM, 1)
        steps(3)
        barrier()
        e0.record(stream)
        steps(a.steps)
        e1.record(stream)
        barrier()
        ms_nc = max_over_ranks(e0.elapsed_time(e1) / a.steps)
        g.set_option(P.OPT_SKIP_COMM, 0)
        try:
            g.check()   # a flag timeout raises; the expected "steps ran with SKIP_COMM" state is cleared
        except P.IggError as ex:
            if ex.status != 2:
                raise
        exposed = {"ms_per_step": ms - ms_nc, "ms_no_comm": ms_nc}
        (app.init_paper if a.init == "paper" else app.init_random)(g, T, T2, Ci)   # results were invalid

    # ---------------- roofline of the dominant kernel (the full-region / inner-box stencil)
    fused_run = a.path == "p2p" and a.fused != 0 and (world > 1 or any(periods)) and not a.kernel
    kernel_name = ("heat_fused_kernel<float> (whole region: stencil + peer stores of the faces)" if f32 and fused_run
                   else "heat_f32_async_kernel (full region)" if f32 else
                   "heat_fused_kernel (whole region: stencil + peer stores of the faces)" if fused_run else
                   "heat_box_list_kernel (full region)" if world == 1 else
                   "heat_box_list_kernel (inner box)")
    peak, peak_src = measured_peak()
    k_avg_ms = k_ms / max(k_n, 1)
    k_bytes = bpc * k_cells / max(k_n, 1)
    achieved = k_bytes / (k_avg_ms * 1e-3) / 1e9 if k_n else None
    tr = dram_traffic_per_launch("traffic_f32.json" if f32 else "traffic_fused.json" if fused_run else "traffic.json")
    if f32 and fused_run:
        tr = None   # (no committed capture of the binary32 fused kernel)
    traffic = None
    if tr and tr.get("n") == n and (tr.get("dims") == list(dims) or fused_run):
        traffic = tr.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "kernel": kernel_name,
                "algorithmic_bytes_per_launch": k_bytes, "avg_launch_ms": k_avg_ms, "launches": k_n,
                "peak_source": peak_src, "share_of_step": k_avg_ms * (k_n / prof_steps) / ms if k_n else None,
                "measured_in": f"a separate pass of {prof_steps} steps with events around the kernel"}

    # ---------------- end to end through the C ABI from pinned host buffers
    e2e = None
    if not a.no_e2e and not f32:   # (igg_heat_run_host is the binary64 entry point)
        nt = 100
        cells = n ** 3
        Th = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
        Ch = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
        Th.copy_(T[0].cpu() if a.init == "random" else torch.full((1,), 1.7, dtype=torch.float64).expand(n, n, n))
        Ch.copy_(Ci[0].cpu())
        g.release_arrays()   # collective: no peer keeps a mapping of the arrays freed next
        del T, T2   # make room for the library's e2e scratch
        torch.cuda.empty_cache()
        T0h = Th.clone()
        reps = 2
        g.heat_run_host(Th, Ch, app.LAM, dt, *d, 2, bw=bw)     # warm the pool
        barrier()
        tt = []
        for _ in range(reps):
            Th.copy_(T0h)
            barrier()
            e0.record(stream)
            g.heat_run_host(Th, Ch, app.LAM, dt, *d, nt, bw=bw)
            e1.record(stream)
            barrier()
            tt.append(max_over_ranks(e0.elapsed_time(e1)))
        t_call = statistics.median(tt)
        g.check()
        h2d = 2 * cells * 8
        d2h = cells * 8
        e2e = {"value": world * BYTES_PER_CELL * cells * nt / (t_call * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": h2d / nt, "d2h_bytes_per_step": d2h / nt,
               "call": "igg_heat_run_host: H2D T,Ci from pinned host + T2 outer layers = T + nt=100 heat steps + D2H T",
               "nt_per_call": nt, "h2d_bytes_per_call": h2d, "d2h_bytes_per_call": d2h,
               "ms_per_call": t_call}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_oracle_baseline(n, f32=f32)

    g.finalize()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
            "config": {"workload": f"3-D heat diffusion {'Float32 variant' if f32 else 'Float64'}, local {n}^3 per GPU, dims "
                                   f"{dims[0]}x{dims[1]}x{dims[2]}, hide_communication {bw} (paper Fig. 1)" +
                                   ("" if (world > 1 or any(periods)) else
                                    "; one GPU: no axis exchanges, so the step is one full-region stencil launch "
                                    "(no boundary slabs to schedule)"),
                       "value_is": "aggregate over all GPUs (N x per-GPU T_eff)",
                       "n_local": n, "dims": list(dims), "bw": list(bw), "path": a.path, "init": a.init,
                       "x_align": a.xalign, "periods": list(periods), "schedule": a.schedule, "fused": a.fused,
                       "skip_comm_INVALID_RESULTS": bool(a.skip_comm),
                       "t_eff_per_gpu_gbs": per_gpu, "cells_per_s": world * n ** 3 / (ms * 1e-3),
                       "l2": "inputs 3 x 1 GiB per GPU > 126 MB L2; no flush needed",
                       "frac_of_8TBs": per_gpu / 8000.0, "frac_of_measured_peak": per_gpu / peak,
                       "stream_2r1w_gbs": stream_ref,
                       "frac_of_stream_2r1w": per_gpu / stream_ref if stream_ref else None,
                       "stencil_variant": a.kernel},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk, "exposed_halo": exposed, "timeline_ms": timeline, "per_rank_ms": per_rank_ms,
            "stats": stats,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ second workload
AC_METRIC = ("T_eff GB/s of the staggered acoustic step, aggregate over GPUs (P, Vx, Vy, Vz read+written once: "
             "64 B/cell)")
AC_BYTES_PER_CELL = 64      # effective: 4 fields x (read + write) x 8 B
AC_V_BYTES_PER_CELL = 56    # compute_V kernel: P, Vx, Vy, Vz read; Vx, Vy, Vz written


def acoustic_cpu_baseline(n: int, steps: int = 0, target_s: float = 12.0):
    """The acoustic oracle as it stands (numpy, one host thread for its elementwise ops) on a bounded
    sample: a full 512 x 512 extent with 34 z-planes per step, as many steps as fit in ~target_s."""
    import numpy as np
    import synthetic_inputs as SI
    from oracle import acoustic3d as OA
    nz = min(n, 34)
    N = (n, n, nz)
    F = SI.global_acoustic_fields(OA.field_shapes(N, (0, 0, 0)))
    d = 1.0 / n
    dt = d / 2.0 / 3 ** 0.5
    co = OA.coefficients(dt, 1.0, 1.0, d, d, d)
    times = []
    t_end = time.perf_counter() + target_s
    while len(times) < max(2, steps) and (steps or time.perf_counter() < t_end or len(times) < 2):
        t0 = time.perf_counter()
        OA.step(*F, (0, 0, 0), co)
        times.append(time.perf_counter() - t0)
        if not steps and len(times) >= 50:
            break
    t = statistics.median(times)
    cells = n * n * nz
    return {"value": AC_BYTES_PER_CELL * cells / t / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{len(times)} acoustic oracle steps (numpy) on a {n}x{n}x{nz} slab of the {n}^3 workload, "
                      f"median {t:.3f} s/step, T_eff = 64 B x cells / t"}, times


def run_acoustic(a):
    """--workload acoustic: one step of igg_acoustic_run on 512^3 cells per GPU, random fields: one fused
    compute_V + compute_P sweep on double-buffered fields when no axis exchanges (1 GPU), else compute_V
    under @hide_communication with update_halo!(Vx, Vy, Vz), then compute_P (igg_acoustic_step)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = a.n
    bw = tuple(int(x) for x in a.bw.split(",")) if a.bw != "16,2,2" else (16, 4, 4)
    if a.impl == "reference":
        if rank != 0:
            return
        cpu, times = acoustic_cpu_baseline(n, steps=a.warmup + a.steps)
        t = sum(times[a.warmup:])
        val = cpu["value"]
        print(json.dumps({
            "impl": "reference", "metric": AC_METRIC, "value": val, "unit": "GB/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": t / a.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"acoustic staggered step Float64, {n}^3 local, CPU oracle sample"},
            "cpu_baseline": cpu, "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist
    import paper_2211_15716_b200 as P
    from paper_2211_15716_b200 import acoustic3d as ac

    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dims = tuple(int(x) for x in a.dims.split(",")) if a.dims else (DIMS.get(world) or P.dims_create(world))
    g = P.init_global_grid(n, n, n, dims=dims, path=a.path, device=local)
    F = ac.alloc_fields(g)
    F2 = ac.alloc_fields(g)   # double-buffered: igg_acoustic_run's fused sweep when no axis exchanges
    ac.init_random(g, F)
    d = ac.spacing(g)
    dt = ac.stable_dt(d)
    stream = torch.cuda.current_stream()
    fused = world == 1   # (no exchanged axis: one fused V+P sweep per step, 64 B/cell)

    def steps(k):
        nonlocal F, F2
        F, F2 = g.acoustic_run(F, F2, k, dt, ac.RHO, ac.K, *d, bw=bw)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    steps(max(a.warmup, 3))
    barrier()
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.4)
    l0 = g.kernel_launches()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps(a.steps)
    e1.record(stream)
    barrier()
    launches = g.kernel_launches() - l0
    ms = max_over_ranks(e0.elapsed_time(e1) / a.steps)
    clk = clocks.stop() if clocks else None
    g.set_option(P.OPT_PROFILE, 1)   # roofline pass, not timed above
    g.profile_stencil()
    prof_steps = min(a.steps, 20)
    steps(prof_steps)
    barrier()
    k_ms, k_n, k_cells = g.profile_stencil()
    g.set_option(P.OPT_PROFILE, 0)
    g.check()
    per_gpu = AC_BYTES_PER_CELL * n ** 3 / (ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    k_avg_ms = k_ms / max(k_n, 1)
    k_bytes = (AC_BYTES_PER_CELL if fused else AC_V_BYTES_PER_CELL) * k_cells / max(k_n, 1)
    achieved = k_bytes / (k_avg_ms * 1e-3) / 1e9 if k_n else None
    tr = dram_traffic_per_launch("traffic_acoustic.json")
    traffic = None
    if tr and tr.get("n") == n and tr.get("dims") == list(dims):
        traffic = tr.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "kernel": ("acoustic_fused_kernel (compute_V + compute_P, one sweep, double-buffered)" if fused
                           else "acoustic_v_kernel (inner box)"),
                "algorithmic_bytes_per_launch": k_bytes, "avg_launch_ms": k_avg_ms, "launches": k_n,
                "peak_source": peak_src, "share_of_step": k_avg_ms * (k_n / prof_steps) / ms if k_n else None}

    e2e = None
    if not a.no_e2e:   # pinned host fields -> device, nt steps through the public API, fields -> host
        nt = 20
        host = [torch.empty(f[0].shape, dtype=torch.float64).pin_memory() for f in F]
        for h, f in zip(host, F):
            h.copy_(f[0])
        barrier()
        e0.record(stream)
        for h, f in zip(host, F):
            f[0].copy_(h, non_blocking=True)
        steps(nt)
        for h, f in zip(host, F):   # (F: the state after the nt steps)
            h.copy_(f[0], non_blocking=True)
        e1.record(stream)
        barrier()
        t_call = max_over_ranks(e0.elapsed_time(e1))
        nbytes = sum(h.numel() * 8 for h in host)
        e2e = {"value": world * AC_BYTES_PER_CELL * n ** 3 * nt / (t_call * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": nbytes / nt, "d2h_bytes_per_step": nbytes / nt,
               "call": f"H2D P,Vx,Vy,Vz from pinned host + {nt} igg_acoustic_step + D2H all four", "nt_per_call": nt,
               "ms_per_call": t_call}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu, _ = acoustic_cpu_baseline(n)
    g.finalize()
    if rank == 0:
        print(json.dumps({
            "metric": AC_METRIC, "value": per_gpu * world, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"staggered acoustic step Float64 (P {n}^3, Vx {n + 1}x{n}x{n}, Vy, Vz) per GPU, "
                                   f"dims {dims[0]}x{dims[1]}x{dims[2]}, hide_communication {bw}",
                       "n_local": n, "dims": list(dims), "bw": list(bw), "path": a.path,
                       "t_eff_per_gpu_gbs": per_gpu, "cells_per_s": world * n ** 3 / (ms * 1e-3),
                       "l2": "inputs 4 x 1 GiB per GPU > 126 MB L2; no flush needed",
                       "frac_of_measured_peak": per_gpu / peak},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
