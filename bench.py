"""bench.py -- grid-point updates/s per RK stage of the B200 HJ level-set step (BASELINE.json metric).

A "step" is one complete odp_hj_solve of the workload: every row of SURVEY.md §8(a) (derivatives,
range reduction, alpha/CFL finalize, Hamiltonian + dissipation + RK stage + BRT min, tau loop,
snapshot) over the whole grid.  value = points x RK stages / device time.

N=1 workload: c4 (6D double integrator, 30^6 = 7.29e8 points, ENO2 + TVD-RK2, BRT over [0,1]) --
the largest config that fits one GPU and the one BASELINE.json's scaling target names.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

--config t1 measures SURVEY.md §8(f3) instead: time-to-reach (Algorithm 3) on the Dubins car at 256^3,
a step = one odp_ttr_solve to convergence, value = node updates (nodes x iterations) / device time.
--config v2 (v0, v1) measures SURVEY.md §8(f4): value iteration (Algorithm 1) on the Dubins-car MDP,
a step = one odp_vi_solve to convergence; the line also carries Table 3's grid shapes in seconds.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point updates/s per RK stage"
UNIT = "point-stages/s"

# algorithmic HBM bytes per point of one launch (SURVEY.md §8(a) table "Bytes per point per stage")
PASS1_BYTES = 4                                     # read W
PASS2_BYTES = {("low", "brt"): 12, ("low", "brs"): 8,                      # Euler: R W, (R V0), W V'
               ("medium", "brt", 1): 8, ("medium", "brs", 1): 8,            # RK stage 1: R Vn, W V1
               ("medium", "brt", 2): 16, ("medium", "brs", 2): 12}          # RK stage 2: R V1, R Vn, (R V0), W Vn
STAGE_BYTES = {("low", "brt"): 16, ("low", "brs"): 12, ("medium", "brt"): 16, ("medium", "brs"): 14}
N_SMSP = 148 * 4                                    # issue slots per cycle of the chip (warp instructions)


def ncu_kernel_profile(name):
    """Per-launch figures of one `ncu --set full` capture of the workload's kernels (committed under
    profiles/, written by tools/make_profiles.py): DRAM bytes, warp instructions, issue-active."""
    prof = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    if not os.path.exists(prof):
        return {}
    try:
        return json.load(open(prof)).get(name, {})
    except Exception:
        return {}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------------------------------------------
# CPU baseline / reference arm: the float64 oracle as it stands, on a bounded sample of the workload
# --------------------------------------------------------------------------------------------------
def oracle_sample(w, target_s: float = 15.0):
    """Time the oracle (as it stands) on a centred sub-box of the workload with the same spacing,
    dynamics and target, for exactly one time step; the box is sized so the run takes about
    target_s seconds.  Returns (point-stages/s, sample description, cores, seconds, point-stages)."""
    import oracle
    from inputs import make_v0
    cores = oracle.max_threads()

    def box(side):
        N = tuple(min(side, n) for n in w.N)
        lo, hi = [], []
        for n_full, n, l, h, p in zip(w.N, N, w.lo, w.hi, w.periodic):
            dx = (h - l) / (n_full if p else n_full - 1)
            c0 = (n_full - n) // 2
            lo.append(l + c0 * dx)
            hi.append(l + (c0 + n - (0 if p else 1)) * dx)
        return w.__class__(**{**w.__dict__, "N": N, "lo": tuple(lo), "hi": tuple(hi)})

    def timed(sub):
        V0 = make_v0(sub)
        L, mn, mx, amax, _, _ = oracle.stage(V0, sub.lo, sub.hi, sub.periodic_mask, sub.dynamics, sub.params,
                                             sub.accuracy)
        dx = [(h - l) / (n if p else n - 1) for n, l, h, p in zip(sub.N, sub.lo, sub.hi, sub.periodic)]
        dt = oracle.cfl_dt(amax, dx, sub.cfl)
        one = sub.__class__(**{**sub.__dict__, "tau": (0.0, dt)})       # exactly one CFL step
        t0 = time.perf_counter()
        r = oracle.solve_workload(one, V0=V0, raise_on_error=False)
        return time.perf_counter() - t0, int(np.prod(sub.N)) * r.stages, r.stages

    side = 10
    el, work, stages = timed(box(side))
    n = len(w.N)
    side = int(side * (target_s / max(el, 1e-3)) ** (1.0 / n))
    side = max(6, min(side, max(w.N)))
    sub = box(side)
    el, work, stages = timed(sub)
    full_s = w.points * (stages * 1.0) / (work / el)
    sample = (f"oracle float64 on a {'x'.join(map(str, sub.N))} centred sub-box of {w.name} (same spacing, "
              f"dynamics, target), one time step = {stages} RK stages, {el:.1f} s; the rate is per point-stage "
              f"(one time step of the full {w.name} grid would take ~{full_s:.0f} s at it)")
    return work / el, sample, cores, el, work


# --------------------------------------------------------------------------------------------------
# time-to-reach (Algorithm 3) -- a step is one odp_ttr_solve to convergence
# --------------------------------------------------------------------------------------------------
TTR_METRIC = "TTR node updates/s (Lax-Friedrichs iteration to convergence)"
TTR_UNIT = "node-iterations/s"
TTR_BYTES = 8      # algorithmic HBM bytes per node per iteration of the interior kernel: read phi, write phi


def ttr_oracle_sample(w, target_s: float = 15.0):
    """The oracle's Gauss-Seidel sweeps (as it stands) on the workload's domain at a coarser node count
    sized to ~target_s seconds.  Returns (node-iterations/s, description, cores, seconds, node-iterations)."""
    import oracle
    from inputs import coarsened, make_v0
    cores = oracle.max_threads()

    def timed(side):
        sub = coarsened(w, (side,) * len(w.N))
        V0 = make_v0(sub)
        t0 = time.perf_counter()
        _, sweeps, _ = oracle.ttr_solve(sub.N, sub.lo, sub.hi, sub.periodic_mask, sub.dynamics, sub.params, V0,
                                        eps=1e-6)
        return time.perf_counter() - t0, sub, sweeps

    el, sub, sweeps = timed(16)
    side = int(16 * (target_s / max(el, 1e-3)) ** (1.0 / (len(w.N) + 1)))     # sweeps grow ~ linearly in side
    side = max(8, min(side, max(w.N)))
    el, sub, sweeps = timed(side)
    work = sub.points * sweeps
    sample = (f"oracle float64 Gauss-Seidel sweeps (Alg. 3 as printed, 8 orderings) on {w.name}'s domain at "
              f"{'x'.join(map(str, sub.N))} nodes, to convergence (eps 1e-6): {sweeps} sweeps, {el:.1f} s, 1 thread")
    return work / el, sample, 1, el, work


def run_ttr(args):
    import torch
    from paper_2204_05520_b200 import capi
    from inputs import TTR_CONFIGS, make_v0
    rank, world, local = dist_env()
    w = TTR_CONFIGS[args.config]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # replicas only: every rank solves its own copy; value = all ranks' node updates
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", init_method="env://", device_id=dev)
    g = capi.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    V0h = make_v0(w)
    V0 = torch.from_numpy(V0h).to(dev)
    phi = torch.empty(w.N, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as tdist
            tdist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as tdist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        capi.ttr_solve(g, w.dynamics, w.params, V0, phi=phi, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters, launches = 0, 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            _, info = capi.ttr_solve(g, w.dynamics, w.params, V0, phi=phi, stream=stream)
            iters += info["iters"]
            launches += g.launch_count()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        _, tinfo = capi.ttr_solve(g, w.dynamics, w.params, V0, phi=phi, stream=stream, use_graph=False)
    clocks = clk.summary()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    value = w.points * iters * world / (total_ms / 1e3)
    # end to end: pinned host V0 -> device -> solve -> host phi, through odp_ttr_solve_host
    V0p = torch.from_numpy(V0h).pin_memory()
    outp = torch.empty(w.N, dtype=torch.float32).pin_memory()
    capi.ttr_solve_host(g, w.dynamics, w.params, V0p.numpy(), phi=outp.numpy())
    barrier()
    t0 = time.perf_counter()
    e2e_it = 0
    for _ in range(max(1, min(args.steps, 3))):
        _, hi = capi.ttr_solve_host(g, w.dynamics, w.params, V0p.numpy(), phi=outp.numpy())
        e2e_it += hi["iters"]
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    peak, peak_kind = measured_peaks()
    it1 = tinfo["iters"]
    interior_ms = tinfo["interior_ms"] / it1
    faces_ms = tinfo["faces_ms"] / it1
    achieved = TTR_BYTES * w.points / (interior_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{w.name}:interior")
        except Exception:
            traffic = None
    line = {
        "metric": TTR_METRIC, "value": value, "unit": TTR_UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name, "grid": list(w.N), "points": w.points, "dynamics": w.dynamics,
                   "params": list(w.params), "eps": 1e-6, "iterations_per_step": iters / args.steps,
                   "order": "Jacobi (reading A35)",
                   "l2": ("inputs larger than L2: 2 x %.0f MB iterates (%.0f MB) per iteration vs 126 MB L2" %
                          (w.points * 4 / 1e6, w.points * 8 / 1e6)) if w.points * 8 > 126e6 else "iterates fit L2",
                   "parallelism": "single GPU" if world == 1 else f"{world} independent replicas"},
        "roofline": {"bound": "hbm", "kernel": ("k_ttr_tile" if len(w.N) >= 3 else "k_ttr_march") + " (Alg. 3 l.5-12, interior update)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind, "bytes_per_point": TTR_BYTES,
                     "avg_launch_ms": interior_ms, "faces_ms_per_iteration": faces_ms},
        "clocks": clocks,
        "e2e": {"value": w.points * e2e_it * world / e2e_s, "unit": TTR_UNIT, "h2d_bytes_per_step": w.points * 4,
                "d2h_bytes_per_step": w.points * 4},
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, sample, cores, el, work = ttr_oracle_sample(w, target_s=args.ref_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": TTR_UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                                "ordering": ("different iteration orders: the oracle runs Alg. 3 as printed (in-place "
                                             "Gauss-Seidel, 8 alternating orderings, §4.3), the GPU Jacobi (reading "
                                             "A35, %d iterations at %s); Gauss-Seidel reaches the same fixed point in "
                                             "fewer sweeps, so the node-iterations/s ratio compares iteration "
                                             "throughput and overstates the time-to-solution ratio" %
                                             (iters // max(1, args.steps), "x".join(map(str, w.N))))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
        tdist.destroy_process_group()


def run_ttr_reference(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            return
    from inputs import TTR_CONFIGS
    w = TTR_CONFIGS[args.config]
    times, work = [], []
    for i in range(args.warmup + args.steps):
        rate, sample, cores, el, wk = ttr_oracle_sample(w, target_s=args.ref_seconds)
        if i >= args.warmup:
            times.append(el)
            work.append(wk)
    value = sum(work) / sum(times)
    line = {"impl": "reference", "metric": TTR_METRIC, "value": value, "unit": TTR_UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "grid": list(w.N)},
            "cpu_baseline": {"value": value, "unit": TTR_UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": TTR_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------------------------------------------
# value iteration (Algorithm 1) -- a step is one odp_vi_solve to convergence
# --------------------------------------------------------------------------------------------------
VI_METRIC = "value-iteration node updates/s (Bellman iterations to convergence)"
VI_UNIT = "node-iterations/s"
VI_BYTES = 12      # algorithmic HBM bytes per node per iteration: read R, read V_t (gathers hit L1/L2), write V_t+1


def vi_oracle_sample(w, target_s: float = 15.0):
    """The oracle's Jacobi value iteration (as it stands, 1 thread) on the workload's domain at a
    node count sized to ~target_s seconds, to the same threshold."""
    import oracle
    from inputs import make_reward
    from dataclasses import replace

    def timed(scale):
        N = tuple(max(4, int(round(n * scale))) for n in w.N)
        sub = replace(w, N=N)
        R = make_reward(sub)
        t0 = time.perf_counter()
        _, it, _ = oracle.vi_solve(sub.N, sub.lo, sub.hi, sub.periodic_mask, sub.model, sub.params, R, threshold=1e-6)
        return time.perf_counter() - t0, sub, it

    el, sub, it = timed(min(1.0, 20.0 / max(w.N)))
    scale = min(1.0, 20.0 / max(w.N)) * (target_s / max(el, 1e-3)) ** (1.0 / 3.0)
    el, sub, it = timed(min(1.0, scale))
    work = sub.points * it
    sample = (f"oracle float64 Jacobi value iteration (Alg. 1, 1 thread) on {w.name}'s MDP at "
              f"{'x'.join(map(str, sub.N))} nodes to threshold 1e-6: {it} iterations, {el:.1f} s")
    return work / el, sample, 1, el, work


def run_vi(args):
    import torch
    from paper_2204_05520_b200 import capi
    from inputs import VI_CONFIGS, make_reward
    rank, world, local = dist_env()
    w = VI_CONFIGS[args.config]
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:                                  # replicas only
        import torch.distributed as tdist
        tdist.init_process_group("nccl", init_method="env://", device_id=dev)
    g = capi.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    Rh = make_reward(w)
    R = torch.from_numpy(Rh).to(dev)
    V = torch.empty(w.N, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            import torch.distributed as tdist
            tdist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as tdist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        capi.vi_solve(g, w.model, w.params, R, V=V, stream=stream)
    # Table 3's grid shapes: seconds per solve, for context (different, unstated MDP)
    table3 = {}
    for name in ("v0", "v1"):
        wt = VI_CONFIGS[name]
        gt = capi.Grid(wt.N, wt.lo, wt.hi, wt.periodic_mask)
        Rt = torch.from_numpy(make_reward(wt)).to(dev)
        capi.vi_solve(gt, wt.model, wt.params, Rt, stream=stream)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        _, ti = capi.vi_solve(gt, wt.model, wt.params, Rt, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        table3["x".join(map(str, wt.N))] = {"seconds": a.elapsed_time(b) / 1e3, "iterations": ti["iters"]}
        gt.close()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters, launches = 0, 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            _, info = capi.vi_solve(g, w.model, w.params, R, V=V, stream=stream)
            iters += info["iters"]
            launches += g.launch_count()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        _, tinfo = capi.vi_solve(g, w.model, w.params, R, V=V, stream=stream, use_graph=False)
    clocks = clk.summary()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    value = w.points * iters * world / (total_ms / 1e3)
    Vp = torch.empty(w.N, dtype=torch.float32).pin_memory()
    Rp = torch.from_numpy(Rh).pin_memory()
    capi.vi_solve_host(g, w.model, w.params, Rp.numpy(), V=Vp.numpy())
    barrier()
    t0 = time.perf_counter()
    e2e_it = 0
    for _ in range(max(1, min(args.steps, 3))):
        _, hi = capi.vi_solve_host(g, w.model, w.params, Rp.numpy(), V=Vp.numpy())
        e2e_it += hi["iters"]
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    peak, peak_kind = measured_peaks()
    it_ms = tinfo["iter_ms"] / tinfo["iters"]
    achieved = VI_BYTES * w.points / (it_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{w.name}:vi")
        except Exception:
            traffic = None
    line = {
        "metric": VI_METRIC, "value": value, "unit": VI_UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name, "grid": list(w.N), "points": w.points, "model": w.model,
                   "params": list(w.params), "threshold": 1e-6, "iterations_per_step": iters / args.steps,
                   "order": "Jacobi (reading A38)",
                   "l2": ("inputs larger than L2: R + 2 iterates = %.0f MB per iteration vs 126 MB L2" %
                          (w.points * 12 / 1e6)) if w.points * 12 > 126e6 else "fits L2",
                   "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                   "table3_shapes": table3},
        "roofline": {"bound": "hbm", "kernel": "k_vi_march (Alg. 1 l.4-8, one Bellman iteration)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind, "bytes_per_point": VI_BYTES, "avg_launch_ms": it_ms},
        "clocks": clocks,
        "e2e": {"value": w.points * e2e_it * world / e2e_s, "unit": VI_UNIT, "h2d_bytes_per_step": w.points * 4,
                "d2h_bytes_per_step": w.points * 4},
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, sample, cores, el, work = vi_oracle_sample(w, target_s=args.ref_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": VI_UNIT, "cores": cores, "kind": "oracle", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
        tdist.destroy_process_group()


def run_vi_reference(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            return
    from inputs import VI_CONFIGS
    w = VI_CONFIGS[args.config]
    times, work = [], []
    for i in range(args.warmup + args.steps):
        rate, sample, cores, el, wk = vi_oracle_sample(w, target_s=args.ref_seconds)
        if i >= args.warmup:
            times.append(el)
            work.append(wk)
    value = sum(work) / sum(times)
    line = {"impl": "reference", "metric": VI_METRIC, "value": value, "unit": VI_UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "grid": list(w.N)},
            "cpu_baseline": {"value": value, "unit": VI_UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": VI_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            return
    from inputs import CONFIGS
    w = CONFIGS[args.config]
    times, work = [], []
    for i in range(args.warmup + args.steps):
        rate, sample, cores, el, pts = oracle_sample(w, target_s=args.ref_seconds)
        if i >= args.warmup:
            times.append(el)
            work.append(pts)
    value = sum(work) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": w.name, "grid": list(w.N), "accuracy": w.accuracy,
                                             "mode": w.mode},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import paper_2204_05520_b200 as odp
    from paper_2204_05520_b200 import dist as odist
    from inputs import CONFIGS
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", init_method="env://", device_id=dev)
    w = CONFIGS[args.config]
    g = odist.partitioned_grid(w, rank, world, local)            # axis-0 slab of this rank (world > 1)
    i0b, n0 = g.local_extent()
    V0h = odist.local_v0(w, rank, world)
    V0 = torch.from_numpy(V0h).to(dev)
    nout = len(w.tau) - 1
    out = torch.empty((nout,) + g.local_N, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def one(timing=False):
        return odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, out=out, cfl=w.cfl,
                            kernel=args.kernel, stream=stream, timing=timing)[1]

    def barrier():
        if world > 1:
            import torch.distributed as tdist
            tdist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as tdist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        info = one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kms = {"pass1": 0.0, "pass2": 0.0, "control": 0.0, "pass2_rk2": 0.0}
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            info = one()                 # the production path (CUDA graphs where they apply)
            launches += g.launch_count()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        # per-kernel device times (roofline): one more solve with per-launch CUDA events recorded
        # on the launching stream by the library (direct launches: events need them)
        tinfo = one(timing=True)
        for k in kms:
            kms[k] += tinfo["kernel_ms"][k]
    clocks = clk.summary()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    P = w.points                                   # whole grid: value is the whole-job aggregate
    stages = info["stages"]
    value = P * stages * args.steps / (total_ms / 1e3)

    # end to end through the C-ABI host entry point: pinned host V0 slab -> device -> solve -> host out
    V0p = torch.from_numpy(V0h).pin_memory()
    outp = torch.empty((nout,) + g.local_N, dtype=torch.float32).pin_memory()
    odp.hj_solve_host(g, w.dynamics, w.params, V0p, w.tau, w.accuracy, w.mode, out=outp, cfl=w.cfl,
                      kernel=args.kernel)
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        odp.hj_solve_host(g, w.dynamics, w.params, V0p, w.tau, w.accuracy, w.mode, out=outp, cfl=w.cfl,
                          kernel=args.kernel)
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e_value = P * stages / e2e_s

    peak, peak_kind = measured_peaks()
    key = (w.accuracy, w.mode)
    Pl = g.points                                  # this rank's points (the kernels' launch unit)
    steps_t = tinfo["steps"]
    pass1_ms = kms["pass1"] / stages               # one pass-1 launch per stage (the timed solve)
    sm_hz = (clocks.get("sm_mhz") or 1900.0) * 1e6
    prof = ncu_kernel_profile(w.name) if world == 1 else {}
    if w.accuracy == "medium":
        p2 = {"pass2_rk1": ((kms["pass2"] - kms["pass2_rk2"]) / steps_t, PASS2_BYTES[key + (1,)]),
              "pass2_rk2": (kms["pass2_rk2"] / steps_t, PASS2_BYTES[key + (2,)])}
    else:
        p2 = {"pass2": (kms["pass2"] / stages, PASS2_BYTES[key])}
    kernels = {"pass1": (pass1_ms, PASS1_BYTES)}
    kernels.update(p2)
    ktab = {}
    for kname, (ms, bpp) in kernels.items():
        ach = bpp * Pl / (ms / 1e3) / 1e9
        ent = {"avg_launch_ms": ms, "bytes_per_point": bpp, "achieved": ach, "frac": ach / peak}
        pk = prof.get(kname)
        if pk:
            # issue roofline: the launch's warp instructions at one per SMSP per cycle, at the live clock
            t_issue = pk["warp_inst"] / (N_SMSP * sm_hz) * 1e3
            ent.update({"traffic": pk["dram_bytes"], "traffic_per_point": pk["dram_bytes"] / Pl,
                        "warp_inst": pk["warp_inst"], "issue_bound_ms": t_issue, "issue_frac": t_issue / ms,
                        "ncu_issue_active": pk["issue_active_pct"] / 100.0})
        ktab[kname] = ent
    # the dominant kernel: pass 2 (the largest share of the step, ~0.57 on c4).  MEDIUM runs it as two
    # instances of one kernel template (RK stage 1 / 2); its roofline is the mean launch:
    # the mean algorithmic bytes (8 and 16 B/pt -> 12) over the mean launch time, the mean ncu traffic
    # and instructions per launch.  The per-stage entries stay in `kernels`.
    if len(p2) > 1:
        ents = [ktab[k] for k in p2]
        ms_m = sum(e["avg_launch_ms"] for e in ents) / len(ents)
        bpp_m = sum(e["bytes_per_point"] for e in ents) / len(ents)
        d = {"avg_launch_ms": ms_m, "bytes_per_point": bpp_m}
        d["achieved"] = bpp_m * Pl / (ms_m / 1e3) / 1e9
        d["frac"] = d["achieved"] / peak
        if all("traffic" in e for e in ents):
            d["traffic"] = sum(e["traffic"] for e in ents) / len(ents)
            d["issue_bound_ms"] = sum(e["issue_bound_ms"] for e in ents) / len(ents)
            d["issue_frac"] = d["issue_bound_ms"] / ms_m
            d["ncu_issue_active"] = sum(e["ncu_issue_active"] for e in ents) / len(ents)
        dom = "pass2_mean"
    else:
        dom = "pass2"
        d = ktab[dom]
    stage_ms = pass1_ms + sum(v[0] for v in p2.values()) / len(p2)
    stage_gbs = STAGE_BYTES[key] * Pl / (stage_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name, "grid": list(w.N), "points": P, "dynamics": w.dynamics,
                   "accuracy": w.accuracy, "mode": w.mode, "cfl": w.cfl, "tau": [w.tau[0], w.tau[-1]],
                   "rk_stages_per_step": stages, "time_steps_per_step": info["steps"], "kernel": args.kernel,
                   "l2": "inputs larger than L2 (2 x %.1f GB working arrays per GPU)" % (Pl * 4 / 1e9)
                   if Pl * 4 > 126e6 else "fits L2",
                   "parallelism": "single GPU" if world == 1 else f"axis-0 slabs x{world} (NCCL halo + allreduce)",
                   "slab": [i0b, n0]},
        "roofline": {"bound": "hbm", "kernel": {"pass2_mean": "pass 2 (D+-, H, dissipation, stage update, BRT min), mean "
                                                              "of its RK stage 1 / 2 launches (8 / 16 B/pt)",
                                                "pass2": "pass 2, Euler stage (D+-, H, dissipation, update, BRT min)"}[dom],
                     "share": kms["pass2"] / max(total_ms / args.steps, 1e-9),
                     "achieved": d["achieved"], "peak": peak, "unit": "GB/s", "frac": d["frac"],
                     "traffic": d.get("traffic"), "peak_kind": peak_kind, "bytes_per_point": d["bytes_per_point"],
                     "avg_launch_ms": d["avg_launch_ms"],
                     "issue": ({"bound_ms": d["issue_bound_ms"], "frac": d["issue_frac"],
                                "ncu_issue_active": d["ncu_issue_active"],
                                "note": "warp instructions per launch (ncu) at 1 per SMSP per cycle at the live SM clock"}
                               if "issue_frac" in d else None),
                     "kernels": ktab,
                     "stage": {"bytes_per_point": STAGE_BYTES[key], "ms": stage_ms, "achieved": stage_gbs,
                               "frac": stage_gbs / peak},
                     "traffic_source": "profiles/ncu_kernels.json (ncu --set full, one launch per kernel and RK stage)"},
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": Pl * 4 * world,
                "d2h_bytes_per_step": Pl * 4 * nout * world},
        "gpu_launches": launches,
        "kernel_ms_share": {k: v / max(total_ms / args.steps, 1e-9) for k, v in kms.items() if k != "pass2_rk2"},
    }
    if launches <= 2 * args.steps:
        # the resident kernel ran (small grid, ODP_KERNEL_RESIDENT: k_init_state + one cooperative launch
        # per solve); the per-launch kernel table above describes the launch-per-pass path of the timed
        # solve instead.  The resident launch IS the solve: its roofline is the whole solve's
        # algorithmic bytes over the solve's device time, against HBM even though the grid sits in L2
        solve_s = total_ms / args.steps / 1e3
        ach = STAGE_BYTES[key] * Pl * stages / solve_s / 1e9
        line["roofline"] = {"bound": "hbm", "kernel": "k_resident (whole solve in one cooperative launch)",
                            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
                            "peak_kind": peak_kind, "bytes_per_point": STAGE_BYTES[key], "avg_launch_ms": solve_s * 1e3,
                            "note": "grid fits in L2: latency-bound (two grid barriers and two L2 round trips "
                                    "per stage), not HBM-bound; launch-per-pass kernel table in roofline_launch_path",
                            "roofline_launch_path": line["roofline"]}
        line["kernel_ms_share"] = {"k_resident": 1.0}
    if args.single_pass_too:
        # the same solve without pass 1 after the first step (alpha^max fixed for a
        # functor whose alpha does not depend on the derivative range); bitwise the two-pass result
        ref = out.clone()
        sp_info = odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, out=out, cfl=w.cfl,
                               kernel=args.kernel, stream=stream, single_pass=True)[1]
        torch.cuda.synchronize()
        same = bool(torch.equal(out, ref))
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            sp_info = odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, out=out, cfl=w.cfl,
                                   kernel=args.kernel, stream=stream, single_pass=True)[1]
        e1.record(stream)
        torch.cuda.synchronize()
        sp_ms = max_over_ranks(e0.elapsed_time(e1))
        line["single_pass"] = {"value": P * stages * args.steps / (sp_ms / 1e3), "unit": UNIT,
                               "ms_per_step": sp_ms / args.steps, "used": bool(sp_info["single_pass"]),
                               "bitwise_equal_to_two_pass": same,
                               "note": "SURVEY.md §8(f1) variant, not the headline (Alg. 2's two passes)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, sample, cores, el, pts = oracle_sample(w, target_s=args.ref_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
        tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "generic", "tiled", "stream", "march"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--single-pass-too", type=int, default=1,
                    help="also time the single-pass variant (SURVEY.md §8(f1)) and report it beside the headline")
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    args = ap.parse_args()
    from inputs import TTR_CONFIGS, VI_CONFIGS
    if args.config in TTR_CONFIGS:
        (run_ttr_reference if args.impl == "reference" else run_ttr)(args)
    elif args.config in VI_CONFIGS:
        (run_vi_reference if args.impl == "reference" else run_vi)(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
