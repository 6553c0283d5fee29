"""Benchmark: one step = one complete GMRES(30) solve (tol 1e-6, x0 = 0) of the all-at-once
KKT system preconditioned by the block-circulant Algorithm 1 -- every row of SURVEY 8(a)
(A1 outer GMRES, A2 kkt_apply, A3 time DFT + T_l^-1, A4-A6 per-frequency block solves with
MG / Chebyshev, A8 T_r^-1 + inverse DFT) -- on BASELINE.json configs[1] (c2: 2-D Stokes,
Q2-Q1 64x64, n_t = 64, beta = 1e-2), synthetic seeded data (synth/).

Metric: space-time DOF/s = N x (GMRES iterations) / solve time, plus
preconditioner applications/s and the HBM roofline fraction of the dominant kernel class.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c2]

N > 1 (torchrun): independent replicas, one per GPU ("replicas only"):
the path has no inter-GPU exchange at this size.  --impl reference times the CPU oracle
(oracle/, the plain paper-order implementation) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time DOF/s & precond applies/s (fp64, 1 B200); % of HBM roofline"
UNIT = "DOF/s"


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.lines = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(gpu_index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def aggregate_replicas(ms, iterations, world, device="cuda"):
    """Whole-job numbers over independent replicas: time = MAX over ranks, work = SUM over ranks.

    Returns (max_ms, total_iterations).  World size 1 needs no process group.
    """
    if world == 1:
        return float(ms), float(iterations)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    it = torch.tensor([float(iterations)], dtype=torch.float64, device=device)
    dist.all_reduce(it, op=dist.ReduceOp.SUM)
    return float(t.item()), float(it.item())


# ---------------------------------------------------------------------------------------------
def oracle_iteration_sample(cfg, reps, warm):
    """The CPU oracle as it stands, timed on one GMRES iteration's work: precond_apply (all n_b
    frequencies) + kkt_apply + modified Gram-Schmidt against 15 basis vectors (the mean Krylov
    dimension of a restart-30 cycle).  Returns (seconds per sample, cores used)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import kkt, precond
    from oracle.problem import Problem
    import synth

    with threadpool_limits(limits=1):
        prob = Problem(cfg, synth.wind(cfg))
        pc = precond.OraclePreconditioner(prob)
        rng = np.random.default_rng(0)
        V = [synth.probe_vector(cfg, seed_offset=i) for i in range(16)]
        V = [v / np.linalg.norm(v) for v in V]
        times = []
        for it in range(warm + reps):
            t0 = time.perf_counter()
            z = pc.apply(V[0])
            w = kkt.kkt_apply(prob, z)
            for i in range(15):
                h = np.dot(w, V[i])
                w = w - h * V[i]
            np.linalg.norm(w)
            if it >= warm:
                times.append(time.perf_counter() - t0)
        del rng
    return times, 1


def run_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return 0
    import synth
    cfg = synth.CONFIGS[args.config]
    times, cores = oracle_iteration_sample(cfg, args.steps, args.warmup)
    t = sum(times) / len(times)
    value = cfg.n_dofs / t
    sample = (f"one GMRES iteration of {cfg.name} per step: oracle precond_apply (all {cfg.n_b} frequencies) "
              f"+ kkt_apply + MGS against 15 basis vectors")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth/, seeded)",
            "config": {"workload": cfg.name, "dim": cfg.dim, "n_cells": cfg.n_cells, "n_t": cfg.n_t,
                       "beta": cfg.beta, "nu": cfg.nu, "n_dofs": cfg.n_dofs, "parallelism": "cpu oracle"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2405_18964_b200 import Context

    rank, world, local = rank_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[args.config]
    ctx = Context.from_config(cfg, synth.wind(cfg))
    stream = torch.cuda.current_stream()
    b = ctx.build_rhs(synth.desired_state(cfg))
    x = torch.zeros_like(b)

    def solve():
        x.zero_()
        return ctx.gmres_solve(b, x, tol=1e-6, restart=30)

    for w in range(args.warmup):
        if w == args.warmup - 1:
            ctx.profile_smoother(True)      # last warm-up: creates the profiling events the timed region reuses
        _, info, hist, rc = solve()
    ctx.profile_read()
    ctx.profile_smoother(False)
    launches_per_step = ctx.last_launch_count()
    its = info["iterations"]

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- timed region: K full solves, device events, max over ranks
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile_smoother(True)   # dominant kernel timed live: events around each velocity-MG launch, same stream
    e0.record(stream)
    its_total = 0
    for _ in range(args.steps):
        _, info, _, _ = solve()
        its_total += info["iterations"]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    sm_ms, sm_bytes, sm_launches = ctx.profile_read()
    ctx.profile_smoother(False)
    ms, its_all = aggregate_replicas(e0.elapsed_time(e1), its_total, world)
    ms_per_step = ms / args.steps
    value = cfg.n_dofs * its_all / (ms / 1e3)

    # ---------------- isolated applications (precond applies/s, kkt DOF/s), after the timed region
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        ctx.precond_apply(r, z)
    torch.cuda.synchronize()
    n_app = 10
    e0.record(stream)
    for _ in range(n_app):
        ctx.precond_apply(r, z)
    e1.record(stream)
    torch.cuda.synchronize()
    precond_ms = e0.elapsed_time(e1) / n_app
    precond_launches = ctx.last_launch_count()
    for _ in range(3):
        ctx.kkt_apply(r, z)
    e0.record(stream)
    for _ in range(n_app):
        ctx.kkt_apply(r, z)
    e1.record(stream)
    torch.cuda.synchronize()
    kkt_ms = e0.elapsed_time(e1) / n_app

    # ---------------- dominant kernel (velocity MG launches) over the timed region, read above
    peaks = load_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    achieved = sm_bytes / (sm_ms / 1e3) / 1e9 if sm_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "smoother_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": "k_mg_cta<2,2>: CTA-resident velocity multigrid solve (4 V-cycles, all levels)" if os.environ.get("AAO_MG_MODE", "0") != "1" else "k_gs<2,2> finest-level multicolour SOR sweeps",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks else "fallback (B200_PROFILING.md)",
                "traffic": traffic, "algorithmic_bytes_per_launch": sm_bytes / max(sm_launches, 1),
                "avg_launch_us": 1e3 * sm_ms / max(sm_launches, 1), "share_of_step": sm_ms / (ms_per_step * args.steps),
                "measured": f"CUDA events around every velocity-MG launch of the {args.steps} timed solves"}

    # ---------------- end to end through the public API with HOST buffers (copies inside)
    bh = torch.empty(ctx.N, dtype=torch.float64).pin_memory()
    bh.copy_(b.cpu())
    xh = torch.zeros(ctx.N, dtype=torch.float64).pin_memory()
    ctx.gmres_solve_host(bh, xh)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    its_e2e = 0
    for _ in range(args.steps):
        xh.zero_()
        _, info_e, _, _ = ctx.gmres_solve_host(bh, xh)
        its_e2e += info_e["iterations"]
    torch.cuda.synchronize()
    e2e_s, its_e2e_all = aggregate_replicas(time.perf_counter() - t0, its_e2e, world)
    e2e_value = cfg.n_dofs * its_e2e_all / e2e_s

    # ---------------- NEXT-1: Algorithm 2 + FGMRES(10) on the same workload (reported, not the value)
    nl = None
    if not args.no_nonlinear:
        ctx_nl = Context.from_config(cfg, synth.wind(cfg), nonlinear=True, inner_eps=1e-2, inner_maxit=60)
        b_nl = ctx_nl.build_rhs(synth.desired_state(cfg))
        ctx_nl.gmres_solve(b_nl, tol=1e-6, restart=10)          # warm-up
        torch.cuda.synchronize()
        e0.record(stream)
        _, info_nl, _, _ = ctx_nl.gmres_solve(b_nl, tol=1e-6, restart=10)
        e1.record(stream)
        torch.cuda.synchronize()
        t_nl = e0.elapsed_time(e1) / 1e3
        nl = {"solver": "Algorithm 2 (inner GMRES per frequency, eps 1e-2) + FGMRES(10), tol 1e-6",
              "fgmres_iterations": info_nl["iterations"], "converged": info_nl["converged"],
              "inner_avg_per_frequency": info_nl["inner_its_total"] / max(1, info_nl["precond_applies"] * cfg.n_f),
              "solve_s": t_nl, "dofs_x_outer_its_per_s": cfg.n_dofs * info_nl["iterations"] / t_nl}
        ctx_nl.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times, cores = oracle_iteration_sample(cfg, 1, 0)
        cpu = {"value": cfg.n_dofs / times[0], "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"one GMRES iteration of {cfg.name}: oracle precond_apply (all {cfg.n_b} frequencies) + "
                         f"kkt_apply + MGS against 15 basis vectors, {times[0]:.1f} s"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (synth/: seeded stream-function desired state, BASELINE configs)",
                "config": {"workload": cfg.name, "problem": cfg.problem, "dim": cfg.dim, "n_cells": cfg.n_cells,
                           "n_t": cfg.n_t, "beta": cfg.beta, "nu": cfg.nu, "n_dofs": cfg.n_dofs,
                           "step": "one GMRES(30) solve to 1e-6 from x0=0", "gmres_iterations": its,
                           "parallelism": f"replicas x{world}",
                           "l2": "no flush: per-step working set (31-vector Krylov basis + 30 preconditioned vectors, "
                                 f"{61 * cfg.n_dofs * 8 / 1e9:.2f} GB) exceeds the 126 MB L2"},
                "precond_applies_per_s": 1e3 / precond_ms, "precond_ms": precond_ms,
                "precond_dofs_per_s": cfg.n_dofs / (precond_ms / 1e3),
                "kkt_ms": kkt_ms, "kkt_dofs_per_s": cfg.n_dofs / (kkt_ms / 1e3),
                "kkt_hbm_frac": (16.0 * cfg.n_dofs / (kkt_ms / 1e3) / 1e9) / peak,
                "roofline": roofline, "clocks": clocks,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * cfg.n_dofs,
                        "d2h_bytes_per_step": 8 * cfg.n_dofs},
                "gpu_launches": launches_per_step * args.steps, "launches_per_precond": precond_launches,
                "nonlinear": nl,
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nonlinear", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
