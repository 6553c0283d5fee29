"""Benchmark of the hot path on the largest single-GPU BASELINE configuration.

Workload (default): c4 at n_t = 512 -- 2-D unsteady Stokes control, Q2-Q1 on 256 x 256 cells, 511 time blocks,
N = 6.05e8 space-time DOFs (BASELINE.json configs[3], the top of its n_t sweep; 34 Krylov-sized vectors of
4.84 GB fill the HBM).  One step = the first restart cycle of right-preconditioned GMRES(30) from x0 = 0
(30 Arnoldi iterations -- each = Algorithm 1's preconditioner (A3 time DFT + T_l^-1, A4-A6 per-frequency
multigrid / Chebyshev block solves, A8 T_r^-1 + inverse DFT), the KKT matvec (A2) and modified Gram-Schmidt
(A1) -- then the restart update x += P^-1(V y) and the true residual): every row of SURVEY 8(a).  The full
c4_512 solve needs many restart cycles (minutes); a cycle is the repeatable unit of the same solve.

Metric: space-time DOF/s = N x (GMRES iterations) / time, plus preconditioner applications/s,
KKT DOF/s and the HBM roofline fraction of the dominant kernel (the velocity multigrid, timed live with CUDA
events around each launch inside the timed region).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c4_512]

N > 1 (torchrun): independent replicas, one per GPU ("replicas only"), weak scaling.
--impl reference times the CPU oracle (oracle/, the plain paper-order implementation) on the host cores on a
bounded, frequency-sampled sample of the same workload (extrapolated), rank 0 only.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
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
RESTART = 30


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def source_hash():
    """Hash of the sources of the dominant kernel and its launch configuration (kernels_stencil.cu, aao.cu,
    aao_internal.h): an ncu traffic record is used only for the build it was captured on."""
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2405_18964_b200", "csrc")
    for f in ("aao.cu", "aao_internal.h", "kernels_stencil.cu"):
        h.update(open(os.path.join(d, f), "rb").read())
    return h.hexdigest()[:16]


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


# --------------------------------------------------------------------------------------------- CPU oracle
_ORACLE_PC = None


def _oracle_block(arg):
    """One frequency block of the oracle's Algorithm 1 (pool worker; forked, inherits _ORACLE_PC)."""
    import numpy as np
    k, seed = arg
    pc = _ORACLE_PC
    f = pc.prob.fine
    rng = np.random.default_rng(seed)
    cz = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    t0 = time.perf_counter()
    pc.block(k, cz(pc.dim, f.nI), cz(pc.dim, f.nI), cz(f.npu), cz(f.npu))
    return time.perf_counter() - t0


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class OracleSample:
    """The CPU oracle as it stands, timed on a bounded sample of one GMRES iteration of `cfg` and extrapolated
    (SURVEY 8(d) D.5):  t_iter = T_blocks * ceil(n_b / P) + t_dft * (dft scale) + t_kkt_mgs * (kkt scale), where
      T_blocks : wall time of P frequency-block solves (Algorithm 1's loop body, k spread over [0, n_b)) run
                 concurrently on P = host cores worker processes;
      t_dft    : the oracle's forward + inverse DFT (timeops.dft / idft) on a slab of spatial columns, scaled to all
                 2 (n_v + n_p) series;
      t_kkt_mgs: kkt_apply + MGS against 15 basis vectors (the mean of a restart-30 cycle) on the config with the
                 same mesh and n_t = 32 (if cfg is larger), scaled by the N ratio (both are linear in N)."""

    def __init__(self, cfg):
        import numpy as np
        from threadpoolctl import threadpool_limits

        import synth
        from oracle import precond
        from oracle.problem import Problem
        global _ORACLE_PC
        self.cfg = cfg
        self.cores = cpu_cores()
        self.limits = threadpool_limits(limits=1)
        self.prob = Problem(cfg, synth.wind(cfg))
        self.pc = precond.OraclePreconditioner(self.prob, cache_blocks=False)
        _ORACLE_PC = self.pc
        import multiprocessing as mp
        self.P = max(1, min(self.cores, cfg.n_b))
        self.pool = mp.get_context("fork").Pool(self.P)
        small = cfg
        if cfg.n_dofs > 4e7 and cfg.problem == "stokes":
            small = synth.Config(cfg.name + "@nt32", cfg.index, cfg.dim, cfg.n_cells, cfg.x_lo, cfg.x_hi, 32, cfg.T,
                                 cfg.beta, cfg.nu, cfg.problem)
        self.small = small
        self.sprob = self.prob if small is cfg else Problem(small, synth.wind(small))
        self.V = [synth.probe_vector(small, seed_offset=i) for i in range(16)]
        self.V = [v / np.linalg.norm(v) for v in self.V]
        self.slab = min(4096, cfg.n_v + cfg.n_p)
        self.step_i = 0

    def step(self):
        import numpy as np
        from oracle import kkt, timeops
        cfg = self.cfg
        ks = [int((self.step_i * 7919 + j * cfg.n_b / self.P)) % cfg.n_b for j in range(self.P)]
        self.step_i += 1
        t0 = time.perf_counter()
        self.pool.map(_oracle_block, [(k, 1000 + k) for k in ks])
        t_blocks = time.perf_counter() - t0
        x = np.random.default_rng(5).standard_normal((cfg.n_b, self.slab))
        t0 = time.perf_counter()
        xh = timeops.dft(x)
        timeops.idft(xh)
        t_dft = (time.perf_counter() - t0) * (2.0 * (cfg.n_v + cfg.n_p) / self.slab)
        t0 = time.perf_counter()
        w = kkt.kkt_apply(self.sprob, self.V[0])
        for i in range(15):
            h = np.dot(w, self.V[i])
            w = w - h * self.V[i]
        np.linalg.norm(w)
        t_km = (time.perf_counter() - t0) * (cfg.n_dofs / self.small.n_dofs)
        t_iter = t_blocks * math.ceil(cfg.n_b / self.P) + t_dft + t_km
        return t_iter, dict(t_blocks=t_blocks, t_dft=t_dft, t_kkt_mgs=t_km, ks=ks)

    def describe(self, t_iter):
        cfg = self.cfg
        return (f"one GMRES iteration of {cfg.name} extrapolated from a sample (SURVEY D.5): {self.P} oracle "
                f"frequency-block solves (Algorithm 1 loop body) run concurrently on {self.P} processes x "
                f"ceil({cfg.n_b}/{self.P}) + the oracle DFT pair on {self.slab} of {2 * (cfg.n_v + cfg.n_p)} series "
                f"scaled + kkt_apply and MGS(15) on {self.small.name} scaled by N; {t_iter:.1f} s per iteration; "
                f"host CPU {cpu_model()}")

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return 0
    import synth
    cfg = synth.CONFIGS[args.config]
    o = OracleSample(cfg)
    for _ in range(args.warmup):
        o.step()
    times = []
    for _ in range(args.steps):
        t, _ = o.step()
        times.append(t)
    o.close()
    t = sum(times) / len(times)
    value = cfg.n_dofs / t          # one iteration per sample: N x 1 / t_iter
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth/, seeded)",
            "config": {"workload": cfg.name, "dim": cfg.dim, "n_cells": cfg.n_cells, "n_t": cfg.n_t,
                       "beta": cfg.beta, "nu": cfg.nu, "n_dofs": cfg.n_dofs, "parallelism": f"cpu oracle x{o.P}",
                       "step": "one GMRES iteration (extrapolated from a frequency-sampled oracle sample)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": o.P, "kind": "oracle", "extrapolated": True,
                             "sample": o.describe(t)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------------- GPU path
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
    max_its = RESTART if args.cycle else 100000

    def step():
        x.zero_()
        return ctx.gmres_solve(b, x, tol=1e-6, restart=RESTART, max_iters=max_its)

    for _ in range(args.warmup):
        _, info, hist, rc = step()
    launches_per_step = ctx.last_launch_count()
    its = info["iterations"]

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------- timed region: K steps, device events on the launching stream, max over ranks
    ctx.profile_smoother(True, reserve=4 * (its + 2) * max(1, math.ceil(cfg.n_f / 16)) * args.steps)
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    its_total = 0
    for _ in range(args.steps):
        _, info, _, _ = step()
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
    relres_step = info["final_relres"]

    # ---------------- isolated applications (precond applies/s, kkt DOF/s), after the timed region
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    z = x
    for _ in range(2):
        ctx.precond_apply(r, z)
    torch.cuda.synchronize()
    n_app = 5
    e0.record(stream)
    for _ in range(n_app):
        ctx.precond_apply(r, z)
    e1.record(stream)
    torch.cuda.synchronize()
    precond_ms = e0.elapsed_time(e1) / n_app
    precond_launches = ctx.last_launch_count()
    ctx.set_timing(True)
    ctx.precond_apply(r, z)
    phase = ctx.phase_ms()
    ctx.set_timing(False)
    for _ in range(2):
        ctx.kkt_apply(r, z)
    e0.record(stream)
    for _ in range(n_app):
        ctx.kkt_apply(r, z)
    e1.record(stream)
    torch.cuda.synchronize()
    kkt_ms = e0.elapsed_time(e1) / n_app
    del r

    # ---------------- dominant kernel (velocity MG launches) over the timed region, read above
    peaks = load_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    achieved = sm_bytes / (sm_ms / 1e3) / 1e9 if sm_ms > 0 else 0.0
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            rec = json.load(open(tpath)).get(cfg.name)
            if rec and rec.get("source_hash") == source_hash():
                traffic, traffic_src = rec["dram_bytes_per_launch"], rec["capture"]
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": "k_mg_cta<2,2,0,1>: CTA-resident velocity multigrid solve (4 V-cycles, "
                "all levels, band-wavefront sweeps on the 513^2 level), one launch per frequency chunk",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks else "fallback (B200_PROFILING.md)",
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": sm_bytes / max(sm_launches, 1),
                "avg_launch_us": 1e3 * sm_ms / max(sm_launches, 1), "launches": sm_launches,
                "share_of_step": sm_ms / (ms_per_step * args.steps),
                "measured": f"CUDA events on the launching stream around every velocity-MG launch of the "
                            f"{args.steps} timed steps (event pool created before the timed region)"}

    # ---------------- end to end through the public API with HOST buffers (copies inside the call)
    bh = torch.empty(ctx.N, dtype=torch.float64).pin_memory()
    bh.copy_(b.cpu())
    xh = torch.zeros(ctx.N, dtype=torch.float64).pin_memory()
    del b, x, z
    torch.cuda.empty_cache()        # the host entry stages b and x on the device itself
    ctx.gmres_solve_host(bh, xh, restart=RESTART, max_iters=max_its)
    torch.cuda.synchronize()
    barrier()
    e2e_steps = min(args.steps, args.e2e_steps)
    t0 = time.perf_counter()
    its_e2e = 0
    for _ in range(e2e_steps):
        xh.zero_()
        _, info_e, _, _ = ctx.gmres_solve_host(bh, xh, restart=RESTART, max_iters=max_its)
        its_e2e += info_e["iterations"]
    torch.cuda.synchronize()
    e2e_s, its_e2e_all = aggregate_replicas(time.perf_counter() - t0, its_e2e, world)
    e2e_value = cfg.n_dofs * its_e2e_all / e2e_s
    dev_gb = ctx.device_bytes() / 1e9
    free_gb = torch.cuda.mem_get_info()[0] / 1e9

    # ---------------- NEXT-1 (optional): Algorithm 2 + FGMRES(10) on the same workload, reported only
    nl = None
    if args.nonlinear:
        ctx.close()
        del bh, xh
        torch.cuda.empty_cache()
        ctx_nl = Context.from_config(cfg, synth.wind(cfg), nonlinear=True, inner_eps=1e-2, inner_maxit=60)
        b_nl = ctx_nl.build_rhs(synth.desired_state(cfg))
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
        o = OracleSample(cfg)
        t_it, parts = o.step()
        o.close()
        cpu = {"value": cfg.n_dofs / t_it, "unit": UNIT, "cores": o.P, "kind": "oracle", "extrapolated": True,
               "sample": o.describe(t_it)}
    if rank == 0:
        step_desc = (f"first GMRES({RESTART}) restart cycle from x0=0 ({RESTART} Arnoldi iterations: precond + kkt "
                     f"+ MGS; then x += P^-1(V y) and the true residual)" if args.cycle
                     else f"one complete GMRES({RESTART}) solve to 1e-6 from x0=0")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (synth/: seeded stream-function desired state, BASELINE configs)",
                "config": {"workload": cfg.name, "problem": cfg.problem, "dim": cfg.dim, "n_cells": cfg.n_cells,
                           "n_t": cfg.n_t, "beta": cfg.beta, "nu": cfg.nu, "n_dofs": cfg.n_dofs,
                           "step": step_desc, "gmres_iterations_per_step": its,
                           "relres_after_step": relres_step, "parallelism": f"replicas x{world}",
                           "l2": f"no flush: every step streams the {RESTART + 1}-vector Krylov basis "
                                 f"({(RESTART + 1) * cfg.n_dofs * 8 / 1e9:.1f} GB) >> 126 MB L2",
                           "device_gb": dev_gb, "free_gb_after": free_gb},
                "precond_applies_per_s": 1e3 / precond_ms, "precond_ms": precond_ms,
                "precond_phase_ms": {"fft_fwd": phase[0], "velocity_mg": phase[1], "pressure_join": phase[2],
                                     "fft_inv": phase[3]},
                "precond_dofs_per_s": cfg.n_dofs / (precond_ms / 1e3),
                "kkt_ms": kkt_ms, "kkt_dofs_per_s": cfg.n_dofs / (kkt_ms / 1e3),
                "kkt_hbm_frac": (16.0 * cfg.n_dofs / (kkt_ms / 1e3) / 1e9) / peak,
                "roofline": roofline, "clocks": clocks,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * cfg.n_dofs,
                        "d2h_bytes_per_step": 8 * cfg.n_dofs, "steps": e2e_steps,
                        "api": "aao_gmres_solve_host (pinned host b, x)"},
                "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
                "launches_per_precond": precond_launches,
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
    ap.add_argument("--config", default="c4_512")
    ap.add_argument("--full-solve", dest="cycle", action="store_false",
                    help="step = a complete GMRES solve to 1e-6 instead of one restart cycle")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nonlinear", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    return run_reference(args) if args.impl == "reference" else run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
