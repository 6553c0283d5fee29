"""Per-config measurements on the GPU for every BASELINE.json workload: precond_apply / kkt_apply times
(CUDA events, warm), device memory, and (where the Krylov basis fits and time allows) a full
GMRES(30) solve to 1e-6 with its iteration count.  Writes one JSON line per config."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402


def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c2b,c3,c4_32,c4_64,c4_128,c4_256,c4_512,c5")
ap.add_argument("--solve", default="c1,c2,c2b,c3,c4_32,c5")
ap.add_argument("--max-iters", type=int, default=2000)
ap.add_argument("--solve-budget-s", type=float, default=240.0)
a = ap.parse_args()
for name in a.configs.split(","):
    cfg = synth.CONFIGS[name]
    out = {"config": name, "N": cfg.n_dofs, "n_b": cfg.n_b, "problem": cfg.problem, "dim": cfg.dim}
    try:
        t0 = time.time()
        ctx = Context.from_config(cfg, synth.wind(cfg))
        out["setup_s"] = time.time() - t0
        r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
        z = torch.empty_like(r)
        out["precond_ms"] = ev_time(lambda: ctx.precond_apply(r, z), 2 if cfg.n_dofs < 2e8 else 1)
        out["kkt_ms"] = ev_time(lambda: ctx.kkt_apply(r, z), 5)
        out["precond_dofs_per_s"] = cfg.n_dofs / (out["precond_ms"] / 1e3)
        out["kkt_dofs_per_s"] = cfg.n_dofs / (out["kkt_ms"] / 1e3)
        out["kkt_hbm_GBs"] = 16.0 * cfg.n_dofs / (out["kkt_ms"] / 1e3) / 1e9
        out["device_bytes_ctx"] = ctx.device_bytes()
        del r, z
        if name in a.solve.split(","):
            free, _ = torch.cuda.mem_get_info()
            need = 36 * 8 * cfg.n_dofs
            est_s = out["precond_ms"] / 1e3 * 500
            if need < free * 0.9:
                b = ctx.build_rhs(synth.desired_state(cfg))
                cap = a.max_iters
                if est_s > a.solve_budget_s:
                    cap = max(30, int(a.solve_budget_s / (out["precond_ms"] / 1e3)))
                torch.cuda.synchronize()
                t0 = time.time()
                x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=30, max_iters=cap)
                torch.cuda.synchronize()
                dt = time.time() - t0
                out.update({"gmres_iterations": info["iterations"], "gmres_converged": info["converged"],
                            "gmres_true_relres": info["true_relres"], "gmres_s": dt, "gmres_cap": cap,
                            "solve_dofs_per_s": cfg.n_dofs * info["iterations"] / dt,
                            "hist_tail": hist[-3:]})
                del b, x
            else:
                out["gmres_skipped"] = f"basis needs {need / 1e9:.0f} GB, free {free / 1e9:.0f} GB"
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    except Exception as e:  # record and continue
        out["error"] = repr(e)[:300]
    print(json.dumps(out), flush=True)
