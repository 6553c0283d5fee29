"""NEXT-2: the paper's Oseen lid-driven cavity solved with Algorithm 2 + FGMRES(10), eps = 1e-2,
Uzawa 6: outer / inner iteration counts and time per (mesh, n_t) -- compare Tables 4-5."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

for nc, nt in ((16, 17), (32, 17), (32, 33), (64, 33), (64, 65)):
    cfg = synth.cavity_config(nc, nt)
    w = synth.cavity_wind(cfg)
    ctx = Context.from_config(cfg, w, nonlinear=True, inner_eps=1e-2, inner_maxit=60)
    b = ctx.build_rhs_general(*synth.cavity_inputs(cfg))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=10, max_iters=200)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(json.dumps({"mesh": f"{nc}x{nc}", "n_t": nt, "N": cfg.n_dofs, "outer": info["iterations"],
                      "converged": info["converged"], "true_relres": info["true_relres"],
                      "inner_avg_per_frequency": info["inner_its_total"] / max(1, info["precond_applies"] * cfg.n_f),
                      "inner_max": info["inner_its_max"], "solve_s": t}), flush=True)
    del ctx
    torch.cuda.empty_cache()
