"""Order-of-magnitude anchors against the paper's iteration tables, on the GPU path.

Settings of P:825-827 (kept "for this and all subsequent experiments"): nu = 1e-2, T = 10, 4 V-cycles,
10 Chebyshev steps, GMRES restart 30; the manufactured v_d and f of P:815-820 are retained, with
the initial / boundary data of the exact v.  Omega = [-1,1]^2, Q2-Q1 here vs P2-P1 in the paper
(so the meshes are not identical: h_c ~ 32^2, h_f ~ 64^2 cells).  Blocks n_b = n_t - 1 match
the tables' "n_t" column (reading 3).
  table1: Algorithm 1 + GMRES(30), tol 1e-6
  table2: Algorithm 2 (eps 1e-2) + FGMRES(10), tol 1e-6
  table45: Oseen lid-driven cavity, Algorithm 2 with P~^(UZ), Uzawa 6   (Tables 4-5)
Writes one JSON line per run to stdout.  Usage: python tools/paper_tables.py [table1|table2|table45 ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

BETAS = (1e-1, 1e-3, 1e-4)
MESHES = (32, 64)
NTS = (16, 32, 64, 128)


def run(kind, nc, nt, beta):
    if kind == "table45":
        cfg = synth.cavity_config(nc, nt, beta=beta)
        w = synth.cavity_wind(cfg)
        data = synth.cavity_inputs(cfg)
    else:
        cfg = synth.mms_config(nc, nt, beta=beta, nu=1e-2, T=10.0)
        w = None
        data = synth.mms_inputs(cfg)
    nl = kind != "table1"
    opts = dict(nonlinear=True, inner_eps=1e-2, inner_maxit=60) if nl else {}
    ctx = Context.from_config(cfg, w, **opts)
    b = ctx.build_rhs_general(*data)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=10 if nl else 30, max_iters=200 if nl else 3000)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    out = {"table": kind, "mesh": f"{nc}x{nc}", "n_t": nt, "n_b": cfg.n_b, "beta": beta, "nu": cfg.nu, "T": cfg.T,
           "N": cfg.n_dofs, "iterations": info["iterations"], "converged": info["converged"],
           "true_relres": info["true_relres"], "solve_s": t}
    if nl:
        out["inner_avg_per_frequency"] = info["inner_its_total"] / max(1, info["precond_applies"] * cfg.n_f)
        out["inner_max"] = info["inner_its_max"]
    print(json.dumps(out), flush=True)
    ctx.close()
    del ctx, b, x
    torch.cuda.empty_cache()


if __name__ == "__main__":
    kinds = sys.argv[1:] or ["table1", "table2", "table45"]
    for kind in kinds:
        for nc in MESHES:
            for nt in NTS:
                for beta in BETAS:
                    run(kind, nc, nt, beta)
