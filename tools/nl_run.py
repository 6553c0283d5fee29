"""Algorithm 2 + FGMRES(10) (eps = 1e-2) on full BASELINE configs: outer/inner iterations and time."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2405_18964_b200 import Context
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c2b", "c3", "c5", "c4_32"]
for name in names:
    cfg = synth.CONFIGS[name]
    try:
        ctx = Context.from_config(cfg, synth.wind(cfg), nonlinear=True, inner_eps=1e-2, inner_maxit=60)
        b = ctx.build_rhs(synth.desired_state(cfg))
        torch.cuda.synchronize()
        t0 = time.time()
        x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=10, max_iters=60)
        torch.cuda.synchronize()
        dt = time.time() - t0
        out = {"config": name, "N": cfg.n_dofs, "fgmres_iterations": info["iterations"], "converged": info["converged"],
               "true_relres": info["true_relres"], "precond_applies": info["precond_applies"],
               "inner_avg_per_freq": info["inner_its_total"] / max(1, info["precond_applies"] * cfg.n_f),
               "inner_max": info["inner_its_max"], "seconds": dt,
               "dofs_it_per_s": cfg.n_dofs * info["iterations"] / dt, "hist": hist}
        ctx.close(); del ctx, b, x; torch.cuda.empty_cache()
    except Exception as e:
        out = {"config": name, "error": repr(e)[:300]}
    print(json.dumps(out), flush=True)
