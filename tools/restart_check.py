"""Is the c3/c5 stagnation a GMRES(30) restart effect?  Solve with a larger restart."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2405_18964_b200 import Context
for name, restart, cap in (("c5", 64, 640), ("c3", 64, 640)):
    cfg = synth.CONFIGS[name]
    ctx = Context.from_config(cfg, synth.wind(cfg))
    b = ctx.build_rhs(synth.desired_state(cfg))
    t0 = time.time()
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=restart, max_iters=cap)
    torch.cuda.synchronize()
    print(json.dumps({"config": name, "restart": restart, "iterations": info["iterations"], "converged": info["converged"],
                      "true_relres": info["true_relres"], "s": time.time() - t0,
                      "hist_every_64": hist[::64] + hist[-1:]}), flush=True)
    ctx.close(); del ctx, b, x; torch.cuda.empty_cache()
