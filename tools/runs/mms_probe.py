import sys; sys.path.insert(0, '.')
import numpy as np, synth
from paper_2405_18964_b200 import Context
from oracle.manufactured import solve_manufactured
for nc, nt in ((4, 8), (8, 16), (16, 32)):
    cfg = synth.mms_config(nc, nt)
    ctx = Context.from_config(cfg, None)
    b = ctx.build_rhs_general(*synth.mms_inputs(cfg))
    for restart in (30,):
        x, info, hist, rc = ctx.gmres_solve(b, tol=1e-10, restart=restart, max_iters=8000)
        xo = solve_manufactured(nc, nt, full=True)[2]
        xg = x.cpu().numpy()
        print(nc, nt, restart, info['iterations'], info['final_relres'], info['true_relres'], np.linalg.norm(xg-xo)/np.linalg.norm(xo), [hist[k] for k in (0, 100, 400, -1) if k < len(hist)], flush=True)
