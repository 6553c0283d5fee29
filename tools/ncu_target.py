"""ncu target: build one context and run `reps` preconditioner applications (and one kkt_apply), or, with
reps < 0, a GMRES(30) solve capped at -reps iterations (MGS, KKT and preconditioner launches of a real step).

usage: python tools/ncu_target.py <config> [reps] [freq_chunk]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = synth.CONFIGS[name]
ctx = Context.from_config(cfg, synth.wind(cfg), freq_chunk=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
if reps < 0:
    b = ctx.build_rhs(synth.desired_state(cfg))
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=30, max_iters=-reps)
    print("gmres", info["iterations"])
else:
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    z = torch.empty_like(r)
    for _ in range(reps):
        ctx.precond_apply(r, z)
    ctx.kkt_apply(r, z)
torch.cuda.synchronize()
print("done", name, ctx.device_bytes() / 1e9)
