"""compute-sanitizer target (racecheck / synccheck / memcheck / initcheck): small configurations through every
kernel family -- c1 linear GMRES (CTA-resident MG, prime-factor transforms, time-marching KKT, on-chip MGS),
the band-wavefront sweeps forced on small levels (shared-memory ring + cp.async), Oseen and 3-D preconditioners,
Algorithm 2 (batched inner GMRES), the host-buffer entry and the RHS kernels.

usage: compute-sanitizer --tool <tool> python tools/sanitize_target.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402


def run(cfg, **kw):
    ctx = Context.from_config(cfg, synth.wind(cfg), **kw)
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    ctx.precond_apply(r)
    ctx.kkt_apply(r)
    b = ctx.build_rhs(synth.desired_state(cfg))
    _, info, _, _ = ctx.gmres_solve(b, tol=1e-6, restart=10 if kw.get("nonlinear") else 30, max_iters=12)
    torch.cuda.synchronize()
    print(cfg.name, kw, "its", info["iterations"], flush=True)
    return ctx


c1 = synth.CONFIGS["c1"]
ctx = run(c1)
ctx.gmres_solve_host(np.ascontiguousarray(ctx.build_rhs(synth.desired_state(c1)).cpu().numpy()), max_iters=5)
vd, f, g, v0 = synth.mms_inputs(synth.mms_config(4, 5))
Context.from_config(synth.mms_config(4, 5)).build_rhs_general(vd, f, g, v0)
os.environ["AAO_WAVE"], os.environ["AAO_WAVE_MIN"] = "1", "9"
run(synth.small_config("wave", 2, 8, 6))
run(synth.small_config("wave_o", 2, 8, 6, problem="oseen", lo=-1.0, hi=1.0, beta=1e-3, nu=0.05, index=3))
del os.environ["AAO_WAVE"], os.environ["AAO_WAVE_MIN"]
run(synth.small_config("s3d", 3, 4, 6, beta=1e-3, nu=1e-2, index=5))
run(synth.small_config("nl", 2, 8, 8, beta=1e-2, nu=1e-2), nonlinear=True, inner_eps=1e-2, inner_maxit=20)
run(synth.small_config("nl_o", 2, 4, 6, problem="oseen", lo=-1.0, hi=1.0, beta=1e-3, nu=0.05, index=3),
    nonlinear=True, inner_eps=1e-2, inner_maxit=20)
print("sanitize target done", flush=True)
