"""Per-phase device times of one GMRES(30) restart cycle (aao_set_timing): precond, kkt, orthogonalisation.

usage: python tools/gmres_phase.py [config] [iterations]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_512"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = synth.CONFIGS[name]
ctx = Context.from_config(cfg, synth.wind(cfg))
b = ctx.build_rhs(synth.desired_state(cfg))
x = torch.zeros_like(b)
ctx.gmres_solve(b, x, tol=1e-6, restart=30, max_iters=its)
ctx.set_timing(True)
x.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_, info, hist, rc = ctx.gmres_solve(b, x, tol=1e-6, restart=30, max_iters=its)
e1.record()
torch.cuda.synchronize()
out = {"config": name, "iterations": info["iterations"], "total_ms": e0.elapsed_time(e1)}
out.update({k: v for k, v in info.items() if k.startswith("ms_")})
print(json.dumps(out))
