"""Profiling driver: a GMRES solve with a capped iteration count (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=40)
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
ctx = Context.from_config(cfg, synth.wind(cfg))
b = ctx.build_rhs(synth.desired_state(cfg))
x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=30, max_iters=a.iters)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=30, max_iters=a.iters)
e.record()
torch.cuda.synchronize()
print(f"{a.config}: {info['iterations']} its, {s.elapsed_time(e):.1f} ms, {s.elapsed_time(e) / info['iterations']:.3f} ms/it")
