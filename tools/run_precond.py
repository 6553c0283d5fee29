"""Small driver for profiling: build a context for a config and run a few precond/kkt applications."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kkt", action="store_true")
ap.add_argument("--nt", type=int, default=0, help="override n_t (fewer frequencies, same mesh)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.nt:
    import dataclasses
    cfg = dataclasses.replace(cfg, n_t=a.nt)
ctx = Context.from_config(cfg, synth.wind(cfg))
r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
z = torch.empty_like(r)
for _ in range(a.reps):
    ctx.precond_apply(r, z)
    if a.kkt:
        ctx.kkt_apply(r, z)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    ctx.precond_apply(r, z)
e.record()
torch.cuda.synchronize()
print(f"{a.config}: precond {s.elapsed_time(e) / a.reps:.3f} ms, launches/apply {ctx.last_launch_count()}")
