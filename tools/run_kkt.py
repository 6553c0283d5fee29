"""Time kkt_apply (and optionally the time transforms) on a config: CUDA events, warm, 16 B/DOF model."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", nargs="+", default=["c2"])
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
for name in a.config:
    cfg = synth.CONFIGS[name]
    ctx = Context.from_config(cfg, synth.wind(cfg))
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        ctx.kkt_apply(r, z)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        ctx.kkt_apply(r, z)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    print(f"{name}: N={ctx.N} kkt {ms:.4f} ms  {16 * ctx.N / ms / 1e6:.1f} GB/s (16 B/DOF)", flush=True)
    del ctx
    torch.cuda.empty_cache()
