#!/bin/bash
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2405_18964_b200 import Context
cfg = synth.CONFIGS["c5"]
for fc in (0, 16, 12, 8):
    ctx = Context.from_config(cfg, synth.wind(cfg), freq_chunk=fc)
    r = torch.from_numpy(synth.probe_vector(cfg)).cuda(); z = torch.empty_like(r)
    ctx.precond_apply(r, z); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): ctx.precond_apply(r, z)
    e1.record(); torch.cuda.synchronize()
    print("c5 freq_chunk", fc, "precond ms", e0.elapsed_time(e1) / 3, flush=True)
    ctx.close(); del ctx, r, z; torch.cuda.empty_cache()
PY
