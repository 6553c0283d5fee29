"""Per-frequency inner iteration counts of one Algorithm-2 application (which blocks hit the cap?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2405_18964_b200 import Context
for name in sys.argv[1].split(","):
    cfg = synth.CONFIGS[name]
    ctx = Context.from_config(cfg, synth.wind(cfg), nonlinear=True)
    b = ctx.build_rhs(synth.desired_state(cfg))
    ctx.precond_apply(b)
    torch.cuda.synchronize()
    print(name, ctx.last_inner_iterations(), flush=True)
    ctx.close()
