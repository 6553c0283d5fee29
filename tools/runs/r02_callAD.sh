#!/bin/bash
python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2405_18964_b200 import Context
ref = json.load(open("tests/golden/gmres_nl_c3.json"))
cfg = synth.Config(**ref["config"])
ctx = Context.from_config(cfg, synth.wind(cfg), nonlinear=True, inner_eps=1e-2, inner_maxit=60)
b = ctx.build_rhs(synth.desired_state(cfg))
r0 = b / torch.linalg.norm(b)
ctx.precond_apply(r0)
g = ctx.last_inner_iterations()
o = ref["inner_per_apply"][0]
print("first apply diffs:", [(k, g[k], o[k]) for k in range(len(o)) if g[k] != o[k]])
x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=10, max_iters=500)
print("gpu its", info["iterations"], "oracle", ref["iterations"])
n = min(len(hist), len(ref["hist"]))
h, hr = np.array(hist[:n]), np.array(ref["hist"][:n])
print("rel dev per iteration:", np.abs(h - hr) / hr)
PY
