#!/bin/bash
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_2405_18964_b200 import Context
os.environ["AAO_STORE_Z"] = "0"
for nocl in ("", "1"):
    if nocl: os.environ["AAO_NO_CTAB"] = "1"
    cfg = synth.mms_config(16, 32)
    ctx = Context.from_config(cfg, None)
    b = ctx.build_rhs_general(*synth.mms_inputs(cfg))
    x, info, hist, rc = ctx.gmres_solve(b, tol=1e-9, restart=30, max_iters=12000)
    h = np.array(hist)
    print("no_ctab" if nocl else "ctab", info["iterations"], info["converged"], info["final_relres"], info["true_relres"], h[::1000][:13])
PY
