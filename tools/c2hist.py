"""History drift of the c2 GMRES(30) solve: GPU vs oracle golden, and GPU vs GPU under a different
summation order (argv[1] = path of a saved history to compare against, optional)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth
from paper_2405_18964_b200 import Context
name = os.environ.get("CASE", "c2")
ref = json.load(open(f"tests/golden/gmres_{name}.json"))
cfg = synth.CONFIGS[name]
ctx = Context.from_config(cfg)
b = ctx.build_rhs(synth.desired_state(cfg))
x, info, hist, rc = ctx.gmres_solve(b, tol=1e-6, restart=30)
h = np.array(hist)
def drift(a, r, tag):
    n = min(len(a), len(r))
    d = np.abs(a[:n] - r[:n]) / r[:n]
    print(tag, "max rel", f"{d.max():.2e}", "at", int(d.argmax()), "per 30-cycle max:",
          [float(f"{d[i:i+30].max():.1e}") for i in range(0, n, 30)])
print(name, "its", info["iterations"], ref["iterations"], "true", info["true_relres"], ref["true_relres"][-1])
drift(h, np.array(ref["hist"]), "gpu-vs-oracle")
out = sys.argv[1] if len(sys.argv) > 1 else None
if out and os.path.exists(out):
    drift(h, np.load(out), "gpu-vs-gpu(other order)")
elif out:
    np.save(out, h)
