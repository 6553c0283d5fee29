"""NEXT-3: Ritz values of P~^{-1} A at GPU scale (aao_arnoldi; the spectra of P:359-367 / Fig. 1).

For each config: m Arnoldi steps on A P^{-1} from a seeded probe vector, eigenvalues of H[:m, :m]; prints one
JSON line with the extreme Ritz values, the sorted real parts and the clustering of |mu| (Fig. 1(d) shows the
ordered real parts of the eigenvalues of P~_C^{-1} A at n_t = 10: two clusters, one positive and one negative,
bounded away from 0, with few outliers)."""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2nt10,c2,c3,c5")
ap.add_argument("--m", type=int, default=80)
a = ap.parse_args()
for name in a.configs.split(","):
    if name.endswith("nt10"):
        cfg = dataclasses.replace(synth.CONFIGS[name[:-4]], n_t=10, name=name)
    else:
        cfg = synth.CONFIGS[name]
    ctx = Context.from_config(cfg, synth.wind(cfg))
    v0 = torch.from_numpy(synth.probe_vector(cfg, seed_offset=7)).cuda()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    H = ctx.arnoldi(v0, a.m)
    e.record()
    torch.cuda.synchronize()
    k = H.shape[1]
    mu = np.linalg.eigvals(H[:k, :k])
    am = np.abs(mu)
    out = {"config": name, "N": cfg.n_dofs, "n_t": cfg.n_t, "steps": k, "arnoldi_s": s.elapsed_time(e) / 1e3,
           "re_min": float(mu.real.min()), "re_max": float(mu.real.max()),
           "abs_min": float(am.min()), "abs_max": float(am.max()), "im_abs_max": float(np.abs(mu.imag).max()),
           "n_re_pos": int((mu.real > 0).sum()), "n_re_neg": int((mu.real < 0).sum()),
           "abs_quantiles_10_50_90": [float(q) for q in np.quantile(am, [0.1, 0.5, 0.9])],
           "re_sorted": [round(float(v), 6) for v in np.sort(mu.real)]}
    print(json.dumps(out), flush=True)
    del ctx
    torch.cuda.empty_cache()
