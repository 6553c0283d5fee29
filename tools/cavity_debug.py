import sys; sys.path.insert(0, '.')
import numpy as np, synth
from oracle import manufactured, fem
from oracle.problem import Problem
from paper_2405_18964_b200 import Context
cfg = synth.cavity_config(8, 8)
w = synth.cavity_wind(cfg)
vd, f, g, v0 = synth.cavity_inputs(cfg)
for label, ww in (("zero wind", 0 * w), ("wind", w)):
    ctx = Context.from_config(cfg, ww)
    b = ctx.build_rhs_general(vd, f, g, v0).cpu().numpy()
    prob = Problem(cfg, ww)
    bo = manufactured.rhs_with_data(prob, vd, f, g, v0, wind=ww)
    d = (b - bo).reshape(2, cfg.n_b, -1)
    i = np.unravel_index(np.argmax(np.abs(d)), d.shape)
    print(label, np.linalg.norm(b - bo) / np.linalg.norm(bo), i, d[i], flush=True)
    if label == "wind":
        # candidate: the difference equals tau * (N - N^T) G or 2 tau N G on state rows?
        lv = fem.Level(2, cfg.n_cells, cfg.x_lo, cfg.x_hi)
        N = lv.conv_q2(ww)
        Iv = prob.fine.Iv
        bmask = np.ones(cfg.n_s, bool); bmask[Iv] = False
        G = np.where(bmask, g[1][0], 0.0)
        tau = cfg.T / cfg.n_t
        for nm, M in (("N", N), ("NT", N.T)):
            t = -tau * (M @ G)[Iv]
            print(nm, np.linalg.norm(d[1, 0, :cfg.n_s][Iv] - 0), np.linalg.norm(t), np.linalg.norm(d[1, 0, :cfg.n_s][Iv] + t), np.linalg.norm(d[1, 0, :cfg.n_s][Iv] - t))
