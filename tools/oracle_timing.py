"""the CPU oracle timed beside the GPU (context only, not a target).

Single core (scipy.sparse is single-threaded; BLAS pinned to 1 thread), on the GPU box's host.  Small
configs: full precond_apply and kkt_apply.  Large configs: the per-frequency block solves of
precond_apply timed at k in {0, 1, n_b/2, n_b-1} and extrapolated linearly to all n_b frequencies the
oracle processes (LABELLED extrapolated), kkt_apply in full where the vectors fit comfortably."""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

import synth  # noqa: E402
from oracle import kkt, precond  # noqa: E402
from oracle.problem import Problem  # noqa: E402

FULL = ["c1", "c2", "c2b", "c4_32"]
SAMPLED = ["c3", "c4_64", "c4_128", "c5"]
KKT_MAX_N = 2e8


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


with threadpool_limits(limits=1):
    for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else FULL + SAMPLED):
        cfg = synth.CONFIGS[name]
        prob = Problem(cfg, synth.wind(cfg))
        pc = precond.OraclePreconditioner(prob, cache_blocks=False)
        r = synth.probe_vector(cfg)
        out = {"config": name, "N": cfg.n_dofs, "cores": 1, "cpu": cpu_model()}
        if name in FULL:
            t0 = time.perf_counter()
            pc.apply(r)
            out["precond_s"] = time.perf_counter() - t0
            out["precond_kind"] = "measured"
        else:
            ks = sorted({0, 1, cfg.n_b // 2, cfg.n_b - 1})
            ts = []
            for k in ks:
                Vh, Ph = pc.forward(r, [k])
                t0 = time.perf_counter()
                pc.block(k, Vh[0, 0], Vh[0, 1], Ph[0, 0], Ph[0, 1])
                ts.append(time.perf_counter() - t0)
            out["block_s_sampled"] = dict(zip([int(k) for k in ks], ts))
            out["precond_s"] = float(np.mean(ts)) * cfg.n_b
            out["precond_kind"] = f"extrapolated from {len(ks)} frequency blocks x n_b = {cfg.n_b} (transforms excluded)"
        if cfg.n_dofs <= KKT_MAX_N:
            t0 = time.perf_counter()
            kkt.kkt_apply(prob, r)
            out["kkt_s"] = time.perf_counter() - t0
        print(json.dumps(out), flush=True)
