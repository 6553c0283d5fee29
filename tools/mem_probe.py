"""Device memory plan probe: total/free HBM, context workspace per config, and isolated apply times.

usage: python tools/mem_probe.py [config ...]   (default c4_512)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2405_18964_b200 import Context  # noqa: E402


def main(names):
    free, total = torch.cuda.mem_get_info()
    print(json.dumps({"device": torch.cuda.get_device_name(0), "free_gb": free / 1e9, "total_gb": total / 1e9}),
          flush=True)
    for name in names:
        cfg = synth.CONFIGS[name]
        ctx = Context.from_config(cfg, synth.wind(cfg))
        r = torch.from_numpy(synth.probe_vector(cfg)).cuda()
        z = torch.empty_like(r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = {"config": name, "N": ctx.N, "vector_gb": 8 * ctx.N / 1e9, "ctx_gb": ctx.device_bytes() / 1e9}
        for what, fn in (("precond", ctx.precond_apply), ("kkt", ctx.kkt_apply)):
            fn(r, z)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(3):
                fn(r, z)
            e1.record()
            torch.cuda.synchronize()
            out[what + "_ms"] = e0.elapsed_time(e1) / 3
        ctx.set_timing(True)
        ctx.precond_apply(r, z)
        out["phase_ms"] = ctx.phase_ms()
        free, _ = torch.cuda.mem_get_info()
        out["free_after_gb"] = free / 1e9
        print(json.dumps(out), flush=True)
        ctx.close()
        del r, z, ctx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c4_512"])
