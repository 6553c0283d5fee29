"""Capture the DRAM traffic of one velocity-MG launch (k_mg_cta<2|3, 2, ...>) with ncu and record it per
config for bench.py's roofline "traffic" (keyed by the CUDA source hash: a stale record is ignored).

usage (on the GPU box): python tools/ncu_traffic.py <config> [out.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

name = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"traffic_{name}.json")
cmd = ["ncu", "--clock-control", "none", "--print-units", "base", "--kernel-name", "regex:k_mg_cta", "--launch-skip", "1", "--launch-count",
       "1", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size",
       "--csv", "--page", "raw", sys.executable, os.path.join(ROOT, "tools", "ncu_target.py"), name, "1"]
res = subprocess.run(cmd, capture_output=True, text=True)
lines = [ln for ln in res.stdout.splitlines() if ln.startswith('"')]
rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
row = rows[-1]
def num(k):
    return float(str(row[k]).replace(",", ""))
rec = {"source_hash": bench.source_hash(), "kernel": row.get("Kernel Name"),
       "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
       "duration_ns": num("gpu__time_duration.sum"), "grid": row.get("launch__grid_size"),
       "capture": "ncu --clock-control none, 2nd k_mg_cta launch of one precond_apply (tools/ncu_traffic.py)"}
rec["dram_bytes_per_launch"] = rec["dram_read"] + rec["dram_write"]
units = {k: row.get(k) for k in row if k.startswith("dram") or k.startswith("gpu__time")}
print(json.dumps(rec), units)
json.dump({name: rec}, open(out, "w"), indent=1)
