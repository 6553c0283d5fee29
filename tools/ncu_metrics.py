"""Print the key metrics of every kernel in an ncu report (`ncu -i X --page raw --csv`)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
STALLS = ["long_scoreboard", "barrier", "short_scoreboard", "mio_throttle", "lg_throttle", "wait", "math_pipe_throttle",
          "not_selected", "no_instruction", "membar", "drain", "branch_resolving", "dispatch_stall", "tex_throttle"]


def main(path):
    if path.endswith(".csv"):   # already exported on the box (tools/ncu_full.sh)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(d["Kernel Name"][:100], "grid", d.get("Grid Size"), "block", d.get("Block Size"))
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]:>14s} {u[h.index(k)]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in d:
                st.append(f"{s}={float(d[k]):.2f}")
        print("   stalls/issue:", " ".join(st))


if __name__ == "__main__":
    main(sys.argv[1])
