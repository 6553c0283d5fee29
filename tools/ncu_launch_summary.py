"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel count, total, share."""
import collections
import csv
import sys

UNIT = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}


def summarise(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * UNIT[r[ui]]
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / T:.1f}% | {v / cnt[k] / 1e3:.2f} |")
    out.append(f"\nTotal {sum(cnt.values())} launches, {T / 1e3:.0f} us of device time.")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
