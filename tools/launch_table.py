"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_table.py gpurun_out/launches.csv [title]
"""
import csv
import sys
from collections import defaultdict


def table(path):
    rows = list(csv.reader(open(path)))
    i = [j for j, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[i]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        if len(r) < len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[h.index("Metric Value")].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(
            r[h.index("Metric Unit")], 1)
        name = r[h.index("Kernel Name")].split("(")[0][:64]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"{'kernel':66s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:66s} {v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:9.2f} {v[1] / tot:6.1%}")
    return "\n".join(out)


if __name__ == "__main__":
    print(table(sys.argv[1]))
