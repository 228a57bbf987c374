"""Top SASS instructions of one kernel in an ncu report by executed count and stall samples.

    python tools/sass_hot.py report.ncu-rep kernel_regex [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[0] == "Address":
        break
    try:
        data.append((int(r[ie] or 0), int(r[st] or 0), r[0], r[1]))
    except ValueError:
        pass
tot_i = sum(d[0] for d in data) or 1
tot_s = sum(d[1] for d in data) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
print("-- by stall samples")
for d in sorted(data, key=lambda x: -x[1])[:top]:
    print(f"{d[1] / tot_s:6.1%} {d[0]:10d} {d[2]} {d[3][:90]}")
print("-- by executed")
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{d[0] / tot_i:6.1%} {d[1]:8d} {d[2]} {d[3][:90]}")
