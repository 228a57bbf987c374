#!/usr/bin/env python
"""Copy one evidence run (gpurun_out/<dir>) into profiles/r02 and print the results table.

    python tools/r02_install.py gpurun_out/r02end
"""
import glob
import json
import os
import shutil
import subprocess
import sys

src = sys.argv[1]
dst = "profiles/r02"
names = ["bench_cfg5_yinyang.json", "bench_reference_cfg5.json", "pytest_gpu.log", "smoke.log",
         "launches_cfg5.csv", "fullsize_parity.jsonl"]
for f in names + [os.path.basename(p) for p in glob.glob(os.path.join(src, "b_*.json"))]:
    p = os.path.join(src, f)
    if os.path.exists(p) and os.path.getsize(p) > 0:
        shutil.copy(p, os.path.join(dst, f))
    else:
        print("missing", p)
t = subprocess.run([sys.executable, "tools/launch_table.py", os.path.join(dst, "launches_cfg5.csv")],
                   capture_output=True, text=True).stdout
open(os.path.join(dst, "launches_cfg5_table.txt"), "w").write(t)
rows = []
for p in sorted(glob.glob(os.path.join(dst, "b_*.json"))) + [os.path.join(dst, "bench_cfg5_yinyang.json")]:
    d = json.loads(open(p).read().strip().splitlines()[-1])
    r = d["roofline"]
    rows.append((d["config"]["workload"], d["strategy"].split(" ")[0], d["ms_per_step"], d["value"],
                 d["e2e"]["value"], r["kernel"], r["bound"], r["frac"]))
for w, s, ms, v, e, k, b, f in rows:
    print(f"| {w} | {s} | {ms:.4g} | {v:,.1f} | {e:,.1f} | {k} {b} {f:.2f} |")
for l in open(os.path.join(dst, "fullsize_parity.jsonl")):
    d = json.loads(l)
    print(d["commit"], d["config"], d["strategy"], d.get("check"), d.get("iterations"),
          d.get("rows_checked_total"), d.get("label_mismatches_non_tie"), d.get("centroids_within_1e-5"),
          sum(d.get("label_differences_per_iteration", [0])), d.get("centroids_bit_equal"))
