#!/usr/bin/env python
"""Per-iteration probe of one trajectory: device ms per iteration, per-class
ms and the work counters, one JSON line per iteration.

    python tools/probe.py cfg5 20 0 yinyang:simt:32 lloyd:tc:0
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.core import RunContext, init_random
    from paper_2010_06654_b200.device import DeviceLloyd
    from paper_2010_06654_b200.pruners import gpu_groups

    wl = sys.argv[1]
    T = int(sys.argv[2])
    n_rows = int(sys.argv[3]) or None
    specs = sys.argv[4:]  # strategy:kernel:groups
    cfg = datasets.CONFIGS[wl]
    t0 = time.time()
    x = datasets.generate(wl, n_rows)
    init = init_random(RunContext(seed=cfg.seed_init), x, cfg.k)
    n, d, k = x.shape[0], cfg.d, cfg.k
    print(json.dumps({"gen_s": time.time() - t0, "n": n}), flush=True)
    for spec in specs:
        strat, kern, groups = spec.split(":")
        g = int(groups) or gpu_groups(strat, n, k, d)
        print(json.dumps({"spec": spec, "groups": g}), flush=True)
        run(x, init, k, strat, kern, g, T, cfg)


def run(x, init, k, strat, kern, g, T, cfg):
    import torch

    from paper_2010_06654_b200.device import DeviceLloyd
    eng = DeviceLloyd(x, k, strat, T, kernel=kern, groups=g, group_seed=cfg.seed_init,
                      record_history=False)
    eng.set_centroids(init)
    eng.profile(True)
    st = torch.cuda.current_stream()
    names = {0: "assign", 1: "filter", 2: "recheck", 3: "refine", 4: "update", 5: "gscan",
             6: "gmerge", 7: "collect", 8: "cand", 9: "ovf", 10: "sort"}
    prev = {c: 0.0 for c in names}
    for t in range(1, T + 1):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        eng.step(t)
        b.record(st)
        torch.cuda.synchronize()
        cls = {}
        for c, nm in names.items():
            v = eng.profile_read(c)[0]
            if v - prev[c] > 1e-4:
                cls[nm] = round(v - prev[c], 3)
            prev[c] = v
        s = eng.stats[t - 1].to("cpu").numpy()
        print(json.dumps({"t": t, "ms": round(a.elapsed_time(b), 3), "cls": cls,
                          "changed": int(s[0]), "active": int(s[2]), "work": int(s[3]),
                          "dist": int(s[4]), "ywl": int(s[9]), "pairs": int(s[10]),
                          "flagged": int(s[1]), "cand": int(s[6]), "ovf": int(s[8])}),
              flush=True)
        if int(s[7]) == 0:
            break
    eng.close()


if __name__ == "__main__":
    main()
