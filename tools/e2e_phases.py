"""Host-side phase timing of one public-API call (run_pruner) on cfg2."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2010_06654_b200 as lk
from paper_2010_06654_b200 import datasets, device as dv
from paper_2010_06654_b200.pruners import gpu_groups

x = datasets.generate("cfg2")
init = datasets.initial_centroids("cfg2", x)
xp = torch.from_numpy(x).pin_memory()
k = 1000
for rep in range(3):
    torch.cuda.synchronize()
    T = {}
    t0 = time.perf_counter()
    eng = dv.DeviceLloyd(xp, k, "yinyang", 15, groups=gpu_groups("yinyang", len(x), k), group_seed=0)
    torch.cuda.synchronize(); T["ctor(alloc,ctx,H2D,scan,quant)"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    out = eng.run(init)
    torch.cuda.synchronize(); T["run"] = time.perf_counter() - t1
    t2 = time.perf_counter()
    h = [np.asarray(a) for a in out["history"]]
    T["history materialize"] = time.perf_counter() - t2
    eng.close()
    T["total"] = time.perf_counter() - t0
    print(rep, {a: round(b * 1e3, 2) for a, b in T.items()}, "iters", out["iterations"])
# inside run(): profile with cProfile once
import cProfile, pstats
eng = dv.DeviceLloyd(xp, k, "yinyang", 15, groups=8, group_seed=0)
pr = cProfile.Profile(); pr.enable(); out = eng.run(init); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
