"""Wall-clock split of one warm public-API call on cfg2 (bench.py's e2e):
input upload + validation, centroid upload / grouping, iterations, results."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_06654_b200 as lk  # noqa: E402
from paper_2010_06654_b200 import datasets, lloyd  # noqa: E402
from paper_2010_06654_b200.core import RunContext, init_random  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = datasets.CONFIGS[wl]
x = datasets.generate(wl)
init = init_random(RunContext(seed=cfg.seed_init), x, cfg.k)
xp = torch.from_numpy(x).pin_memory()
for _ in range(3):
    lk.run_pruner(xp, cfg.k, "yinyang", init=init, t_max=15)
torch.cuda.synchronize()
eng = lloyd._ENGINE_CACHE["engine"]
for rep in range(3):
    t0 = time.perf_counter()
    lk.run_pruner(xp, cfg.k, "yinyang", init=init, t_max=15)
    t1 = time.perf_counter()
    s = torch.cuda.synchronize
    a = time.perf_counter(); eng.rebind(xp); s(); b = time.perf_counter()
    eng.set_centroids(init); s(); c = time.perf_counter()
    out = eng.run(init); s(); d = time.perf_counter()
    print(f"call {1e3 * (t1 - t0):.2f} ms | rebind {1e3 * (b - a):.3f} set_centroids {1e3 * (c - b):.3f} "
          f"run {1e3 * (d - c):.3f} ms")
