"""Host-side phase timing of the public-API call (run_pruner) on a workload,
with the cached device context warm (what bench.py's e2e measures).

    python tools/e2e_phases.py [cfg2] [yinyang]
"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_06654_b200 as lk  # noqa: E402
from paper_2010_06654_b200 import datasets  # noqa: E402
from paper_2010_06654_b200.core import RunContext, init_random  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
strategy = sys.argv[2] if len(sys.argv) > 2 else "yinyang"
cfg = datasets.CONFIGS[wl]
x = datasets.generate(wl)
init = init_random(RunContext(seed=cfg.seed_init), x, cfg.k)
xp = torch.from_numpy(x).pin_memory()
T = 15


def call():
    return lk.run_pruner(xp, cfg.k, strategy, init=init, t_max=T)


call()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = call()
    torch.cuda.synchronize()
    print(f"call {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms, {len(res.iterations)} iterations, "
          f"device iteration ms {[round((s.assign_nanos + s.refine_nanos) / 1e6, 3) for s in res.iterations]}")
pr = cProfile.Profile()
pr.enable()
res = call()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
