"""Small runs of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

SIMT Lloyd / Hamerly / fused Yinyang (cfg2, d=2), Elkan's per-centroid bounds
and Regroup (cfg1, d=16), the tensor-core paths (cfg5 d=32: two-row-tile pass,
group-tile Yinyang; cfg3 d=128: K-chunked pass), the debug bound validator and
the GPU k-means++ D^2 updates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2010_06654_b200 as lk  # noqa: E402
from paper_2010_06654_b200 import datasets  # noqa: E402

for name, n, k, strategies in (("cfg2", 20000, 200, ("yinyang", "hamerly", "lloyd")),
                               ("cfg1", 8000, 64, ("yinyang", "elkan", "regroup")),
                               ("cfg5", 6000, 300, ("lloyd", "hamerly", "yinyang")),
                               ("cfg3", 3000, 200, ("lloyd", "yinyang"))):
    x = datasets.generate(name, n)
    init = lk.make_init(lk.RunContext(seed=1), x, k, "random")
    for s in strategies:
        ctx = lk.RunContext(seed=3, debug_validate=(s != "lloyd" and name == "cfg1"))
        r = lk.run_lloyd(x, k, init=init, t_max=5) if s == "lloyd" else \
            lk.run_pruner(x, k, s, init=init, t_max=5, ctx=ctx)
        assert not ctx.violations, ctx.violations[:3]
        print(name, s, len(r.iterations), [len(h) for h in r.assign_history][:1], flush=True)
c = lk.make_init(lk.RunContext(seed=2), datasets.generate("cfg1", 70000), 16)  # GPU k-means++
print("kmeanspp", c.shape)
