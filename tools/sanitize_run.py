"""Small runs of every kernel family, for compute-sanitizer (memcheck /
racecheck):  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

import paper_2010_06654_b200 as lk  # noqa: E402
from paper_2010_06654_b200 import datasets  # noqa: E402

for name, n, k, strategies in (("cfg2", 20000, 200, ("yinyang", "hamerly", "lloyd")),
                               ("cfg1", 8000, 64, ("yinyang", "elkan")),
                               ("cfg5", 6000, 300, ("lloyd", "hamerly", "yinyang")),
                               ("cfg3", 3000, 200, ("lloyd",))):
    x = datasets.generate(name, n)
    init = lk.make_init(lk.RunContext(seed=1), x, k, "random")
    for s in strategies:
        r = lk.run_lloyd(x, k, init=init, t_max=5) if s == "lloyd" else \
            lk.run_pruner(x, k, s, init=init, t_max=5)
        print(name, s, len(r.iterations), [len(h) for h in r.assign_history][:1])
c = lk.make_init(lk.RunContext(seed=2), datasets.generate("cfg1", 70000), 16)  # GPU k-means++
print("kmeanspp", c.shape)
