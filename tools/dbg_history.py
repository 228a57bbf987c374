import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from conftest import load_golden
from paper_2010_06654_b200.device import DeviceLloyd
g = load_golden("ac01_c0_s0")
x, init, k = g["data"], g["init"], int(g["k"])
for ug in (False, True):
    for ce in (1, 4):
        e = DeviceLloyd(x, k, "lloyd", 5)
        out = e.run(init, use_graphs=ug, check_every=ce)
        ok = [np.array_equal(a, b) for a, b in zip(out["history"], g["history"])]
        print("graphs", ug, "check_every", ce, "iters", out["iterations"], ok)
