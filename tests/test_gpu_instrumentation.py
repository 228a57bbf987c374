"""Per-iteration timing under CUDA-graph replay (IterationStats.assign_nanos /
refine_nanos, lloyd.py:113-118 in the reference): the library stamps the
device clock at every update's start and end (LK_BUF_TSTAMP), so the
assign / refine split survives graph replay."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["lloyd", "hamerly", "yinyang"])
def test_assign_refine_split_under_graphs(strategy):
    import paper_2010_06654_b200 as m
    from paper_2010_06654_b200 import datasets
    x = datasets.generate("cfg1", 60000)
    init = m.make_init(m.RunContext(seed=2001), x, 100, "random")
    res = (m.run_lloyd(x, 100, init=init, t_max=12) if strategy == "lloyd"
           else m.run_pruner(x, 100, strategy, init=init, t_max=12))
    a = np.array([s.assign_nanos for s in res.iterations], dtype=np.float64)
    r = np.array([s.refine_nanos for s in res.iterations], dtype=np.float64)
    assert np.all(a > 0) and np.all(r > 0), (a, r)
    # the refinement of k = 100 centroids is a small share of an iteration
    assert np.median(r) < np.median(a) + 1e6, (a, r)
