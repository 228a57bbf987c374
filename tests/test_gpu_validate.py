"""Debug shadow validation of the device bounds (RunContext.debug_validate).

Reference: validate_bounds (bounds.py:280-328) at "iter{t}:decayed" and
"iter{t}:post" (pruners.py:896-902), violations as (label, where, kind,
worst overshoot) in ctx.violations; tests/test_bounds.py:181-202 checks that a
corrupted bound is reported.  Here the check runs on the device
(lk_validate_bounds) against exact fp64 distances.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

CASES = [n for n in golden_names() if "history" in load_golden(n)]


def lk():
    import paper_2010_06654_b200 as m
    return m


@pytest.mark.parametrize("strategy", ["hamerly", "yinyang", "elkan"])
@pytest.mark.parametrize("name", CASES)
def test_golden_runs_have_no_violations(name, strategy):
    g = load_golden(name)
    m = lk()
    ctx = m.RunContext(seed=1, debug_validate=True)
    res = m.run_pruner(g["data"], int(g["k"]), strategy, init=g["init"], t_max=int(g["t_max"]), ctx=ctx)
    assert ctx.violations == [], ctx.violations[:5]
    assert len(res.assign_history) == len(g["history"])


@pytest.mark.parametrize("strategy,d,k,kernel", [("hamerly", 8, 50, "simt"), ("yinyang", 16, 64, "simt"),
                                                 ("yinyang", 32, 300, "tc"), ("hamerly", 40, 60, "tc"),
                                                 ("yinyang", 40, 60, "tc")])
def test_validate_clean_on_every_path(strategy, d, k, kernel):
    rng = np.random.default_rng(d + k)
    x = (rng.uniform(-20, 20, size=(k // 3, d))[rng.integers(0, k // 3, 6000)]
         + rng.normal(size=(6000, d))).astype(np.float32)
    m = lk()
    ctx = m.RunContext(seed=2, debug_validate=True)
    init = m.make_init(m.RunContext(seed=3), x, k, "random")
    m.run_pruner(x, k, strategy, init=init, t_max=8, ctx=ctx, kernel=kernel)
    assert ctx.violations == [], ctx.violations[:5]


@pytest.mark.parametrize("strategy,kernel", [("hamerly", "simt"), ("yinyang", "simt"), ("yinyang", "tc")])
def test_corrupted_bounds_are_reported(strategy, kernel):
    """An upper bound below the true distance and group / global lower bounds
    above it are each reported with their kind."""
    import torch
    from paper_2010_06654_b200.device import DeviceLloyd
    rng = np.random.default_rng(5)
    x = rng.normal(size=(4000, 32)).astype(np.float32)
    k = 200
    init = x[rng.choice(4000, k, replace=False)].astype(np.float64)
    eng = DeviceLloyd(x, k, strategy, 6, kernel=kernel, groups=8)
    try:
        eng.set_centroids(init)
        eng.step(1)
        eng.step(2)
        assert eng.validate(True) == {}
        eng.ub[17] = -1e9
        bad = eng.validate(True)
        assert "ub" in bad and bad["ub"] > 1e8
        eng.ub[17] = 1e9  # (ub too large is valid)
        eng.lb.view(-1)[:] = 1e9
        bad = eng.validate(True)
        if strategy == "hamerly":
            assert "lb_global" in bad
        else:
            assert any(k_.startswith("lb_group[") for k_ in bad), bad
        torch.cuda.synchronize()
    finally:
        eng.close()
