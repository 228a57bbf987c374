"""Block-sparse Yinyang on the tensor cores (group tiles; lk_tgy.cu +
k_assign_tgy in lk_tc.cu): d <= 32, k <= 4096 group-bound strategies run the
filter -> label-sorted worklist -> (row-tile pair x failing group tile) MMAs.

Same contract as every other path (tests/test_gpu_parity.py): the oracle's
labels at every iteration (near-tie exemption), centroids within 1e-5, the
same iteration count -- plus the pruning the path exists for: later
iterations evaluate far fewer than n*k distances.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from test_gpu_parity import centroid_ok, check_trajectory

pytestmark = pytest.mark.gpu


def lk():
    import paper_2010_06654_b200 as m
    return m


def blobs(n, d, k_true, seed, spread=40.0, sigma=1.5):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-spread, spread, size=(k_true, d))
    lab = rng.integers(0, k_true, size=n)
    return (centres[lab] + rng.normal(0, sigma, size=(n, d))).astype(np.float32)


@pytest.mark.parametrize("d,k", [(32, 600), (32, 128), (32, 1000), (8, 300), (16, 257), (24, 640)])
@pytest.mark.parametrize("strategy", ["yinyang", "elkan", "regroup"])
def test_group_tiles_match_oracle(oracle, d, k, strategy):
    n = 24000
    x = blobs(n, d, max(8, k // 3), seed=d * 7 + k)
    m = lk()
    init = m.make_init(m.RunContext(seed=k), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 12)
    res = m.run_pruner(x, k, strategy, init=init, t_max=12, kernel="tc")
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"d={d} k={k} {strategy}")
    assert res.converged == ref["converged"]
    assert len(res.iterations) == ref["iterations"]
    assert centroid_ok(res.centroids, ref["centroids"], x)


def test_group_tiles_prune(oracle):
    """Well-separated blobs: from iteration 3 on the group tiles evaluate a
    small fraction of the n*k distances, and the labels stay the oracle's."""
    n, d, k = 200000, 32, 512
    x = blobs(n, d, 128, seed=5, spread=60.0, sigma=1.0)
    m = lk()
    init = m.make_init(m.RunContext(seed=9), x, k, "random")
    res = m.run_pruner(x, k, "yinyang", init=init, t_max=10, kernel="tc")
    ref = oracle.run_lloyd(x, k, init, 10)
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], "prune")
    dist = [it.dist_comps for it in res.iterations]
    assert dist[0] == n * k
    late = dist[3:]
    assert late and max(late) < 0.5 * n * k, dist


def test_group_tiles_4096_centroids(oracle):
    """32 full group tiles (k = 4096, the cfg5 shape) on a cfg5 row sample."""
    from paper_2010_06654_b200 import datasets
    x = datasets.generate("cfg5", 60000)
    k = 4096
    m = lk()
    init = m.make_init(m.RunContext(seed=2005), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 5)
    res = m.run_pruner(x, k, "yinyang", init=init, t_max=5)
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], "cfg5 k=4096")
    assert centroid_ok(res.centroids, ref["centroids"], x)


def test_streaming_filter_partial_groups_ragged_rows(oracle):
    """The thread-per-row streaming filter (128-byte points and group tables)
    with 29 of 32 group slots in use and a row count that is not a multiple of
    the 128-row tile."""
    from paper_2010_06654_b200 import datasets
    x = datasets.generate("cfg5", 33333)
    k = 3700
    m = lk()
    init = m.make_init(m.RunContext(seed=77), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 6)
    res = m.run_pruner(x, k, "yinyang", init=init, t_max=6)
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], "k=3700 ragged")
    assert centroid_ok(res.centroids, ref["centroids"], x)
    assert len(res.iterations) == ref["iterations"]


OFF_CASE = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
from oracle import oracle
import paper_2010_06654_b200 as m
from test_gpu_parity import check_trajectory, centroid_ok
from test_gpu_tgy import blobs
x = blobs(20000, 32, 100, seed=3)
init = m.make_init(m.RunContext(seed=4), x, 300, "random")
ref = oracle.run_lloyd(x, 300, init, 8)
res = m.run_pruner(x, 300, "yinyang", init=init, t_max=8, kernel="tc")
check_trajectory(oracle, x, init, res.assign_history, ref["history"], "LK_TGY=0")
assert centroid_ok(res.centroids, ref["centroids"], x)
print("ok")
"""


def test_group_tiles_off_knob():
    """LK_TGY=0 (A/B knob) restores the full-rescan tensor-core Yinyang path."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tests = os.path.join(repo, "tests")
    env = dict(os.environ, LK_TGY="0")
    r = subprocess.run([sys.executable, "-c", OFF_CASE.format(repo=repo, tests=tests)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


TGY_CASE = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
from oracle import oracle
import paper_2010_06654_b200 as m
from paper_2010_06654_b200 import datasets
from test_gpu_parity import check_trajectory, centroid_ok
x = datasets.generate("cfg5", 40000)
k = 4096
init = m.make_init(m.RunContext(seed=31), x, k, "random")
ref = oracle.run_lloyd(x, k, init, 6)
res = m.run_pruner(x, k, "yinyang", init=init, t_max=6)
check_trajectory(oracle, x, init, res.assign_history, ref["history"], "group-tile variant")
assert centroid_ok(res.centroids, ref["centroids"], x)
assert len(res.iterations) == ref["iterations"]
print("ok")
"""


@pytest.mark.parametrize("env_set", [{"LK_TGY_FILTER": "0"}, {"LK_TGY_FILTER": "2"}, {"LK_TGY_FILTER": "3"},
                                     {"LK_TGY_STAGES": "3"}, {"LK_TGY_BUCKET": "1"}])
def test_group_tile_variants(env_set):
    """The group-tile path's A/B knobs -- the filter from global memory
    (LK_TGY_FILTER=0 / 3), the 8-lanes-per-row streaming filter (2), the
    three-stage streaming filter (LK_TGY_STAGES=3), the mask-bucket partition
    of the worklist before the label sort (LK_TGY_BUCKET=1) -- all land on the
    oracle's trajectory at the cfg5 shape (d = 32, k = 4096)."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tests = os.path.join(repo, "tests")
    env = dict(os.environ, **env_set)
    r = subprocess.run([sys.executable, "-c", TGY_CASE.format(repo=repo, tests=tests)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("d,kernel", [(2, "simt"), (16, "simt"), (32, "simt"), (40, "auto")])
def test_regroup_rebuilds_groups_and_matches_oracle(oracle, d, kernel):
    """Regroup (pruners.py:500-504): the device rebuilds the group map after
    every centroid update (regroup_pass, bounds.py:199-212) and remaps the
    bounds (bounds.py:215-228); labels stay the oracle's."""
    n, k = 20000, 240
    # (overlapping blobs: the first iterations move the centroids far enough
    # that the nearest-group-mean pass changes the map)
    x = blobs(n, d, 60, seed=d + 11, spread=30.0 if d <= 32 else 6.0, sigma=2.0)
    m = lk()
    init = m.make_init(m.RunContext(seed=d), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 12)
    ctx = m.RunContext(seed=1, debug_validate=True)
    res = m.run_pruner(x, k, "regroup", init=init, t_max=12, kernel=kernel, ctx=ctx)
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"regroup d={d}")
    assert centroid_ok(res.centroids, ref["centroids"], x)
    assert sum(res.extra["regrouped"]) > 0, res.extra["regrouped"]
    assert ctx.violations == [], ctx.violations[:5]
