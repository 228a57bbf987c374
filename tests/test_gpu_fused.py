"""GPU parity of the fused Yinyang kernel (lk_yy_fused.cu, d <= 32 and
t <= 32 groups) and its drift-offset ("lazy") bound encoding, across the
template instances it dispatches to (d in {2, 4, 8, 16, 32} padded, group
slots in {4, 8, 16, 32}), against the CPU oracle's Lloyd trajectory.

Reference semantics: Yinyang (pruners.py:387-497) returns Lloyd's labels at
every iteration (tests/test_pruners.py:38-49), so the oracle's run_lloyd
trajectory is the expected output for every grouping.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from test_gpu_parity import centroid_ok, check_trajectory

pytestmark = pytest.mark.gpu


def blobs(n, d, centers, sigma, seed, dup_frac=0.0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-20, 20, size=(centers, d))
    lab = rng.integers(0, centers, size=n)
    x = (c[lab] + rng.normal(0, sigma, size=(n, d))).astype(np.float32)
    if dup_frac:
        m = int(n * dup_frac)
        x[:m] = x[rng.integers(0, n, size=m)]  # exact duplicates: tie-heavy rows
    return x


def run_groups(x, k, init, t_max, groups):
    from paper_2010_06654_b200.device import DeviceLloyd
    eng = DeviceLloyd(x, k, "yinyang", t_max, groups=groups, group_seed=1)
    try:
        return eng.run(init)
    finally:
        eng.close()


@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 13, 16, 24, 32])
@pytest.mark.parametrize("groups", [4, 8, 16, 32])
def test_fused_dims_and_groups(oracle, d, groups):
    n, k, t_max = 6000, 96, 12
    x = blobs(n, d, 24, 1.5, seed=100 + d, dup_frac=0.05)
    rng = np.random.default_rng(7 + d)
    init = x[rng.choice(n, k, replace=False)].astype(np.float64)
    out = run_groups(x, k, init, t_max, groups)
    ref = oracle.run_lloyd(x, k, init, t_max)
    check_trajectory(oracle, x, init, out["history"], ref["history"], f"d={d} t={groups}")
    assert out["converged"] == ref["converged"]
    assert centroid_ok(out["centroids"], ref["centroids"], x)


def test_fused_more_groups_than_centroids(oracle):
    """k < t: empty group slots carry +inf bounds and are never scanned."""
    x = blobs(3000, 2, 5, 1.0, seed=5)
    init = x[:6].astype(np.float64)
    out = run_groups(x, 6, init, 10, 16)
    ref = oracle.run_lloyd(x, 6, init, 10)
    check_trajectory(oracle, x, init, out["history"], ref["history"], "k<t")


def test_fused_multi_chunk_queue(oracle):
    """Enough rows per block that the block-local queue fills and drains many
    times within one launch (several chunks per persistent block)."""
    x = blobs(400_000, 2, 300, 3.0, seed=11)
    k = 300
    init = x[np.random.default_rng(2).choice(len(x), k, replace=False)].astype(np.float64)
    out = run_groups(x, k, init, 6, 16)
    ref = oracle.run_lloyd(x, k, init, 6)
    check_trajectory(oracle, x, init, out["history"], ref["history"], "multi-chunk")
    assert centroid_ok(out["centroids"], ref["centroids"], x)


SMALL_QUEUE = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
from oracle import oracle
from test_gpu_fused import blobs, run_groups
from test_gpu_parity import check_trajectory
x = blobs(60_000, 2, 120, 2.0, seed=3)
k = 128
init = x[np.random.default_rng(4).choice(len(x), k, replace=False)].astype(np.float64)
out = run_groups(x, k, init, 8, 32)
ref = oracle.run_lloyd(x, k, init, 8)
check_trajectory(oracle, x, init, out["history"], ref["history"], "small queue")
print("ok")
"""


def test_fused_tiny_pair_buffer():
    """LK_YY_PCAP=256: a chunk's pairs overflow the block's pair buffer, so
    rows of one chunk are queued across several drains (the enqueue loop)."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tests = os.path.join(repo, "tests")
    env = dict(os.environ, LK_YY_PCAP="256")
    r = subprocess.run([sys.executable, "-c", SMALL_QUEUE.format(repo=repo, tests=tests)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


CENTER_CASE = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
from oracle import oracle
import paper_2010_06654_b200 as m
from paper_2010_06654_b200 import datasets
from test_gpu_parity import check_trajectory, centroid_ok
x = datasets.generate({name!r}, {n})
init = m.make_init(m.RunContext(seed=5), x, {k}, "random")
ref = oracle.run_lloyd(x, {k}, init, 6)
for strat in ("lloyd", "hamerly"):
    res = (m.run_lloyd(x, {k}, init=init, t_max=6, kernel="tc") if strat == "lloyd"
           else m.run_pruner(x, {k}, strat, init=init, t_max=6, kernel="tc"))
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], strat)
    assert centroid_ok(res.centroids, ref["centroids"], x)
print("ok")
"""


@pytest.mark.parametrize("name,n,k,center", [("cfg5", 30000, 600, "1"), ("cfg5", 30000, 600, "0"),
                                              ("cfg3", 8000, 300, "1"), ("cfg4", 3000, 256, "1")])
def test_tensor_core_tile_centering(name, n, k, center):
    """The centered tensor-core pass (label-sorted rows, tiles shifted by a
    centroid, bias rows from the k x k table) and the plain one, forced on and
    off by LK_TC_CENTER, both land on the oracle's trajectory."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tests = os.path.join(repo, "tests")
    env = dict(os.environ, LK_TC_CENTER=center)
    code = CENTER_CASE.format(repo=repo, tests=tests, name=name, n=n, k=k)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("env_set", [{"LK_TC2": "0"}, {"LK_TC2": "0", "LK_TC_CL": "2"},
                                     {"LK_TC2": "0", "LK_TC_CL": "4"}, {"LK_TC_FAST": "0", "LK_TC2": "0"},
                                     {"LK_TC_SPLIT": "0"}])
def test_tensor_core_d32_variants(env_set):
    """The d <= 32 tensor-core variants behind the A/B knobs -- the single-row-
    tile kernel (LK_TC2=0), its 2- and 4-CTA multicast clusters (LK_TC_CL), the
    per-column top-2 epilogue (LK_TC_FAST=0), one unordered accumulator
    (LK_TC_SPLIT=0) -- all land on the oracle's trajectory (an odd number of row
    tiles and k not a multiple of 128 exercise the dummy tiles and padding)."""
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    tests = os.path.join(repo, "tests")
    env = dict(os.environ, **env_set)
    code = CENTER_CASE.format(repo=repo, tests=tests, name="cfg5", n=20000, k=600)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("strategy", ["yinyang", "hamerly", "lloyd"])
def test_history_drained_mid_run(oracle, strategy):
    """A label-history log holding 2 iterations is drained and rewound mid-run
    (history_iters < t_max; a larger check_every is clamped to it): the
    rebuilt assign_history still equals the oracle's at every iteration."""
    from paper_2010_06654_b200.device import DeviceLloyd
    x = blobs(5000, 8, 20, 2.0, seed=21)
    k, t_max = 40, 9
    init = x[np.random.default_rng(3).choice(len(x), k, replace=False)].astype(np.float64)
    eng = DeviceLloyd(x, k, strategy, t_max, groups=8 if strategy == "yinyang" else 0,
                      history_iters=2)
    try:
        out = eng.run(init, check_every=5)
    finally:
        eng.close()
    ref = oracle.run_lloyd(x, k, init, t_max)
    check_trajectory(oracle, x, init, out["history"], ref["history"], f"drain {strategy}")
    assert out["converged"] == ref["converged"]


@pytest.mark.parametrize("d,k,groups", [(40, 300, 8), (48, 500, 16), (16, 2000, 40)])
def test_simt_multikernel_yinyang(oracle, d, k, groups):
    """The SIMT multi-kernel Yinyang path (k_filter_yinyang -> k_yy_pairs ->
    k_yy_merge with per-group scans), taken for d > 32 or more than 32 groups
    on kernel="simt": the oracle's trajectory."""
    from paper_2010_06654_b200.device import DeviceLloyd
    rng = np.random.default_rng(d + k)
    c = rng.uniform(-25, 25, size=(k // 4, d))
    x = (c[rng.integers(0, k // 4, 12000)] + rng.normal(0, 1.5, size=(12000, d))).astype(np.float32)
    m = __import__("paper_2010_06654_b200")
    init = m.make_init(m.RunContext(seed=d), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 8)
    eng = DeviceLloyd(x, k, "yinyang", 8, kernel="simt", groups=groups)
    try:
        assert not eng.group_cap == 128  # not the group-tile path
        out = eng.run(init)
        hist = out["history"]
        assert len(hist) == ref["iterations"]
        from test_gpu_parity import check_trajectory, centroid_ok
        check_trajectory(oracle, x, init, hist, ref["history"], f"simt yinyang d={d} t={groups}")
        assert centroid_ok(out["centroids"], ref["centroids"], x)
        # the group scans ran (not only full rescans)
        assert sum(r.group_dists for r in out["records"][1:]) > 0
    finally:
        eng.close()
