"""GPU parity: the CUDA path (through the C ABI, via the drop-in entry points)
against the reference's own outputs (tests/golden/) and the pinned CPU oracle.

Contract (BASELINE.json north_star):
  * identical labels at every iteration, except rows whose fp64 top-two
    distance gap is within 1e-5 relative (LABEL_GAP_EXEMPT);
  * centroids within 1e-5 relative (CENTROID_RTOL, plus CENTROID_ATOL_FRAC of
    max|X| for coordinates near zero);
  * the same iteration count.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

LABEL_GAP_EXEMPT = 1e-5
CENTROID_RTOL = 1e-5
CENTROID_ATOL_FRAC = 1e-9
SSE_RTOL = 1e-9

RUN_CASES = [n for n in golden_names() if "history" in load_golden(n)]


def lk():
    import paper_2010_06654_b200 as m
    return m


def centroid_ok(got, ref, x):
    atol = CENTROID_ATOL_FRAC * float(np.max(np.abs(x)))
    return np.all(np.abs(got - ref) <= CENTROID_RTOL * np.abs(ref) + atol)


def oracle_centroid_path(oracle, x, init, history):
    """c_0 = init, c_t = refine_full(x, h_t, c_{t-1}) (lloyd.py:78-97)."""
    cs = [np.asarray(init, dtype=np.float64)]
    for h in history:
        cs.append(oracle.refine_full(x, h, cs[-1])[0])
    return cs


def check_trajectory(oracle, x, init, gpu_hist, ref_hist, what):
    """Per-iteration label equality with the near-tie exemption."""
    assert len(gpu_hist) == len(ref_hist), f"{what}: iteration count {len(gpu_hist)} vs {len(ref_hist)}"
    cs = None
    for t, (a, b) in enumerate(zip(gpu_hist, ref_hist)):
        bad = np.nonzero(np.asarray(a) != np.asarray(b))[0]
        if len(bad) == 0:
            continue
        if cs is None:
            cs = oracle_centroid_path(oracle, x, init, ref_hist)
        gap = oracle.relative_top2_gap(np.asarray(x, dtype=np.float64)[bad], cs[t])
        assert np.all(gap <= LABEL_GAP_EXEMPT), \
            f"{what}: iteration {t + 1}: {int(np.sum(gap > LABEL_GAP_EXEMPT))} non-tie label mismatches"


@pytest.mark.parametrize("strategy", ["lloyd", "hamerly", "yinyang", "elkan"])
@pytest.mark.parametrize("name", RUN_CASES)
def test_golden_runs(oracle, name, strategy):
    g = load_golden(name)
    m = lk()
    k, t_max = int(g["k"]), int(g["t_max"])
    if strategy == "lloyd":
        res = m.run_lloyd(g["data"], k, init=g["init"], t_max=t_max)
    else:
        res = m.run_pruner(g["data"], k, strategy, init=g["init"], t_max=t_max)
    ref_hist = list(g["history"].astype(np.int64))
    check_trajectory(oracle, g["data"], g["init"], res.assign_history, ref_hist, name)
    assert res.converged == bool(g["converged"])
    assert centroid_ok(res.centroids, g["centroids"], g["data"]), name
    assert [s.changed for s in res.iterations] == g["changed"].tolist()
    sse_ref = g["sse"]
    sse_got = np.array([s.sse for s in res.iterations])
    # relative to the SSE itself; the absolute floor is scale- and
    # translation-invariant (the data's centered energy)
    xd = np.asarray(g["data"], dtype=np.float64)
    scale = float(np.sum((xd - xd.mean(axis=0)) ** 2))
    assert np.all(np.abs(sse_got - sse_ref) <= SSE_RTOL * np.abs(sse_ref) + 1e-13 * scale)
    if strategy == "lloyd":
        n = g["data"].shape[0]
        assert [s.dist_comps for s in res.iterations] == [n * k] * len(res.iterations)


@pytest.mark.parametrize("offset,dtype", [(1e3, np.float32), (1e6, np.float64), (-5e4, np.float32)])
def test_sse_far_from_origin(oracle, offset, dtype):
    """SSE (core.py:172-179) of data far from the origin: the fixed-point sums
    are of x - m (m = middle of the data's range), so Q - |S|^2 / n does not
    cancel; the SSE matches the oracle's direct sum to 1e-9 relative."""
    rng = np.random.default_rng(11)
    k = 12
    centres = rng.uniform(-5.0, 5.0, size=(k, 6))
    lab = rng.integers(0, k, size=4000)
    x = (centres[lab] + rng.normal(scale=0.3, size=(4000, 6)) + offset).astype(dtype)
    m = lk()
    init = m.make_init(m.RunContext(seed=11), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 10)
    for s in ("lloyd", "yinyang"):
        res = m.run_lloyd(x, k, init=init, t_max=10) if s == "lloyd" else \
            m.run_pruner(x, k, s, init=init, t_max=10)
        check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"offset {s}")
        got = np.array([it.sse for it in res.iterations])
        assert np.all(got > 0)
        assert np.allclose(got, ref["sse"], rtol=1e-9, atol=0), (s, got, ref["sse"])
        assert centroid_ok(res.centroids, ref["centroids"], x)


def test_tie_break_prefers_lowest_index():
    g = load_golden("tie_break")
    res = lk().run_lloyd(g["data"], 3, init=g["init"], t_max=1)
    assert res.assign_history[0].tolist() == [0, 2]


def test_empty_cluster_keeps_previous_centroid():
    g = load_golden("empty_cluster")
    res = lk().run_lloyd(g["data"], 3, init=g["init"], t_max=3)
    assert np.array_equal(res.centroids[2], [99.0, 99.0])
    assert centroid_ok(res.centroids, g["centroids"], g["data"])


def test_strategies_are_bit_identical():
    """pruners.py:9-11: every strategy refines through the same kernel, so
    centroids are bit-equal to the Lloyd run (fixed-point sums make this hold
    on the GPU too)."""
    g = load_golden("pruners_blobs")
    m = lk()
    a = m.run_lloyd(g["data"], int(g["k"]), init=g["init"], t_max=8)
    for s in ("hamerly", "yinyang", "elkan", "regroup"):
        b = m.run_pruner(g["data"], int(g["k"]), s, init=g["init"], t_max=8)
        assert np.array_equal(a.centroids, b.centroids), s
        for u, v in zip(a.assign_history, b.assign_history):
            assert np.array_equal(u, v), s


@pytest.mark.parametrize("strategy", ["hamerly", "yinyang", "elkan"])
def test_bounded_strategies_prune_later_iterations(strategy):
    g = load_golden("pruners_blobs")
    k = int(g["k"])
    res = lk().run_pruner(g["data"], k, strategy, init=g["init"], t_max=8)
    n = g["data"].shape[0]
    assert res.iterations[0].dist_comps == n * k
    assert all(s.dist_comps <= n * k for s in res.iterations)
    assert min(s.dist_comps for s in res.iterations[1:]) < n * k


@pytest.mark.parametrize("k", [1, 2, 3])
def test_tiny_k(oracle, k):
    rng = np.random.default_rng(5)
    x = rng.uniform(size=(120, 4))
    m = lk()
    init = m.make_init(m.RunContext(seed=5), x, k)
    ref = oracle.run_lloyd(x, k, init, 8)
    for s in ("lloyd", "hamerly", "yinyang", "elkan"):
        res = m.run_lloyd(x, k, init=init, t_max=8) if s == "lloyd" else \
            m.run_pruner(x, k, s, init=init, t_max=8)
        check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"k={k} {s}")
        assert centroid_ok(res.centroids, ref["centroids"], x)


def test_n_equals_k(oracle):
    rng = np.random.default_rng(6)
    x = rng.normal(size=(7, 2))
    m = lk()
    init = m.make_init(m.RunContext(seed=6), x, 7)
    ref = oracle.run_lloyd(x, 7, init, 10)
    res = m.run_pruner(x, 7, "hamerly", init=init, t_max=10)
    assert centroid_ok(res.centroids, ref["centroids"], x)


def test_t_max_zero_returns_init():
    m = lk()
    x = np.random.default_rng(0).normal(size=(20, 3))
    init = x[:4].copy()
    res = m.run_lloyd(x, 4, init=init, t_max=0)
    assert res.iterations == [] and not res.converged
    assert np.array_equal(res.centroids, init)


def test_contract_errors():
    m = lk()
    with pytest.raises(m.ContractError):
        m.run_lloyd(np.ones(5), 2)
    with pytest.raises(m.ContractError):
        m.run_lloyd(np.array([[1.0, np.nan]]), 1)
    with pytest.raises(ValueError):
        m.run_lloyd(np.ones((5, 2)), 2, init=np.ones((3, 2)))
    with pytest.raises(m.ContractError):
        m.run_pruner(np.ones((5, 2)), 2, "warp")


# --- BASELINE configs at oracle-feasible sizes (same generators, prefixes) ----

SCALED = [("cfg1", 100_000, None, 50), ("cfg2", 100_000, None, 100), ("cfg3", 10_000, None, 15),
          ("cfg4", 5_000, None, 15), ("cfg5", 50_000, None, 3)]


@pytest.mark.parametrize("strategy", ["lloyd", "hamerly", "yinyang"])
@pytest.mark.parametrize("name,n,k,t_max", SCALED)
def test_scaled_configs_match_oracle(oracle, name, n, k, t_max, strategy):
    from paper_2010_06654_b200 import datasets
    cfg = datasets.CONFIGS[name]
    x = datasets.generate(name, n)
    k = k or cfg.k
    m = lk()
    init = m.make_init(m.RunContext(seed=cfg.seed_init), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, t_max)
    if strategy == "lloyd":
        res = m.run_lloyd(x, k, init=init, t_max=t_max)
    else:
        res = m.run_pruner(x, k, strategy, init=init, t_max=t_max)
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"{name} {strategy}")
    assert res.converged == ref["converged"]
    assert centroid_ok(res.centroids, ref["centroids"], x), name


@pytest.mark.parametrize("name,n,k,d_strat", [("cfg3", 6000, 300, "lloyd"), ("cfg4", 3000, 256, "hamerly"),
                                               ("cfg5", 20000, 1000, "hamerly")])
def test_tensor_core_and_simt_paths_agree(oracle, name, n, k, d_strat):
    """The tcgen05 3xTF32 path and the fp32 SIMT path certify labels
    independently; both must land on the oracle's trajectory, bit-identically."""
    from paper_2010_06654_b200 import datasets
    x = datasets.generate(name, n)
    m = lk()
    init = m.make_init(m.RunContext(seed=3), x, k, "random")
    runs = {}
    for kern in ("simt", "tc"):
        if d_strat == "lloyd":
            runs[kern] = m.run_lloyd(x, k, init=init, t_max=6, kernel=kern)
        else:
            runs[kern] = m.run_pruner(x, k, d_strat, init=init, t_max=6, kernel=kern)
    ref = oracle.run_lloyd(x, k, init, 6)
    for kern, res in runs.items():
        check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"{name} {kern}")
    assert np.array_equal(runs["simt"].centroids, runs["tc"].centroids)
    # the TC path must actually certify most rows itself
    assert sum(runs["tc"].extra["recheck_rows"]) < 0.05 * n * len(runs["tc"].iterations)


@pytest.mark.parametrize("strategy", ["lloyd", "hamerly", "yinyang"])
def test_k_above_int16(oracle, strategy):
    """Any 1 <= k <= n is accepted (core.py:186-187): k = 33 000 > 2^15."""
    rng = np.random.default_rng(12)
    x = rng.uniform(-1.0, 1.0, size=(36000, 3)).astype(np.float32)
    k = 33000
    m = lk()
    init = m.make_init(m.RunContext(seed=12), x, k, "random")
    ref = oracle.run_lloyd(x, k, init, 3)
    res = m.run_lloyd(x, k, init=init, t_max=3) if strategy == "lloyd" else \
        m.run_pruner(x, k, strategy, init=init, t_max=3)
    check_trajectory(oracle, x, init, res.assign_history, ref["history"], f"k=33000 {strategy}")
    assert centroid_ok(res.centroids, ref["centroids"], x)


def test_engine_full_profile_raises():
    """KnobConfig(bound_strategy="full") at index_mode="none" goes to
    run_pruner in the reference, which rejects the name (pruners.py:868-869)."""
    m = lk()
    with pytest.raises(m.ContractError):
        m.run_engine(np.ones((10, 2)), 2, m.KnobConfig(bound_strategy="full"), init=np.ones((2, 2)))
