"""The CPU oracle (oracle/lk_oracle.c) is pinned to the reference: every golden
fixture in tests/golden/ was produced by the reference itself
(tests/golden/make_golden.py), and the oracle must reproduce it bit for bit."""

import numpy as np
import pytest

from conftest import golden_names, load_golden

RUN_CASES = [n for n in golden_names() if "history" in load_golden(n)]


@pytest.mark.parametrize("name", RUN_CASES)
def test_oracle_reproduces_reference_run(oracle, name):
    g = load_golden(name)
    k, t_max = int(g["k"]), int(g["t_max"])
    out = oracle.run_lloyd(g["data"], k, g["init"], t_max, nthreads=2)
    assert out["iterations"] == len(g["history"])
    for t, (a, b) in enumerate(zip(out["history"], g["history"])):
        assert np.array_equal(a, b), f"{name}: labels differ at iteration {t + 1}"
    assert np.array_equal(out["centroids"], g["centroids"]), name
    assert np.array_equal(out["changed"], g["changed"]), name
    assert np.array_equal(out["sse"], g["sse"]), name
    assert out["converged"] == bool(g["converged"])


def test_tie_break_lowest_index(oracle):
    g = load_golden("tie_break")
    lab, d1, d2 = oracle.assign_full(g["data"], g["init"])
    assert lab.tolist() == g["labels"].tolist() == [0, 2]
    assert d1[0] == d2[0]  # an exact tie


def test_empty_cluster_keeps_previous(oracle):
    g = load_golden("empty_cluster")
    out, counts = oracle.refine_full(g["data"], np.array([0, 0, 1]), g["init"])
    assert np.array_equal(out, g["refined"])
    assert counts.tolist() == [2, 1, 0]


@pytest.mark.parametrize("d", [1, 2, 3, 7, 8, 9, 16, 31, 32, 33, 127, 128, 129, 200, 256, 300, 784])
def test_pairwise_distance_matches_numpy_order(oracle, d):
    """core.py:98-108: numpy's reduction order over d (checked against numpy here)."""
    rng = np.random.default_rng(d)
    x = rng.normal(size=(5, d)) * rng.uniform(0.1, 100, size=(5, d))
    c = rng.normal(size=(3, d)) * 10
    ref = np.sqrt(np.sum((x[:, None, :] - c[None, :, :]) ** 2, axis=2))
    assert np.array_equal(oracle.dist_matrix(x, c), ref)


def test_pairwise_sum_matches_numpy(oracle):
    rng = np.random.default_rng(7)
    for n in (1, 5, 8, 100, 129, 1000, 4099):
        a = rng.normal(size=n) * 1e3
        assert oracle.pairwise_sum(a) == np.sum(a)


def test_threads_do_not_change_results(oracle):
    g = load_golden("ac01_c9_s0")
    a = oracle.assign_full(g["data"], g["init"], nthreads=1)
    b = oracle.assign_full(g["data"], g["init"], nthreads=7)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("name", ["pruners_blobs", "pruners_dups", "pruners_uniform",
                                  "cfg1_small", "cfg2_small", "cfg5_small", "ac01_c8_s1"])
def test_oracle_hamerly_is_label_identical(oracle, name):
    """The CPU Hamerly port (bench baseline) reproduces the reference trajectory."""
    g = load_golden(name)
    k, t_max = int(g["k"]), int(g["t_max"])
    out = oracle.run_hamerly(g["data"], k, g["init"], t_max, nthreads=3)
    assert out["iterations"] == len(g["history"])
    for a, b in zip(out["history"], g["history"]):
        assert np.array_equal(a, b)
    assert np.array_equal(out["centroids"], g["centroids"])
    n = g["data"].shape[0]
    assert out["dist_comps"][0] == n * k
    if len(out["dist_comps"]) > 2:
        assert min(out["dist_comps"][1:]) < n * k
