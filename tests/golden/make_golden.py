"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
(/root/reference/pkg/src/lloydkit, imported read-only in the build container).

    python tests/golden/make_golden.py

The fixtures pin the CPU oracle (tests/test_oracle.py) and the GPU path
(tests/test_gpu_parity.py) to what the reference itself returns.  The
reference does not exist on the GPU box; only these .npz files travel.

Cases (all small, so the reference finishes in seconds):
  * lloyd_blobs_s{0,1,2}   tests/test_lloyd.py:38-49 data, k-means++ init, t_max 8
  * tie_break              tests/test_lloyd.py:52-57 ([0,0],[4,0] vs duplicate centres)
  * pruners_{blobs,uniform,dups}  tests/test_pruners.py:16-27 data, Lloyd + Hamerly /
                           Yinyang / Elkan histories (identical by construction)
  * ac01_c{i}_s{seed}      tests/test_acceptance.py:71-76 cells (gen_gaussian,
                           k-means++ init, T_MAX 5)
  * cfg{1..5}_small        prefixes of the BASELINE configs with random init
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from lloydkit.bench import gen_gaussian  # noqa: E402
from lloydkit.core import RunContext, make_init  # noqa: E402
from lloydkit.lloyd import assign_full, refine_full, run_lloyd  # noqa: E402
from lloydkit.pruners import run_pruner  # noqa: E402

from paper_2010_06654_b200 import datasets  # noqa: E402


def pack(res):
    return {
        "history": np.array(res.assign_history, dtype=np.int32),
        "centroids": res.centroids,
        "changed": np.array([s.changed for s in res.iterations], dtype=np.int64),
        "sse": np.array([s.sse for s in res.iterations]),
        "dist_comps": np.array([s.dist_comps for s in res.iterations], dtype=np.int64),
        "converged": np.array(res.converged),
    }


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def blobs(n=90, d=2, k=3, seed=0, spread=0.4):
    rng = np.random.default_rng(seed)
    centers = rng.uniform(size=(k, d)) * 10
    labels = rng.integers(0, k, size=n)
    return centers[labels] + rng.normal(0, spread, size=(n, d))


def pruner_data(kind, seed=0):
    rng = np.random.default_rng(seed)
    if kind == "blobs":
        centers = rng.uniform(size=(6, 3)) * 8
        labels = rng.integers(0, 6, size=150)
        return centers[labels] + rng.normal(0, 0.3, size=(150, 3))
    if kind == "uniform":
        return rng.uniform(size=(120, 4))
    base = rng.normal(size=(30, 2))
    return np.repeat(base, 4, axis=0)


def main():
    for seed in (0, 1, 2):
        data = blobs(seed=seed)
        init = make_init(RunContext(seed=seed), data, 3)
        res = run_lloyd(data, 3, init=init, t_max=8, ctx=RunContext(seed=seed))
        save(f"lloyd_blobs_s{seed}", data=data, init=init, k=3, t_max=8, **pack(res))

    data = np.array([[0.0, 0.0], [4.0, 0.0]])
    centers = np.array([[1.0, 0.0], [1.0, 0.0], [3.0, 0.0]])
    lab = assign_full(RunContext(seed=0), data, centers)
    res = run_lloyd(data, 3, init=centers, t_max=1, ctx=RunContext(seed=0))
    save("tie_break", data=data, init=centers, k=3, t_max=1, labels=lab, **pack(res))

    data = np.array([[0.0, 0.0], [1.0, 0.0], [10.0, 0.0]])
    centers = np.array([[0.5, 0.0], [10.0, 0.0], [99.0, 99.0]])
    res = run_lloyd(data, 3, init=centers, t_max=3, ctx=RunContext(seed=0))
    ref = refine_full(RunContext(seed=0), data, np.array([0, 0, 1]), centers)
    save("empty_cluster", data=data, init=centers, k=3, t_max=3, refined=ref, **pack(res))

    for kind in ("blobs", "uniform", "dups"):
        data = pruner_data(kind)
        k = 5 if kind != "dups" else 4
        init = make_init(RunContext(seed=0), data, k)
        out = {}
        ref = run_lloyd(data, k, init=init, t_max=8, ctx=RunContext(seed=0))
        out.update(pack(ref))
        for strat in ("hamerly", "yinyang", "elkan"):
            r = run_pruner(data, k, strat, init=init, t_max=8, ctx=RunContext(seed=0))
            assert all(np.array_equal(a, b) for a, b in zip(r.assign_history, ref.assign_history))
            out[f"dist_comps_{strat}"] = np.array([s.dist_comps for s in r.iterations])
        save(f"pruners_{kind}", data=data, init=init, k=k, t_max=8, **out)

    cells = [(200, 2, 2), (200, 2, 10), (200, 8, 10), (200, 8, 50), (200, 32, 2),
             (200, 32, 50), (2000, 2, 10), (2000, 8, 2), (2000, 8, 50), (2000, 32, 10)]
    for ci, (n, d, k) in enumerate(cells):
        for seed in (0, 1):
            data, _ = gen_gaussian(n, d, max(2, k // 2), 0.01, seed=17 * ci + seed)
            init = make_init(RunContext(seed=seed), data, k)
            res = run_lloyd(data, k, init=init, t_max=5, ctx=RunContext(seed=seed))
            save(f"ac01_c{ci}_s{seed}", data=data, init=init, k=k, t_max=5, **pack(res))

    small = {"cfg1": (4000, 50), "cfg2": (4000, 40), "cfg3": (3000, 12), "cfg4": (1500, 8),
             "cfg5": (6000, 6)}
    for name, (n, t_max) in small.items():
        cfg = datasets.CONFIGS[name]
        x = datasets.generate(name, n)
        k = min(cfg.k, n // 4)
        from lloydkit.core import init_random
        init = init_random(RunContext(seed=cfg.seed_init), x, k)
        res = run_lloyd(x, k, init=init, t_max=t_max, ctx=RunContext(seed=cfg.seed_init))
        save(f"{name}_small", data=x, init=init, k=k, t_max=t_max, **pack(res))
        print(name, "iters", len(res.iterations), "converged", res.converged)


if __name__ == "__main__":
    main()
