#!/usr/bin/env python
"""Full-size parity of the GPU path against the CPU oracle (BASELINE sizes).

    python tools/fullsize_parity.py cfg5 --strategies lloyd,hamerly,yinyang \
        --rows 1000000 --out profiles/r02/fullsize_parity.jsonl [--tc-vs-simt]

The oracle cannot replay cfg3-cfg5 end to end (hours), so every GPU iteration
is checked on its own, which by induction checks the whole trajectory:

  * labels of iteration t: the oracle (assign_full, lloyd.py:69-75, fp64,
    numpy's pairwise order) re-decides rows from the oracle centroids of
    iteration t-1; ALL rows at iterations 1, the middle one and the last (with
    --all-rows-at), a random sample of --rows rows at the others; a mismatch
    must be a near-tie (fp64 top-2 gap <= 1e-5 relative);
  * centroids of iteration t: refine_full (lloyd.py:78-97, row-order fp64) of
    the GPU's label vector of iteration t from the oracle centroids of t-1; the
    GPU's final centroids must match within 1e-5 relative;
  * iteration count / stop rule: changed counts equal the label-vector
    differences, a converged run's last two vectors are equal;
  * --tc-vs-simt: the same run on the tensor cores and on the fp32 SIMT path
    (both certify labels independently): every label of every iteration equal.

One JSON line per (config, strategy[, kernel]) is appended to --out, stamped
with the git commit of the tree it ran.
"""

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def git_head() -> str:
    if os.environ.get("LK_COMMIT"):  # (the GPU box gets the tree without .git)
        return os.environ["LK_COMMIT"]
    try:
        return subprocess.run(["git", "-C", REPO, "rev-parse", "--short", "HEAD"], capture_output=True,
                              text=True).stdout.strip() or "unknown"
    except OSError:
        return "unknown"


def gpu_run(x32, k, init, strategy, t_max, kernel):
    import paper_2010_06654_b200 as lk
    if strategy == "lloyd":
        return lk.run_lloyd(x32, k, init=init, t_max=t_max, kernel=kernel)
    return lk.run_pruner(x32, k, strategy, init=init, t_max=t_max, kernel=kernel)


def check(oracle, x64, init, res, rows_per_iter, all_at, seed, gap_exempt=1e-5):
    """Per-iteration oracle re-decision of the GPU labels (see module doc)."""
    n = x64.shape[0]
    hist = res.assign_history
    T = len(hist)
    rng = np.random.default_rng(seed)
    c_prev = np.asarray(init, dtype=np.float64)
    prev = np.full(n, -1, dtype=np.int64)
    per = []
    bad_total = 0
    exempt_total = 0
    checked_total = 0
    for t in range(T):
        t0 = time.time()
        h = np.asarray(hist[t])
        full = (t + 1) in all_at or rows_per_iter >= n
        if full:
            lab, d1, d2 = oracle.assign_full(x64, c_prev)
            mism = np.nonzero(lab != h)[0]
            nchk = n
        else:
            rows = np.sort(rng.choice(n, size=rows_per_iter, replace=False))
            lab, d1, d2 = oracle.assign_full(x64[rows], c_prev)
            sel = np.nonzero(lab != h[rows])[0]
            mism = rows[sel]
            d1, d2 = d1[sel], d2[sel]
            nchk = rows_per_iter
        if full:
            d1, d2 = d1[mism], d2[mism]
        with np.errstate(invalid="ignore", divide="ignore"):
            gap = (d2 - d1) / np.where(d2 > 0, d2, 1.0)
        gap[~np.isfinite(d2)] = np.inf
        n_bad = int(np.sum(gap > gap_exempt))
        n_ex = int(len(mism) - n_bad)
        changed = int(np.count_nonzero(h != prev))
        if changed != res.iterations[t].changed:
            raise AssertionError(f"t={t + 1}: changed {res.iterations[t].changed} vs label diff {changed}")
        c_next, _ = oracle.refine_full(x64, h, c_prev)
        per.append({"t": t + 1, "rows_checked": int(nchk), "all_rows": bool(full),
                    "non_tie_mismatch": n_bad, "tie_exempt": n_ex, "changed": changed,
                    "s": round(time.time() - t0, 2)})
        bad_total += n_bad
        exempt_total += n_ex
        checked_total += nchk
        c_prev, prev = c_next, h
    err = np.abs(res.centroids - c_prev)
    tol = 1e-5 * np.abs(c_prev) + 1e-9 * float(np.abs(x64).max())
    out = {"iterations": T, "converged": bool(res.converged),
           "label_mismatches_non_tie": bad_total, "label_tie_exempt": exempt_total,
           "rows_checked_total": int(checked_total),
           "max_centroid_rel_err": float(np.max(err / np.maximum(np.abs(c_prev), 1e-30))),
           "centroids_within_1e-5": bool(np.all(err <= tol)),
           "per_iteration": per}
    if res.converged and T >= 2:
        out["stop_rule_ok"] = bool(np.array_equal(np.asarray(hist[-1]), np.asarray(hist[-2])))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--strategies", default="lloyd,hamerly,yinyang")
    ap.add_argument("--rows", type=int, default=250000, help="sampled rows per iteration")
    ap.add_argument("--t-max", type=int, default=0)
    ap.add_argument("--all-rows-at", default="first,middle,last")
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--tc-vs-simt", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    from oracle import oracle
    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.core import RunContext, init_random

    cfg = datasets.CONFIGS[args.workload]
    t_max = args.t_max or cfg.t_max
    t0 = time.time()
    x32 = datasets.generate(args.workload)
    init = init_random(RunContext(seed=cfg.seed_init), x32, cfg.k)
    gen_s = time.time() - t0
    x64 = None
    head = git_head()
    for strategy in args.strategies.split(","):
        t1 = time.time()
        res = gpu_run(x32, cfg.k, init, strategy, t_max, args.kernel)
        gpu_s = time.time() - t1
        if args.tc_vs_simt:
            res2 = gpu_run(x32, cfg.k, init, strategy, t_max, "simt")
            T = len(res.assign_history)
            same_T = T == len(res2.assign_history)
            diff = [int(np.count_nonzero(np.asarray(res.assign_history[t]) != np.asarray(res2.assign_history[t])))
                    for t in range(min(T, len(res2.assign_history)))]
            line = {"commit": head, "config": args.workload, "strategy": strategy,
                    "check": "tc_vs_simt_all_labels_all_iterations", "n": cfg.n, "k": cfg.k,
                    "d": cfg.d, "iterations": [T, len(res2.assign_history)],
                    "label_differences_per_iteration": diff,
                    "centroids_bit_equal": bool(np.array_equal(res.centroids, res2.centroids)),
                    "ok": bool(same_T and not any(diff))}
        else:
            if x64 is None:
                x64 = x32.astype(np.float64)
            T = len(res.assign_history)
            marks = {"first": 1, "middle": max(1, (T + 1) // 2), "last": T}
            all_at = {marks[m] for m in args.all_rows_at.split(",") if m in marks}
            t2 = time.time()
            rep = check(oracle, x64, init, res, min(args.rows, cfg.n), all_at, cfg.seed_data + 77)
            line = {"commit": head, "config": args.workload, "strategy": strategy,
                    "kernel": args.kernel, "check": "oracle_per_iteration", "n": cfg.n, "d": cfg.d,
                    "k": cfg.k, "t_max": t_max, "gen_s": round(gen_s, 1),
                    "gpu_call_s": round(gpu_s, 2), "oracle_s": round(time.time() - t2, 1),
                    "oracle_threads": oracle.default_threads(), **rep,
                    "ok": rep["label_mismatches_non_tie"] == 0 and rep["centroids_within_1e-5"]}
        print(json.dumps(line), flush=True)
        if args.out:
            os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
            with open(args.out, "a") as f:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
