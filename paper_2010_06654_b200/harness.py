"""Benchmark-harness integration: GPU runs as cells of the reference's sweep.

Reference: lloydkit bench.py -- load_dataset (:30-58), run_benchmark
(:249-297), summarize (:304-329), make_report (:343-349).  The same sweep
driver runs every (dataset, k, seed) cell through the GPU drop-in
(run_engine) and returns schema-v1 RunLogs (runlog.py), so a GPU log file and
a CPU log file written by lloydkit concatenate into one make_report input:
the labels carry the configuration, the dataset / k / seed identify the cell.

Beside the reference's text loader there is a binary one: ``.npy`` files load
without parsing (a cfg5-sized CSV -- 1.6e9 numbers -- is impractical to parse
in Python).
"""

from __future__ import annotations

import math

import numpy as np

from .core import ContractError, RunContext, as_points, make_init
from .engine import KnobConfig, run_engine
from .runlog import RunLog, runlog_from_result


def load_dataset(path: str) -> np.ndarray:
    """A dataset file as a float64 [n, d] matrix.

    ``.npy``: numpy's binary format (memory-mapped, then validated: 2-D,
    non-empty, finite).  Anything else: the reference's headerless text table
    (CSV or whitespace separated; errors name the 1-based row)."""
    if path.endswith(".npy"):
        arr = np.load(path, mmap_mode="r", allow_pickle=False)
        if arr.ndim != 2 or arr.shape[0] == 0 or arr.shape[1] == 0:
            raise ContractError(f"{path}: expected a non-empty 2-D array, got shape {arr.shape}")
        if not np.issubdtype(arr.dtype, np.number):
            raise ContractError(f"{path}: non-numeric dtype {arr.dtype}")
        out = np.asarray(arr, dtype=np.float64)
        bad = ~np.isfinite(out)
        if bad.any():
            row = int(np.nonzero(bad.any(axis=1))[0][0]) + 1
            raise ContractError(f"{path}: row {row}: non-finite value")
        return out
    rows: list[list[float]] = []
    width = -1
    with open(path, encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            parts = line.split(",") if "," in line else line.split()
            try:
                vals = [float(p) for p in parts]
            except ValueError as exc:
                raise ContractError(f"{path}: row {lineno}: {exc}") from None
            if width == -1:
                width = len(vals)
            elif len(vals) != width:
                raise ContractError(f"{path}: row {lineno}: expected {width} columns, got {len(vals)}")
            if not all(math.isfinite(v) for v in vals):
                raise ContractError(f"{path}: row {lineno}: non-finite value")
            rows.append(vals)
    if not rows:
        raise ContractError(f"{path}: empty dataset")
    return np.asarray(rows, dtype=np.float64)


def save_dataset(path: str, data) -> None:
    """Write a matrix in the binary loader's format (float32 when exact)."""
    x = np.asarray(data)
    if x.dtype == np.float64 and np.array_equal(x.astype(np.float32).astype(np.float64), x):
        x = x.astype(np.float32)
    np.save(path, np.ascontiguousarray(x), allow_pickle=False)


def run_benchmark(datasets, ks, configs, *, seeds=(0,), init_method: str = "kmeanspp",
                  validate: bool = False):
    """Every configuration on every (dataset, k, seed) cell, on the GPU.

    Same contract as the reference's sweep: plain Lloyd is always included
    (it anchors the speedups); a run raising ContractError is logged with its
    error and skipped in the aggregation; violations of the debug shadow check
    abort.  Tree index modes raise ContractError on the GPU and
    are therefore logged as failed cells.  Returns (logs, summary)."""
    if not datasets or not ks or not configs:
        raise ContractError("need at least one dataset, k, and configuration")
    all_configs = list(configs)
    if not any(c.label() == "lloyd" for c in all_configs):
        ref = configs[0]
        all_configs.insert(0, KnobConfig(t_max=ref.t_max, capacity=ref.capacity))
    logs: list[RunLog] = []
    lloyd_wall: dict[tuple, int] = {}
    violations: list = []
    for dataset_id, data in datasets:
        data = as_points(data)
        n, d = int(data.shape[0]), int(data.shape[1])
        for k in ks:
            for seed in seeds:
                init = make_init(RunContext(seed=seed), data, k, init_method)
                for config in all_configs:
                    config = KnobConfig(**{**config.__dict__, "seed": seed})
                    try:
                        ctx = RunContext(seed=seed, debug_validate=validate)
                        res = run_engine(data, k, config, init=init, ctx=ctx)
                        violations.extend(ctx.violations)
                        log = runlog_from_result(res, dataset_id=dataset_id, n=n, d=d, k=k,
                                                 config=config, init_seed=seed)
                    except ContractError as exc:
                        log = RunLog(run_id=f"{dataset_id}-k{k}-s{seed}-{config.label()}-failed",
                                     dataset_id=dataset_id, n=n, d=d, k=k,
                                     config=config.__dict__.copy(), init_seed=seed, error=str(exc))
                    logs.append(log)
                    if log.error is None and config.label() == "lloyd":
                        lloyd_wall[(dataset_id, k, seed)] = log.wall_nanos()
    if violations:
        raise AssertionError(f"{len(violations)} invariant violations: {violations[:3]}")
    return logs, summarize(logs, lloyd_wall)


def _cell(log: RunLog) -> tuple:
    return (log.dataset_id, log.k, log.init_seed)


def summarize(logs, lloyd_wall: dict | None = None) -> dict:
    """Per-label aggregates; speedups against Lloyd in the same cell."""
    if lloyd_wall is None:
        lloyd_wall = {_cell(g): g.wall_nanos() for g in logs if g.error is None and g.label == "lloyd"}
    summary: dict[str, dict] = {}
    by_label: dict[str, list] = {}
    for log in logs:
        by_label.setdefault(log.label, []).append(log)
    for label, group in by_label.items():
        ok = [g for g in group if g.error is None]
        speedups = [lloyd_wall[_cell(g)] / g.wall_nanos() for g in ok
                    if _cell(g) in lloyd_wall and g.wall_nanos() > 0]
        powers = [it["pruning_power"] for g in ok for it in g.iterations]
        summary[label] = {
            "runs": len(group),
            "failed": len(group) - len(ok),
            "mean_speedup": float(np.mean(speedups)) if speedups else float("nan"),
            "median_speedup": float(np.median(speedups)) if speedups else float("nan"),
            "mean_pruning_power": float(np.mean(powers)) if powers else 0.0,
            "mean_dist_comps": float(np.mean([g.totals["dist_comps"] for g in ok])) if ok else 0.0,
            "mean_data_accesses": float(np.mean([g.totals["data_accesses"] for g in ok])) if ok else 0.0,
            "mean_bound_accesses": float(np.mean([g.totals["bound_accesses"] for g in ok])) if ok else 0.0,
            "mean_footprint_bytes": float(np.mean([g.footprint_bytes_estimate for g in ok])) if ok else 0.0,
        }
    return summary


def make_report(logs) -> list[dict]:
    """Rows per label sorted by mean speedup, best first (bench.py:343-349)."""
    if not logs:
        raise ContractError("no run logs to report on")
    rows = [{"label": label, **stats} for label, stats in summarize(logs).items()]
    rows.sort(key=lambda r: (-(r["mean_speedup"] if r["mean_speedup"] == r["mean_speedup"]
                               else float("-inf")), r["label"]))
    return rows
