"""Run logs in the reference harness's JSONL wire format (schema v1), so GPU
runs sit next to CPU runs in lloydkit's run_benchmark / make_report
(reference: bench.py:129-203 -- RunLog, _check_totals, runlog_from_result,
write_runlogs).  One JSON object per line with exactly the reference's keys;
per-iteration counters come from the device (IterationStats, lloyd.py)."""

from __future__ import annotations

import json
import uuid
from dataclasses import dataclass, field

from .core import ContractError
from .engine import KnobConfig

SCHEMA_VERSION = 1
_SUMMED = ("wall_nanos", "dist_comps", "data_accesses", "bound_accesses", "bound_updates")


@dataclass
class RunLog:
    """One benchmark run, serializable as a single JSON line (bench.py:129-163)."""

    run_id: str
    dataset_id: str
    n: int
    d: int
    k: int
    config: dict
    init_seed: int
    iterations: list = field(default_factory=list)
    totals: dict = field(default_factory=dict)
    footprint_bytes_estimate: float = 0.0
    error: str | None = None
    schema_version: int = SCHEMA_VERSION

    @property
    def label(self) -> str:
        return KnobConfig(**self.config).label()

    def wall_nanos(self) -> int:
        return int(self.totals.get("wall_nanos", 0))

    def to_json(self) -> str:
        return json.dumps(self.__dict__)

    @classmethod
    def from_json(cls, line: str) -> "RunLog":
        obj = json.loads(line)
        if obj.get("schema_version") != SCHEMA_VERSION:
            raise ContractError(f"unknown run-log schema {obj.get('schema_version')!r}")
        out = cls(**obj)
        check_totals(out)
        return out


def check_totals(log: RunLog):
    """Totals equal the per-iteration sums; pruning power in [0, 1] (bench.py:169-178)."""
    if log.error is not None:
        return
    for key in _SUMMED:
        total = sum(int(it[key]) for it in log.iterations)
        if int(log.totals.get(key, -1)) != total:
            raise ContractError(f"{log.run_id}: totals[{key}] != per-iteration sum")
    for it in log.iterations:
        if not 0.0 <= it["pruning_power"] <= 1.0:
            raise ContractError(f"{log.run_id}: pruning power outside [0, 1]")


def runlog_from_result(result, *, dataset_id: str, n: int, d: int, k: int, config: KnobConfig,
                       init_seed: int) -> RunLog:
    """A RunResult of run_lloyd / run_pruner / run_engine as a RunLog (bench.py:181-203).
    The GPU path builds no tree, so the footprint estimate is 0."""
    iters = []
    for st in result.iterations:
        iters.append({
            "iter": st.index,
            "wall_nanos": int(st.assign_nanos + st.refine_nanos),
            "dist_comps": int(st.dist_comps),
            "data_accesses": int(st.data_accesses),
            "bound_accesses": int(st.bound_accesses),
            "bound_updates": int(st.bound_updates),
            "pruning_power": float(min(1.0, max(0.0, st.pruning_power(n, k)))),
            "sse": float(st.sse),
        })
    totals = {key: sum(int(it[key]) for it in iters) for key in _SUMMED}
    return RunLog(
        run_id=f"{dataset_id}-k{k}-s{init_seed}-{config.label()}-{uuid.uuid4().hex[:8]}",
        dataset_id=dataset_id, n=n, d=d, k=k, config=config.__dict__.copy(), init_seed=init_seed,
        iterations=iters, totals=totals, footprint_bytes_estimate=0.0,
    )


def write_runlogs(path: str, logs: list):
    with open(path, "w", encoding="utf-8") as fh:
        for log in logs:
            fh.write(log.to_json() + "\n")


def read_runlogs(path: str) -> list:
    with open(path, encoding="utf-8") as fh:
        return [RunLog.from_json(line) for line in fh if line.strip()]
