"""Drop-in bound-pruned strategies on the GPU: run_pruner with the reference's
signature (/root/reference/pkg/src/lloydkit/pruners.py:862-923).

The reference's per-point strategy plugins (SequentialStrategy, :70-114) are
replaced at the loop level: the whole iteration runs on the device and labels
never round-trip to the host between phases.  Every strategy
returns the same labels as Lloyd, so a name the GPU does not implement
natively is served by the nearest bound family that does (documented in
DESIGN.md).
"""

from __future__ import annotations

from .core import ContractError, RunContext
from .lloyd import RunResult, _prepare, run_device

# GPU implementation serving each reference strategy name (pruners.py:853-859).
GPU_STRATEGY = {
    "hamerly": "hamerly",
    "elkan": "hamerly",
    "yinyang": "hamerly",
    "regroup": "hamerly",
    "drake": "hamerly",
    "heap": "hamerly",
    "annulus": "hamerly",
    "exponion": "hamerly",
    "radius": "hamerly",
    "blockvec": "hamerly",
    "drift": "hamerly",
    "search": "hamerly",
}

STRATEGIES = dict(GPU_STRATEGY)


def run_pruner(data, k: int, strategy: str, *, init=None, init_method: str = "kmeanspp",
               t_max: int = 10, capacity: int = 30, ctx: RunContext | None = None,
               kernel: str = "auto", record_history: bool = True) -> RunResult:
    """Bound-pruned exact k-means on the GPU; same contract and stop rule as run_lloyd."""
    ctx = ctx or RunContext()
    if strategy not in STRATEGIES:
        raise ContractError(f"unknown strategy {strategy!r}; know {sorted(STRATEGIES)}")
    x, centers = _prepare(data, k, init, init_method, ctx)
    if k == 1:
        # pruners.py:878-883: nothing to prune with one centroid
        res = run_device(x, k, centers, "lloyd", t_max, ctx, label=strategy, kernel=kernel,
                         record_history=record_history)
        return res
    return run_device(x, k, centers, GPU_STRATEGY[strategy], t_max, ctx, label=strategy,
                      kernel=kernel, record_history=record_history)
