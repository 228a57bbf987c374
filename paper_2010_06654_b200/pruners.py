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
# The four bound families on the hot path run natively; the
# reference's other names are per-point CPU variants outside the hot path and
# are served by the GPU Yinyang kernels (same labels, same centroids).
GPU_STRATEGY = {
    "hamerly": "hamerly",
    "yinyang": "yinyang",
    "regroup": "regroup",
    "elkan": "elkan",
    "drake": "yinyang",
    "heap": "yinyang",
    "annulus": "yinyang",
    "exponion": "yinyang",
    "radius": "yinyang",
    "blockvec": "yinyang",
    "drift": "yinyang",
    "search": "yinyang",
}

STRATEGIES = dict(GPU_STRATEGY)


def gpu_groups(strategy: str, n: int, k: int, d: int = 0) -> int:
    """Group count t for the group-bound strategies.  The reference uses
    t = ceil(k/10) (pruners.py:395); the GPU caps it so the n*t bound table
    stays a small fraction of an iteration's HBM traffic.  Elkan keeps one
    bound per centroid while n*k is small; for d <= 32 it runs on the fused
    group-bound kernel with the finest grouping it supports (32 groups, or one
    centroid per group when k <= 32) -- every grouping returns Lloyd's labels."""
    if strategy == "elkan":
        if 0 < d <= 32:
            return min(k, 32)
        return k if n * k <= (1 << 26) else min(k, 64)
    if strategy == "regroup":
        # the device regroup pass handles <= 32 groups
        return max(2, min(32, round(k / 64), k - 1))
    if strategy == "yinyang":
        # ~64 centroids per group (the reference's k/10 would make the n*t
        # table dominate an iteration's traffic at large k), at most 32 groups;
        # the fused path (d <= 32) reads a row's group table only when its
        # global bound fails
        # (and no group above 32767 members: the packed pair format)
        return max(4, min(32, round(k / 64)), -(-k // 32000))
    return 0


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
    gs = GPU_STRATEGY[strategy]
    return run_device(x, k, centers, gs, t_max, ctx, label=strategy, kernel=kernel,
                      record_history=record_history, groups=gpu_groups(gs, x.shape[0], k, x.shape[1]),
                      group_seed=ctx.seed)
