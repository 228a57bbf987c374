"""KnobConfig / run_engine drop-in for the index_mode="none" seam
(/root/reference/pkg/src/lloydkit/engine.py:58-95, :828-853).

Only the bound-pruned and plain-Lloyd branches belong to the GPU hot path;
tree index modes (engine.py:260-952) are out of scope and
raise ContractError here rather than silently running something else.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import ContractError, RunContext, as_points, make_init
from .lloyd import RunResult, run_lloyd
from .pruners import run_pruner

INDEX_MODES = ("none", "pure", "single", "multiple", "adaptive")
BOUND_STRATEGIES = ("none", "elkan", "hamerly", "drake", "heap", "yinyang", "regroup",
                    "annulus", "exponion", "radius", "blockvec", "drift", "full")


@dataclass(frozen=True)
class KnobConfig:
    index_mode: str = "none"
    bound_strategy: str = "none"
    use_search: bool = False
    index_kind: str = "ball"
    capacity: int = 30
    t_max: int = 10
    seed: int = 0

    def validate(self) -> "KnobConfig":
        if self.index_mode not in INDEX_MODES:
            raise ContractError(f"index_mode must be one of {INDEX_MODES}")
        if self.bound_strategy not in BOUND_STRATEGIES:
            raise ContractError(f"bound_strategy must be one of {BOUND_STRATEGIES}")
        if self.index_kind not in ("ball", "kd"):
            raise ContractError("index_kind must be 'ball' or 'kd'")
        if self.capacity < 1:
            raise ContractError("capacity must be >= 1")
        if self.t_max < 0:
            raise ContractError("t_max must be >= 0")
        if self.index_mode == "pure" and self.bound_strategy != "none":
            raise ContractError("pure traversal keeps no bounds; use bound_strategy='none'")
        if self.use_search and (self.index_mode != "none" or self.bound_strategy != "none"):
            raise ContractError("search pre-assignment replaces both index and bounds")
        return self

    def label(self) -> str:
        if self.use_search:
            return "search"
        if self.index_mode == "none":
            return self.bound_strategy if self.bound_strategy != "none" else "lloyd"
        tag = f"{self.index_kind}-{self.index_mode}"
        if self.bound_strategy != "none":
            tag += f"+{self.bound_strategy}"
        return tag


def run_engine(data, k: int, config: KnobConfig, *, init=None, init_method: str = "kmeanspp",
               ctx: RunContext | None = None, kernel: str = "auto") -> RunResult:
    """Run under one knob configuration; Lloyd-identical assignments."""
    config.validate()
    ctx = ctx or RunContext(seed=config.seed)
    x = as_points(data)
    if init is None:
        init = make_init(ctx, x, k, init_method)
    init = np.array(init, dtype=np.float64, copy=True)
    if init.shape != (k, x.shape[1]):
        raise ValueError(f"init shape {init.shape} does not match (k={k}, d={x.shape[1]})")
    if config.use_search:
        res = run_pruner(x, k, "search", init=init, t_max=config.t_max,
                         capacity=config.capacity, ctx=ctx, kernel=kernel)
    elif config.index_mode == "none":
        if config.bound_strategy == "none":
            # "full" is a tree-engine profile (engine.py:129); at index_mode="none"
            # the reference hands it to run_pruner, which raises (pruners.py:868-869)
            res = run_lloyd(x, k, init=init, t_max=config.t_max, ctx=ctx, kernel=kernel)
        else:
            res = run_pruner(x, k, config.bound_strategy, init=init, t_max=config.t_max,
                             ctx=ctx, kernel=kernel)
    elif k == 1:
        res = run_lloyd(x, k, init=init, t_max=config.t_max, ctx=ctx, kernel=kernel)
    else:
        raise ContractError(f"index_mode={config.index_mode!r} (tree engine) is outside the "
                            "GPU hot path; use index_mode='none'")
    res.label = config.label()
    return res
