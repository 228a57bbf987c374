"""Multi-GPU exact Lloyd: one process per GPU, rows sharded, centroids
replicated, one all-reduce per iteration.

The reference is single-process; the only cross-row quantities
of the iteration are the per-cluster member sums / counts and the global
changed count (lloyd.py:165, :78-97), so the exchange is exactly one sum over
ranks of the int64 delta buffer [k*d sums | k counts | k sum|x|^2 | changed].
Because the sums are fixed-point integers the reduction is exact and order
free: every rank computes bit-identical centroids and no broadcast is needed.

`ShardedLloyd` is the protocol, independent of the compute engine:

  bind     all-reduce(MAX) of the per-dimension magnitude exponents, so every
           rank quantizes with the same fixed-point scale
  loop     engine.assign(t) -> delta; all-reduce(SUM, delta); engine.update(t);
           stop after the first iteration whose global changed == 0

`DeviceLloyd` (device.py) is the B200 engine; tests/test_distributed.py drives
the same protocol with world_size 2 over gloo on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [r0, r1) of rank ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return n * rank // world, n * (rank + 1) // world


@dataclass
class ShardedResult:
    iterations: int
    converged: bool
    centroids: np.ndarray
    local_labels: np.ndarray
    changed: list = field(default_factory=list)
    sse: list = field(default_factory=list)


class ShardedLloyd:
    """The per-iteration protocol over a torch.distributed group."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.group = group

    def _all_reduce(self, tensor, op):
        import torch.distributed as dist
        if self.group is not None or (dist.is_available() and dist.is_initialized()):
            dist.all_reduce(tensor, op=op, group=self.group)

    def bind(self):
        import torch.distributed as dist
        q = self.engine.qexp()
        self._all_reduce(q, dist.ReduceOp.MAX)
        self.engine.set_quant()

    def run(self, init, t_max: int, check_every: int = 8, use_graphs: bool = True) -> ShardedResult:
        """Iterations 1..t_max without a host sync per iteration: the engine
        stops itself once an iteration's global changed count is 0 (later
        iterations are device no-ops, their all-reduced deltas are zero), and
        the host reads the counters every ``check_every`` iterations and once
        at the end.  From iteration 2 on an engine that can capture one
        iteration (assign + all-reduce + update) as a CUDA graph replays it."""
        import torch.distributed as dist
        eng = self.engine
        eng.set_centroids(init)
        it = 0
        converged = False
        changed_all = []
        graphs = False
        checked = 0
        for t in range(1, t_max + 1):
            if t == 2 and use_graphs and hasattr(eng, "capture"):
                graphs = eng.capture(t)
            if graphs:
                eng.replay()
            else:
                delta = eng.assign(t)
                self._all_reduce(delta, dist.ReduceOp.SUM)
                eng.update(t)
            if t % check_every == 0 or t == t_max:
                chg = eng.changed_range(checked, t)  # one host sync
                changed_all.extend(chg)
                z = [i for i, c in enumerate(chg) if c == 0]
                if z:
                    it = checked + z[0] + 1
                    converged = True
                    break
                checked = it = t
        changed = changed_all[:it]
        sse = eng.sse_range(0, it)
        return ShardedResult(iterations=it, converged=converged, centroids=eng.centroids(),
                             local_labels=eng.labels(), changed=changed, sse=sse)


def gather_labels(local: np.ndarray, group=None) -> np.ndarray | None:
    """Concatenate every rank's label shard in rank order (all ranks get it)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return local
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, np.asarray(local), group=group)
    return np.concatenate(parts)


class DeviceEngine:
    """Adapter exposing a DeviceLloyd (one GPU, one row shard) to ShardedLloyd."""

    def __init__(self, dev):
        self.dev = dev

    def qexp(self):
        return self.dev.qexp

    def set_quant(self):
        from . import _native as nat
        nat.check(self.dev.lib.lk_set_quant(self.dev.ctx, self.dev.stream_handle()),
                  "lk_set_quant")

    def set_centroids(self, init):
        self.dev.set_centroids(init)

    def assign(self, t):
        from . import _native as nat
        nat.check(self.dev.lib.lk_step_assign(self.dev.ctx, int(t), self.dev.stream_handle()),
                  "lk_step_assign")
        return self.dev.delta

    def update(self, t):
        from . import _native as nat
        nat.check(self.dev.lib.lk_step_update(self.dev.ctx, int(t), self.dev.stream_handle()),
                  "lk_step_update")

    def capture(self, t):
        return self.dev.capture(t)

    def replay(self):
        self.dev.replay()

    def changed_range(self, t0, t1):
        """Global changed counts of iterations t0+1..t1 (one device->host copy)."""
        from . import _native as nat
        return [int(v) for v in self.dev.stats[t0:t1, nat.STAT["changed_global"]].to("cpu").tolist()]

    def sse_range(self, t0, t1):
        return [float(v) for v in self.dev.sse_buf[t0:t1].to("cpu").tolist()]

    def centroids(self):
        return self.dev.c64.to("cpu").numpy().copy()

    def labels(self):
        return self.dev.labels.to("cpu").numpy().astype(np.int64)
