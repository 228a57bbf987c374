"""Run bookkeeping shared by every entry point: errors, counters, run context,
input validation and seeding.

Mirrors the reference's core module (/root/reference/pkg/src/lloydkit/core.py)
for the names the hot path needs -- ContractError (:29-30), Counters (:33-56),
RunContext (:59-71), input validation (:74-83), init_random (:182-189),
init_kmeanspp (:192-217), make_init (:223-228), sse (:172-179) -- so code
written against the reference keeps working.  Seeding stays on the host with
numpy's PCG64 so the GPU path starts from exactly the centroids the reference
would pick.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

RNG_NAME = "pcg64"


class ContractError(ValueError):
    """An operation was called with arguments violating its contract."""


@dataclass
class Counters:
    """Work counters for one run (same fields as the reference's Counters)."""

    dist_comps: int = 0
    pivot_dist_comps: int = 0
    bound_dist_comps: int = 0
    data_accesses: int = 0
    node_accesses: int = 0
    bound_accesses: int = 0
    bound_updates: int = 0
    iterations: int = 0
    wall_nanos: int = 0

    def copy(self) -> "Counters":
        return dataclasses.replace(self)

    def delta(self, earlier: "Counters") -> "Counters":
        return Counters(**{f.name: getattr(self, f.name) - getattr(earlier, f.name)
                           for f in dataclasses.fields(self)})


@dataclass
class RunContext:
    """Per-run bundle of counters, RNG, and debug switches."""

    seed: int = 0
    counters: Counters = field(default_factory=Counters)
    debug_validate: bool = False
    violations: list = field(default_factory=list)
    rng: np.random.Generator = None  # type: ignore[assignment]

    def __post_init__(self):
        if self.rng is None:
            self.rng = np.random.default_rng(self.seed)


def as_matrix(data) -> np.ndarray:
    """Validate and return data as a float64 (n, d) matrix (reference semantics)."""
    x = np.asarray(data, dtype=np.float64)
    _validate(x)
    return x


def as_points(data):
    """Validate without widening: float32 input stays float32 (it is upcast to
    fp64 exactly wherever fp64 is needed), anything else becomes float64.

    Accepts numpy arrays, nested sequences and torch tensors (CPU, pinned or
    CUDA; those are returned as-is after validation)."""
    try:
        import torch
        if isinstance(data, torch.Tensor):
            if data.ndim != 2:
                raise ContractError(f"expected a 2-D array, got shape {tuple(data.shape)}")
            if data.shape[0] == 0 or data.shape[1] == 0:
                raise ContractError(f"empty data matrix with shape {tuple(data.shape)}")
            if data.dtype not in (torch.float32, torch.float64):
                data = data.to(torch.float64)
            if data.is_cuda:
                if not bool(torch.isfinite(data).all()):
                    raise ContractError("data contains non-finite values")
            # host tensors: checked on the device right after the upload
            # (DeviceLloyd._bind), before any iteration runs
            return data
    except ImportError:  # pragma: no cover
        pass
    x = np.asarray(data)
    if x.dtype != np.float32:
        x = np.asarray(x, dtype=np.float64)
    _validate(x)
    return x


def _validate(x):
    if x.ndim != 2:
        raise ContractError(f"expected a 2-D array, got shape {x.shape}")
    if x.shape[0] == 0 or x.shape[1] == 0:
        raise ContractError(f"empty data matrix with shape {x.shape}")
    if not np.isfinite(x).all():
        raise ContractError("data contains non-finite values")


def _host64(data) -> np.ndarray:
    try:
        import torch
        if isinstance(data, torch.Tensor):
            return data.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(data, dtype=np.float64)


def init_random(ctx: RunContext, data, k: int) -> np.ndarray:
    """k distinct rows chosen uniformly (ctx.rng.choice without replacement)."""
    x = as_points(data)
    n = x.shape[0]
    if not 1 <= k <= n:
        raise ContractError(f"k={k} out of range for n={n}")
    idx = ctx.rng.choice(n, size=k, replace=False)
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x[torch.as_tensor(idx)].to("cpu", torch.float64).numpy().copy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x[idx], dtype=np.float64).copy()


def init_kmeanspp(ctx: RunContext, data, k: int) -> np.ndarray:
    """D^2 seeding with the reference's draw sequence (first row via
    rng.integers, later rows via rng.choice(p=d2/sum), uniform over the
    unchosen rows when every weight is zero).  Host numpy; the squared
    distances are formed with the same elementwise ops so the probabilities,
    hence the draws, are identical."""
    pts = as_points(data)
    n = pts.shape[0]
    if not 1 <= k <= n:
        raise ContractError(f"k={k} out of range for n={n}")
    if k > 1 and n * pts.shape[1] >= KMEANSPP_DEVICE_MIN:
        dev = _kmeanspp_device(ctx, pts, k)
        if dev is not None:
            return dev
    x = _host64(pts)
    picks = np.empty(k, dtype=np.int64)
    picks[0] = ctx.rng.integers(n)
    d2 = np.sum((x - x[picks[0]]) ** 2, axis=1)
    for j in range(1, k):
        total = d2.sum()
        if total > 0.0:
            picks[j] = ctx.rng.choice(n, p=d2 / total)
        else:
            picks[j] = ctx.rng.choice(np.setdiff1d(np.arange(n), picks[:j]))
        d2 = np.minimum(d2, np.sum((x - x[picks[j]]) ** 2, axis=1))
    return x[picks].copy()


# k-means++ moves its D^2 updates to the GPU from this many elements on
KMEANSPP_DEVICE_MIN = 1 << 16


def _kmeanspp_device(ctx: RunContext, pts, k: int):
    """init_kmeanspp with the D^2 updates on the GPU (lk_d2_update: fp64,
    numpy's pairwise order, so d2 is bit-identical to the host expression) and
    the draws on the host with the same numpy calls on the same d2 array
    (core.py:205-215 of the reference: d2.sum(), d2 / total, rng.choice), so
    the picks are the reference's.  None when no CUDA device / library."""
    try:
        import torch
        if not torch.cuda.is_available():
            return None
        from . import _native as nat
        lib = nat.load()
    except Exception:  # noqa: BLE001  (no device or no library: host path)
        return None
    import ctypes
    n, d = pts.shape
    if isinstance(pts, torch.Tensor):
        src = pts.detach()
    else:
        src = torch.from_numpy(np.ascontiguousarray(pts))
    xd = src.to("cuda").contiguous()
    is32 = xd.dtype == torch.float32
    x64h = _host64(pts)
    d2d = torch.empty(n, dtype=torch.float64, device="cuda")
    d2h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    cd = torch.empty(d, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    sh = ctypes.c_void_p(stream.cuda_stream)
    x32p = ctypes.c_void_p(xd.data_ptr()) if is32 else None
    x64p = None if is32 else ctypes.c_void_p(xd.data_ptr())

    def update(row: int, first: int):
        cd.copy_(xd[row])  # device-side widening of the chosen row (exact)
        nat.check(lib.lk_d2_update(x32p, x64p, n, d, d, ctypes.c_void_p(cd.data_ptr()),
                                   ctypes.c_void_p(d2d.data_ptr()), first, sh), "lk_d2_update")
        d2h.copy_(d2d, non_blocking=True)
        stream.synchronize()
        return d2h.numpy()

    picks = np.empty(k, dtype=np.int64)
    picks[0] = ctx.rng.integers(n)
    d2 = update(int(picks[0]), 1)
    for j in range(1, k):
        total = d2.sum()
        if total > 0.0:
            picks[j] = ctx.rng.choice(n, p=d2 / total)
        else:
            picks[j] = ctx.rng.choice(np.setdiff1d(np.arange(n), picks[:j]))
        if j < k - 1:
            d2 = update(int(picks[j]), 0)
    return x64h[picks].copy()


INITS = {"random": init_random, "kmeanspp": init_kmeanspp}


def make_init(ctx: RunContext, data, k: int, method: str = "kmeanspp") -> np.ndarray:
    if method not in INITS:
        raise ContractError(f"unknown init method {method!r}")
    return INITS[method](ctx, data, k)


def sse(data, centers, assign) -> float:
    """Sum of squared distances to the assigned centroid (host, instrumentation)."""
    x = _host64(data)
    diff = x - np.asarray(centers, dtype=np.float64)[np.asarray(assign)]
    return float(np.sum(diff * diff))
