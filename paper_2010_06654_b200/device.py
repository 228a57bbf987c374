"""Device-resident Lloyd engine: binds one block of points to one GPU and runs
the exact iteration through the C ABI (include/lloydkit_b200.h).

Layout in HBM (one torch uint8 workspace, carved by the library):
  X32 [n, ldx] fp32 points (ldx = d rounded up to 4 for d > 2), optional X64
  [n, d] when the input is not fp32-exact; C64 [k, d] fp64 master centroids
  plus an fp32 copy; labels int32 [n]; ub fp32 [n] and lb fp32 [n, nlb] for the
  bounded strategies; fixed-point member sums int64 [k, d] + counts + sum of
  squared norms; the all-reduce payload int64 [k*d + 2k + 8]; worklists.

One process drives one GPU.  With ``comm`` (a torch.distributed group) the
rows are one shard of a larger matrix and the per-iteration delta buffer is
summed across ranks between the assignment and the update phase.
"""

from __future__ import annotations

import ctypes
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import ContractError


def _torch():
    import torch
    return torch


class _nvtx:
    """NVTX range (nsys / ncu --nvtx timelines; a no-op without a profiler)."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        try:
            _torch().cuda.nvtx.range_push(self.name)
            self.on = True
        except Exception:  # pragma: no cover
            self.on = False
        return self

    def __exit__(self, *a):
        if self.on:
            _torch().cuda.nvtx.range_pop()


def _world_size(comm) -> int:
    import torch.distributed as dist
    return dist.get_world_size(comm)


GROUP_STRATEGIES = ("yinyang", "elkan", "regroup")


_GROUP_CACHE: dict = {}


def group_centroids(centers: np.ndarray, t: int, seed: int = 0, n_iters: int = 5,
                    capacity: int = 0) -> np.ndarray:
    """Partition k centroids into t groups by a few Lloyd passes over the
    centroids (the idea of bounds.py:175-196; any grouping yields the same
    labels, it only changes how much the group bounds prune).  capacity > 0
    caps every group's size (the tensor-core group tiles hold 128 centroids).
    The last result is cached (a pure function of the arguments)."""
    key = (hash(centers.tobytes()), centers.shape, t, seed, n_iters, capacity)
    hit = _GROUP_CACHE.get("key")
    if hit == key:
        return _GROUP_CACHE["groups"].copy()
    if capacity > 0:
        g = _tile_groups(centers, t, capacity)
    else:
        g = _group_centroids(centers, t, seed, n_iters)
    _GROUP_CACHE.update(key=key, groups=g.copy())
    return g


def _group_centroids(centers: np.ndarray, t: int, seed: int, n_iters: int) -> np.ndarray:
    k = centers.shape[0]
    t = max(1, min(t, k))
    if t == k:
        return np.arange(k, dtype=np.int32)
    rng = np.random.default_rng(seed)
    means = centers[rng.choice(k, size=t, replace=False)].copy()
    cn = np.sum(centers * centers, axis=1)
    g = np.zeros(k, dtype=np.int64)
    for _ in range(n_iters):
        d2 = cn[:, None] - 2.0 * centers @ means.T + np.sum(means * means, axis=1)[None, :]
        g = np.argmin(d2, axis=1)
        cnt = np.bincount(g, minlength=t)
        sums = np.zeros_like(means)
        np.add.at(sums, g, centers)
        nz = cnt > 0
        means[nz] = sums[nz] / cnt[nz, None]
    return g.astype(np.int32)


def _tile_groups(centers: np.ndarray, t: int, cap: int) -> np.ndarray:
    """Balanced, spatially compact groups of at most ``cap`` centroids: recursive
    bisection at the (size-proportional) quantile of the projection on the
    principal axis (a balanced PCA tree).  A k-means grouping under a size cap
    scatters a large cluster's surplus centroids into far-away groups, which
    then fail for every row of that cluster; bisection keeps every group a
    compact region instead."""
    k = centers.shape[0]
    t = max(1, min(t, k))
    if t * cap < k:
        raise ValueError(f"{t} groups of at most {cap} cannot hold {k} centroids")
    out = np.zeros(k, dtype=np.int32)

    def split(idx, g0, gn):
        if gn == 1:
            out[idx] = g0
            return
        gl = gn // 2
        gr = gn - gl
        m = len(idx)
        nl = int(round(m * gl / gn))
        nl = min(max(nl, m - gr * cap), gl * cap)
        pts = centers[idx]
        c = pts - pts.mean(axis=0)
        if m > 1 and np.any(c):
            _, _, vt = np.linalg.svd(c, full_matrices=False)
            proj = c @ vt[0]
        else:
            proj = np.zeros(m)
        order = np.argsort(proj, kind="stable")
        split(idx[order[:nl]], g0, gl)
        split(idx[order[nl:]], g0 + gl, gr)

    split(np.arange(k), 0, t)
    return out


def _balance_groups(centers: np.ndarray, g: np.ndarray, t: int, cap: int, rounds: int = 3):
    """Capacity-constrained regrouping: (centroid, group) pairs in increasing
    distance to the group means, each centroid to the nearest group with room;
    the means are recomputed and the assignment repeated a few times."""
    k = centers.shape[0]
    t = max(1, min(t, k))
    if t * cap < k:
        raise ValueError(f"{t} groups of at most {cap} cannot hold {k} centroids")
    cn = np.sum(centers * centers, axis=1)
    for _ in range(rounds):
        cnt = np.bincount(g, minlength=t)
        means = np.zeros((t, centers.shape[1]))
        np.add.at(means, g, centers)
        nz = cnt > 0
        means[nz] /= cnt[nz, None]
        d2 = cn[:, None] - 2.0 * centers @ means.T + np.sum(means * means, axis=1)[None, :]
        order = np.argsort(d2, axis=None, kind="stable").tolist()
        out = [-1] * k
        room = [cap] * t
        left = k
        for e in order:
            j, q = divmod(e, t)
            if out[j] < 0 and room[q] > 0:
                out[j] = q
                room[q] -= 1
                left -= 1
                if left == 0:
                    break
        g = np.asarray(out, dtype=np.int64)
    return g.astype(np.int32)


@dataclass
class IterRecord:
    changed: int
    flagged: int
    candidate: int
    active: int
    work: int
    group_dists: int
    sse: float
    assign_ms: float
    update_ms: float
    tile_mode: bool = False  # group tiles: group_dists counts every distance the pass evaluated
    per_centroid: bool = False  # Elkan's per-centroid bounds: group_dists counts every distance
    regrouped: int = 0  # Regroup: the group map was rebuilt before this iteration


class DeviceLogChunk:
    """The moved-row log of iterations t0+1..t1, kept on the device until the
    history is first read (most callers never read it)."""

    def __init__(self, t0: int, t1: int, offs: np.ndarray, log):
        self.t0, self.t1, self.offs, self.log = t0, t1, offs, log

    def download(self):
        torch = _torch()
        if self.log is None:
            log = np.empty((0, 2), dtype=np.int32)
        else:
            host = torch.empty(tuple(self.log.shape), dtype=torch.int32, pin_memory=True)
            host.copy_(self.log)
            log = host.numpy()
        out = []
        for t in range(self.t0, self.t1):
            seg = log[self.offs[t - self.t0]: self.offs[t - self.t0 + 1]]
            out.append((t, seg[:, 0], seg[:, 1]))
        self.log = None
        return out


class LabelHistory(Sequence):
    """assign_history (lloyd.py:140) rebuilt lazily from the device's moved-row
    log: iteration 1 sets every row, iteration t applies its (row, label)
    moves to iteration t-1's vector.  Behaves like the reference's list of
    int64 arrays (len, indexing, iteration)."""

    def __init__(self, n: int, parts, iters: int | None = None):
        self._n = n
        self._parts = parts
        self._iters = len(parts) if iters is None else iters
        self._cache = {}

    def __len__(self):
        return self._iters

    def _resolve(self):
        """Device chunks (t0, t1, offsets, device log) -> host (t, rows, labels)
        parts, downloaded once on first access."""
        if self._parts and isinstance(self._parts[0], DeviceLogChunk):
            parts = []
            for ch in self._parts:
                parts.extend(ch.download())
            self._parts = [p for p in parts if p[0] < self._iters]

    def _build(self, t: int) -> np.ndarray:
        self._resolve()
        """Materialize iteration t from the nearest cached vector at or
        before it; keeps the last vector plus a checkpoint every 8 iterations
        (bounded host memory for long runs at large n)."""
        if t in self._cache:
            return self._cache[t]
        start = max((s for s in self._cache if s < t), default=-1)
        cur = (self._cache[start].copy() if start >= 0 else np.full(self._n, -1, dtype=np.int64))
        for s in range(start + 1, t + 1):
            _, rows, labels = self._parts[s]
            cur[rows] = labels
            if s % 8 == 7 and s < t:
                self._cache[s] = cur.copy()
        for s in [s for s in self._cache if s % 8 != 7]:
            del self._cache[s]
        self._cache[t] = cur
        return cur

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self._build(i).copy()

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


class DeviceLloyd:
    """One GPU context over an (n, d) block of rows."""

    def __init__(self, data, k: int, strategy: str = "lloyd", t_max: int = 10, *,
                 device=None, kernel: str = "auto", groups: int = 0, comm=None,
                 n_total: int | None = None, group_seed: int = 0,
                 record_history: bool = True, history_iters: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise nat.NativeError("no CUDA device: the B200 path has no CPU fallback")
        self.lib = nat.load()
        if strategy not in nat.STRAT_IDS:
            raise ContractError(f"strategy {strategy!r} has no GPU implementation")
        if kernel not in nat.KERNEL_IDS:
            raise ContractError(f"unknown kernel {kernel!r}")
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None
                                else (device.index if isinstance(device, torch.device)
                                      else int(device)))
        self.comm = comm
        self.strategy = strategy
        self.group_seed = group_seed
        self.groups_req = int(groups)
        self.graph_ready = False
        self.k = int(k)
        self.t_max = int(t_max)

        src = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
        if src.ndim != 2:
            raise ContractError(f"expected a 2-D array, got shape {tuple(src.shape)}")
        self.n, self.d = int(src.shape[0]), int(src.shape[1])
        has_x64 = False
        if src.dtype == torch.float64:
            s32 = src.to(torch.float32)
            has_x64 = not bool(torch.equal(s32.to(torch.float64), src))
        if n_total is None:
            n_total = self.n
            if comm is not None:
                import torch.distributed as dist
                t = torch.tensor([self.n], dtype=torch.int64, device=self.dev)
                dist.all_reduce(t, group=comm)
                n_total = int(t.item())
        self.n_total = int(n_total)

        # the history log holds the moves of history_iters iterations between
        # drains (every iteration moves at most n rows); by default all t_max
        # iterations within a 4 GB log, so a run needs no mid-run host sync
        if history_iters <= 0:
            per_iter = max(1, self.n) * 8
            history_iters = max(8, min(max(1, self.t_max), (4 << 30) // per_iter))
        self.history_iters = int(history_iters)
        self.history_cap = self.n * self.history_iters if record_history and self.n else 0
        cfg = nat.LkConfig(n_local=self.n, n_total=self.n_total, d=self.d, k=self.k,
                           strategy=nat.STRAT_IDS[strategy], groups=int(groups),
                           t_max=max(1, self.t_max), kernel=nat.KERNEL_IDS[kernel],
                           has_x64=int(has_x64), device=self.dev.index,
                           history_cap=self.history_cap,
                           ranks=self._ranks(comm))
        self.cfg = cfg
        nbytes = ctypes.c_uint64(0)
        nat.check(self.lib.lk_workspace_bytes(ctypes.byref(cfg), ctypes.byref(nbytes)),
                  "lk_workspace_bytes")
        with torch.cuda.device(self.dev):
            self.ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.dev)
        h = ctypes.c_void_p()
        nat.check(self.lib.lk_ctx_create(ctypes.byref(h), ctypes.byref(cfg),
                                          ctypes.c_void_p(self.ws.data_ptr()), nbytes.value),
                  "lk_ctx_create")
        self.ctx = h
        ldx, dl, nlb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        nat.check(self.lib.lk_layout(h, ctypes.byref(ldx), ctypes.byref(dl), ctypes.byref(nlb)),
                  "lk_layout")
        self.ldx, self.delta_len, self.nlb = ldx.value, dl.value, nlb.value
        gt, gc = ctypes.c_int32(), ctypes.c_int32()
        nat.check(self.lib.lk_group_shape(h, ctypes.byref(gt), ctypes.byref(gc)), "lk_group_shape")
        # group-tile path (capacity 128): the library fixes t = ceil(k / 128)
        self.group_count, self.group_cap = gt.value, gc.value

        self.x32 = self._view("x32", torch.float32, (self.n, self.ldx))
        self.x64 = self._view("x64", torch.float64, (self.n, self.d)) if has_x64 else None
        self.c64 = self._view("c64", torch.float64, (self.k, self.d))
        self.labels = self._view("labels", torch.int32, (self.n,))
        self.delta = self._view("delta", torch.int64, (self.delta_len,))
        self.stats = self._view("stats", torch.int64, (max(1, self.t_max), nat.NSTAT))
        self.sse_buf = self._view("sse", torch.float64, (max(1, self.t_max),))
        self.qexp = self._view("qexp", torch.int32, (3 * self.d + 1,))
        self.counts = self._view("counts", torch.int64, (self.k,))
        self.hlog = (self._view("hlog", torch.int32, (self.history_cap, 2))
                     if self.history_cap else None)
        self.hlog_off = self._view("hlog_off", torch.int64, (max(1, self.t_max) + 1,))
        self.tstamp = self._view("tstamp", torch.int64, (max(1, self.t_max) + 1, 2))
        if strategy != "lloyd":
            self.ub = self._view("ub", torch.float32, (self.n,))
            self.lb = self._view("lb", torch.float32, (self.nlb, self.n))
        self.h2d_bytes = 0
        self._bind(src, has_x64)

    def _ranks(self, comm) -> int:
        """Ranks sharing the rows: > 1 whenever this context holds one shard
        (a communicator, or n_total > n), so every delta is produced before
        the caller's all-reduce."""
        if comm is not None:
            return max(2, _world_size(comm))
        return 2 if self.n_total != self.n else 0

    # -- plumbing ---------------------------------------------------------
    def _view(self, name, dtype, shape):
        torch = _torch()
        off, size = ctypes.c_uint64(), ctypes.c_uint64()
        nat.check(self.lib.lk_buffer(self.ctx, nat.BUF[name], ctypes.byref(off),
                                     ctypes.byref(size)), "lk_buffer")
        numel = int(np.prod(shape))
        esz = torch.empty((), dtype=dtype).element_size()
        if numel * esz > size.value:
            raise nat.NativeError(f"buffer {name} too small ({size.value} < {numel * esz})")
        return self.ws[off.value: off.value + numel * esz].view(dtype).view(*shape)

    def stream_handle(self):
        torch = _torch()
        return ctypes.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def _bind(self, src, has_x64):
        torch = _torch()
        with torch.cuda.device(self.dev):
            if self.ldx != self.d:
                self.x32.zero_()
            if has_x64:
                self.x64.copy_(src, non_blocking=True)
                self.x32[:, : self.d].copy_(self.x64.to(torch.float32))
                self.h2d_bytes += src.numel() * 8
            else:
                s32 = src if src.dtype == torch.float32 else src.to(torch.float32)
                if self.ldx == self.d:
                    self.x32.copy_(s32, non_blocking=True)
                else:
                    self.x32[:, : self.d].copy_(s32, non_blocking=True)
                self.h2d_bytes += s32.numel() * 4
            if isinstance(src, torch.Tensor) and not src.is_cuda:
                # host tensors are validated here, on the device copy (core.as_points)
                chk = self.x64 if has_x64 else self.x32[:, : self.d]
                if not bool(torch.isfinite(chk).all()):
                    from .core import ContractError as _CE
                    raise _CE("data contains non-finite values")
            st = self.stream_handle()
            nat.check(self.lib.lk_scan_points(self.ctx, st), "lk_scan_points")
            if self.comm is not None:
                import torch.distributed as dist
                dist.all_reduce(self.qexp, op=dist.ReduceOp.MAX, group=self.comm)
            nat.check(self.lib.lk_set_quant(self.ctx, st), "lk_set_quant")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.lk_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- iteration --------------------------------------------------------
    def set_groups(self, group_of):
        g = np.ascontiguousarray(group_of, dtype=np.int32)
        nat.check(self.lib.lk_set_groups(self.ctx, ctypes.c_void_p(g.ctypes.data),
                                         self.stream_handle()), "lk_set_groups")

    def set_centroids(self, init):
        torch = _torch()
        if self.strategy in GROUP_STRATEGIES and self.group_cap != 1:
            # (capacity 1: Elkan's per-centroid bounds, no grouping)
            if self.group_cap == 128:
                t, cap = self.group_count, self.group_cap
            else:
                t = min(self.groups_req, self.nlb) if self.groups_req > 0 else self.nlb
                cap = 0
            self.set_groups(group_centroids(np.asarray(init, dtype=np.float64), t,
                                            seed=self.group_seed, capacity=cap))
        with torch.cuda.device(self.dev):
            c = torch.as_tensor(np.ascontiguousarray(init, dtype=np.float64)) \
                if not isinstance(init, torch.Tensor) else init.to(torch.float64)
            self.c64.copy_(c, non_blocking=True)
            self.h2d_bytes += c.numel() * 8
            nat.check(self.lib.lk_set_centroids(self.ctx, ctypes.c_void_p(self.c64.data_ptr()),
                                                self.stream_handle()), "lk_set_centroids")

    def step(self, t: int):
        """One iteration: assign (+recheck, +deltas), all-reduce, update."""
        st = self.stream_handle()
        with _nvtx(f"lk assign t={t}"):
            nat.check(self.lib.lk_step_assign(self.ctx, int(t), st), "lk_step_assign")
        if self.comm is not None:
            import torch.distributed as dist
            with _nvtx(f"lk all-reduce t={t}"):
                dist.all_reduce(self.delta, group=self.comm)
        with _nvtx(f"lk update t={t}"):
            nat.check(self.lib.lk_step_update(self.ctx, int(t), st), "lk_step_update")

    def validate(self, decayed: bool) -> dict:
        """Shadow check of the stored bounds against exact fp64 distances
        (lk_validate_bounds; validate_bounds, bounds.py:280-328): the worst
        overshoot per kind, only kinds that were violated."""
        nout = 2 + max(1, self.group_count)
        out = (ctypes.c_double * nout)()
        nat.check(self.lib.lk_validate_bounds(self.ctx, int(decayed), out, nout, self.stream_handle()),
                  "lk_validate_bounds")
        if self.group_cap == 1:  # Elkan's per-centroid bounds (bounds.py:304-305)
            names = ["ub", "lb_center"]
        else:
            names = ["ub", "lb_global"] + [f"lb_group[{g}]" for g in range(nout - 2)]
        return {nm: float(v) for nm, v in zip(names, out) if v > 0.0}

    def launch_count(self) -> int:
        return int(self.lib.lk_launch_count(self.ctx))

    def profile(self, enable: bool):
        nat.check(self.lib.lk_profile(self.ctx, int(enable)), "lk_profile")

    def profile_read(self, cls: int):
        ms, nl = ctypes.c_double(), ctypes.c_int64()
        nat.check(self.lib.lk_profile_read(self.ctx, cls, ctypes.byref(ms), ctypes.byref(nl)),
                  "lk_profile_read")
        return ms.value, nl.value

    def capture(self, t: int) -> bool:
        """Capture one iteration t >= 2 as a CUDA graph; the iteration index
        lives on the device, so the graph replays every later iteration.

        Single process: assign + update captured natively (lk_graph_capture).
        With a communicator: a torch CUDA graph of lk_step_assign, the
        all-reduce of the delta payload (NCCL is stream-capturable) and
        lk_step_update -- one launch per iteration and no host sync.  A
        backend that cannot be captured (gloo) returns False: eager steps."""
        if t < 2:
            return False
        if self.comm is None:
            nat.check(self.lib.lk_graph_capture(self.ctx, int(t), self.stream_handle()),
                      "lk_graph_capture")
            self.graph_ready = True
            return True
        import torch.distributed as dist
        if dist.get_backend(self.comm) != "nccl":
            return False
        torch = _torch()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.graph(g, stream=side):
            st = ctypes.c_void_p(side.cuda_stream)
            nat.check(self.lib.lk_step_assign(self.ctx, int(t), st), "lk_step_assign")
            dist.all_reduce(self.delta, group=self.comm)
            nat.check(self.lib.lk_step_update(self.ctx, int(t), st), "lk_step_update")
        self._torch_graph = g
        self.graph_ready = True
        return True

    def replay(self):
        g = getattr(self, "_torch_graph", None)
        if g is not None:
            g.replay()
            return
        nat.check(self.lib.lk_graph_replay(self.ctx, self.stream_handle()), "lk_graph_replay")

    def rebind(self, data):
        """Upload new points into this context (same n, d, dtype class)."""
        torch = _torch()
        src = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
        if tuple(src.shape) != (self.n, self.d):
            raise ContractError("rebind: shape mismatch")
        has_x64 = self.x64 is not None
        if src.dtype == torch.float64 and not has_x64:
            if not bool(torch.equal(src.to(torch.float32).to(torch.float64), src)):
                raise ContractError("rebind: fp64 input not fp32-exact on an fp32 context")
        self._bind(src, has_x64)

    def run(self, init, *, record_history: bool = True, check_every: int = 0,
            use_graphs: bool = True, validate: bool = False):
        """Run up to t_max iterations from ``init``; stop after the first with
        changed == 0 (lloyd.py:169-171).  Returns a dict of host arrays.

        validate: debug shadow check of the bounds after every assignment
        ("iter{t}:post") and every centroid update ("iter{t+1}:decayed"), as
        run_pruner does under ctx.debug_validate (pruners.py:896-902); eager
        launches, one host sync per check; res["violations"] lists
        (where, kind, worst overshoot).

        Iterations are launched ahead of the stop test (``check_every``):
        once an iteration reports changed == 0 the device marks the run done
        and every later kernel returns immediately, so iterations launched
        past convergence change nothing."""
        torch = _torch()
        self.set_centroids(init)
        T = self.t_max
        if check_every <= 0 or check_every > self.history_iters:
            # the log holds history_iters iterations: drain at least that often
            check_every = self.history_iters
        res = {"iterations": 0, "converged": False, "history": [], "records": [], "violations": []}
        validate = validate and self.strategy != "lloyd"
        if validate:
            use_graphs = False
            check_every = 1
        if T <= 0:
            res["centroids"] = np.array(init, dtype=np.float64, copy=True)
            res["labels"] = np.full(self.n, -1, dtype=np.int64)
            return res
        record_history = record_history and self.hlog is not None
        with torch.cuda.device(self.dev):
            stream = torch.cuda.current_stream(self.dev)
            chg = torch.zeros(T, dtype=torch.int64, pin_memory=True)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                   torch.cuda.Event(enable_timing=True)) for _ in range(T)]
            log_parts = []      # (iteration, rows, labels) drained from the device log
            graphs = False
            iters = T
            converged = False
            checked = 0
            for t in range(1, T + 1):
                e0, e1, e2 = ev[t - 1]
                if t == 2 and use_graphs:
                    # the graph of a cached context is reused across calls
                    graphs = self.graph_ready or self.capture(2)
                e0.record(stream)
                nv = _nvtx(f"lk iteration {t}")
                nv.__enter__()
                if graphs:
                    self.replay()  # assign + update; timed as one phase
                    e1.record(stream)
                else:
                    nat.check(self.lib.lk_step_assign(self.ctx, t, self.stream_handle()),
                              "lk_step_assign")
                    if validate:
                        for kind, v in self.validate(False).items():
                            res["violations"].append((f"iter{t}:post", kind, v))
                    if self.comm is not None:
                        import torch.distributed as dist
                        dist.all_reduce(self.delta, group=self.comm)
                    e1.record(stream)
                    nat.check(self.lib.lk_step_update(self.ctx, t, self.stream_handle()),
                              "lk_step_update")
                    if validate and t < T:
                        for kind, v in self.validate(True).items():
                            res["violations"].append((f"iter{t + 1}:decayed", kind, v))
                e2.record(stream)
                nv.__exit__()
                chg[t - 1].copy_(self.stats[t - 1, nat.STAT["changed_global"]], non_blocking=True)
                if t % check_every == 0 or t == T:  # (t=1 cannot converge: n rows move)
                    stream.synchronize()
                    z = np.nonzero(chg[checked:t].numpy() == 0)[0]
                    t_end = checked + int(z[0]) + 1 if len(z) else t
                    if record_history:
                        # iterations launched past convergence were no-ops and
                        # wrote no log offsets: drain only up to t_end
                        self._drain_history(checked, t_end, log_parts)
                    if len(z):
                        iters = t_end
                        converged = True
                        break
                    checked = t
            # one sync for every result: stats, SSE, centroids, int64 labels
            # (widened on the device) into pinned buffers
            h_stats = torch.empty(tuple(self.stats[:iters].shape), dtype=self.stats.dtype, pin_memory=True)
            h_sse = torch.empty(tuple(self.sse_buf[:iters].shape), dtype=self.sse_buf.dtype, pin_memory=True)
            h_c64 = torch.empty(tuple(self.c64.shape), dtype=self.c64.dtype, pin_memory=True)
            h_ts = torch.empty((iters + 1, 2), dtype=torch.int64, pin_memory=True)
            h_ts.copy_(self.tstamp[: iters + 1], non_blocking=True)
            lab = torch.empty(self.n, dtype=torch.int64, pin_memory=True)
            h_stats.copy_(self.stats[:iters], non_blocking=True)
            h_sse.copy_(self.sse_buf[:iters], non_blocking=True)
            h_c64.copy_(self.c64, non_blocking=True)
            lab.copy_(self.labels, non_blocking=True)
            stream.synchronize()
            stats = h_stats.numpy().copy()
            sse = h_sse.numpy().copy()
            if self.comm is not None:
                import torch.distributed as dist
                st_t = torch.as_tensor(stats, device=self.dev)
                dist.all_reduce(st_t, group=self.comm)
                g = st_t.to("cpu").numpy()
                g[:, nat.STAT["changed_global"]] = stats[:, nat.STAT["changed_global"]]
                stats = g
            # assign / refine split from the device-clock stamps of the library
            # (valid under graph replay); host events where a stamp is missing
            ts = h_ts.numpy().astype(np.uint64)
            recs = []
            for t in range(iters):
                e0, e1, e2 = ev[t]
                s_prev, u0, u1 = ts[t, 1], ts[t + 1, 0], ts[t + 1, 1]
                if max(s_prev, u0, u1) < np.uint64(1 << 63) and s_prev <= u0 <= u1:
                    a_ms, u_ms = float(u0 - s_prev) / 1e6, float(u1 - u0) / 1e6
                else:
                    a_ms, u_ms = e0.elapsed_time(e1), e1.elapsed_time(e2)
                recs.append(IterRecord(
                    changed=int(stats[t, nat.STAT["changed_global"]]),
                    flagged=int(stats[t, nat.STAT["flagged"]]),
                    candidate=int(stats[t, nat.STAT["candidate"]]),
                    active=int(stats[t, nat.STAT["active"]]),
                    work=int(stats[t, nat.STAT["work"]]),
                    group_dists=int(stats[t, nat.STAT["dist"]]),
                    sse=float(sse[t]),
                    assign_ms=a_ms,
                    update_ms=u_ms,
                    tile_mode=self.group_cap == 128, per_centroid=self.group_cap == 1,
                    regrouped=int(stats[t, nat.STAT["regrouped"]])))
            res["iterations"] = iters
            res["converged"] = converged
            res["records"] = recs
            res["centroids"] = h_c64.numpy().copy()
            res["labels"] = lab.numpy()  # int64 labels (lloyd.py:52)
            if record_history:
                res["history"] = LabelHistory(self.n, [c for c in log_parts if c.t0 < iters],
                                              iters=iters)
        return res

    def _drain_history(self, t0: int, t1: int, parts: list):
        """Copy the device history log of iterations t0+1..t1 to the host and
        rewind the log (it holds at most check_every iterations of moves)."""
        offs = self.hlog_off[t0: t1 + 1].to("cpu").numpy()
        if np.any(offs < 0):
            raise nat.NativeError("label-history log overflow")
        # the segment stays on the device (a copy: the log is rewound and reused)
        # and is downloaded when the history is first read
        log = self.hlog[: offs[-1]].clone() if offs[-1] > 0 else None
        parts.append(DeviceLogChunk(t0, t1, offs, log))
        self.hlog_off[t1].zero_()
