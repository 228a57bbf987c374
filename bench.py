#!/usr/bin/env python
"""Benchmark of the exact Lloyd iteration on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg5] [--strategy yinyang] [--kernel auto]

Default workload: BASELINE configs[4] = cfg5 (n=5e7, d=32, k=4096), the largest
configuration that fits one GPU, with the group-tile Yinyang path.

A "step" is one Lloyd iteration (assignment over all n points -- full scan or
bound-pruned, labels identical to Lloyd -- plus refinement) over the whole
workload, continuing one trajectory from the reference's random init: W
untimed iterations, then K timed ones (iterations W+1 .. W+K).

metric  "Lloyd iterations/sec": value = K / (sum of the K iterations' device
        time, max over ranks).  Inputs are resident in HBM; L2 is flushed
        (256 MB write) between timed iterations, outside the timed events.
e2e     the same metric through the public API (run_pruner / run_lloyd with
        a pinned host matrix): H2D of the points and init, the iterations,
        D2H of per-iteration labels (history) and the final centroids.
roofline  the dominant kernel class of the timed window (per-class CUDA
        events inside the library, a second pass over the same iterations),
        achieved algorithmic GB/s or TFLOP/s against MEASURED_PEAKS.json.
cpu_baseline  the CPU oracle port (oracle/, fp64, all host threads) on a
        bounded row sample of the same workload, extrapolated linearly in n.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

L2_FLUSH_BYTES = 256 << 20
FP32_FLOP_PER_SM_CLK = 256  # 128 FP32 lanes x FMA
N_SMS = 148


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"],
                "sm_max_mhz": j.get("sm_max_mhz", 1965.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        busy = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard_rows(n: int, ws: int, rank: int):
    return n * rank // ws, n * (rank + 1) // ws


# ---------------------------------------------------------------------------
# CPU baseline (oracle port) on a bounded sample


def cpu_sample_rate(workload: str, strategy: str, warmup: int, steps: int, budget_s: float = 15.0):
    """Oracle port (fp64, all host threads) over the first n_s rows with the
    same k and init rule; returns (iterations/s scaled to full n, info)."""
    from oracle import oracle as O
    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.core import RunContext, init_random

    cfg = datasets.CONFIGS[workload]
    threads = O.default_threads()
    # size the sample so one full-scan iteration is ~budget/(W+K) seconds at
    # ~1 ns per (row, centroid, dim) per thread
    per_row = cfg.k * max(cfg.d, 4) * 1.0e-9 / threads
    n_s = int(budget_s / max(1, warmup + steps) / per_row)
    n_s = max(4 * cfg.k, min(cfg.n, n_s))
    x = datasets.generate(workload, n_s)
    init = init_random(RunContext(seed=cfg.seed_init), x, cfg.k)
    t_total = warmup + steps
    fn = O.run_hamerly if strategy != "lloyd" else O.run_lloyd
    t0 = time.perf_counter()
    fn(x, cfg.k, init, warmup, nthreads=threads, record_history=False) if warmup else None
    t1 = time.perf_counter()
    out = fn(x, cfg.k, init, t_total, nthreads=threads, record_history=False)
    t2 = time.perf_counter()
    it_done = out["iterations"]
    timed_its = max(1, it_done - warmup)
    timed_s = max(1e-9, (t2 - t1) - (t1 - t0))
    rate = timed_its / timed_s * (n_s / cfg.n)
    info = {"n_sample": n_s, "iterations": timed_its, "seconds": round(t2 - t1 + (t1 - t0), 3),
            "threads": threads, "strategy": "hamerly" if strategy != "lloyd" else "lloyd"}
    return rate, info


# ---------------------------------------------------------------------------


def algorithmic_work(cls: int, strategy: str, n: int, d: int, k: int, recs, kernel_tc: bool,
                     groups: int = 1, tiles: bool = False):
    """Algorithmic units of one kernel class summed over the timed iterations:
    ("flop", F) or ("byte", B).  Per-unit figures are listed in DESIGN.md.
    tiles: the block-sparse group-tile Yinyang path (d <= 32 on the tensor
    cores), whose pass counts every (row, centroid) product it evaluates."""
    ldx = d if d <= 2 else (d + 3) // 4 * 4
    if tiles:
        nlb = (groups + 3) // 4 * 4
        if cls == 0:  # k_assign_tgy: 2*d flops per evaluated (row, centroid) pair
            return "flop", sum(2.0 * (n * k if r["t"] == 1 else r["group_dists"]) * d for r in recs)
        if cls == 1:  # k_filter_tgy: label/ub/glb per row; point + group-table row per
            # row failing the global gate; worklist entry (row, mask, bound) per listed row
            return "byte", sum(12.0 * n + r["active"] * (4.0 * ldx + 4.0 * nlb) + 16.0 * r["work"]
                               for r in recs)
        if cls == 10:  # sort + centered gather: worklist entry and label in, point in,
            # hi/lo rows and the 32-byte record out, per listed row
            return "byte", sum(r["work"] * (20.0 + 12.0 * ldx + 32.0) for r in recs)
    if cls == 7:  # tensor-core candidate pass over the ambiguous rows
        return "flop", sum(2.0 * r["candidate"] * k * d for r in recs)
    if cls == 9:  # fp32 rescan of candidate-overflow rows
        return "flop", sum(2.0 * r["overflow"] * k * d for r in recs)
    if cls == 8:  # fp64 over <= 16 candidates: 3 fp64 flops per (candidate, dim)
        return "flop", sum(3.0 * r["candidate"] * 4 * d for r in recs)
    if cls == 0:  # assignment: 2*d flops per (row, centroid) pair evaluated
        rows = sum(n if (strategy == "lloyd" or r["t"] == 1) else r["work"] for r in recs)
        return "flop", 2.0 * rows * k * d
    if cls == 1 and strategy in ("yinyang", "elkan") and d <= 32 and groups <= 32:
        # fused Yinyang kernel (lazy bounds): label + ub + global bound of every
        # row; the group table, point and ub/glb rewrites of the rows failing
        # the global bound; label/ub/glb + one bound per scanned group of the
        # rows that reach the group scans
        t = max(1, groups)
        return "byte", sum(12.0 * n + r["active"] * (4.0 * t + 4.0 * d + 8.0)
                           + 12.0 * r["ywl"] + 4.0 * r["pairs"] for r in recs)
    if cls == 1 and strategy in ("yinyang", "elkan"):
        # group filter: label/ub/lb-table traffic + tightened rows + group scans
        t = max(1, groups)
        return "byte", sum(n * (12.0 + 8.0 * t) + 4.0 * d * r["active"] for r in recs)
    if cls == 1:  # Hamerly filter: label 4 + ub 4 + lb 4 read, ub 4 + lb 4 written,
        # 4 per appended row, + the tightened rows' point (4d)
        return "byte", sum(20.0 * n + 4.0 * r["work"] + 4.0 * d * r["active"] for r in recs)
    if cls == 5:  # group scans: 2*d flops per (row, centroid) evaluated
        return "flop", sum(2.0 * r.get("group_dists", 0) * d for r in recs)
    if cls == 6:  # merge: worklist entry 16 + 8, pair results 24 per scan, bound writes
        return "byte", sum(24.0 * r["ywl"] + 28.0 * r["pairs"] for r in recs)
    if cls == 2:  # recheck: fp64 flops 3*d per pair (sub, mul, add)
        return "flop", sum(3.0 * r["flagged"] * k * d for r in recs)
    if cls == 3:  # refine: moved rows (4d read + 8 move record + 4 label) + 2 sums rows (8d rmw)
        return "byte", sum(r["changed"] * (4.0 * d + 12.0 + 32.0 * d) for r in recs)
    # update: k*d int64 sums + fp64 centroids read/write, delta read
    return "byte", len(recs) * k * d * (8.0 * 5 + 4.0)


CLASS_NAMES = {0: "assign", 1: "filter", 2: "recheck_fp64", 3: "refine", 4: "update",
               5: "group_scan", 6: "group_merge", 7: "tc_collect", 8: "cand_recheck",
               9: "ovf_rescan", 10: "sort_gather"}


def measure_tf32_tflops(reps: int = 12) -> float:
    """Dense TF32 tensor throughput of this GPU: torch.matmul fp32 8192^3 with
    allow_tf32 (cuBLAS), best of ``reps`` timed with CUDA events."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        nn = 8192
        a = torch.randn(nn, nn, device="cuda")
        b = torch.randn(nn, nn, device="cuda")
        for _ in range(3):
            torch.matmul(a, b)
        best = float("inf")
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * nn ** 3 / (best / 1e3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def run_ours(args):
    import torch

    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.core import RunContext, init_random
    from paper_2010_06654_b200.device import DeviceLloyd

    ws, rank, local = dist_env()
    # one process per GPU; LK_DIST_BACKEND=gloo (host-staged exchange) lets the
    # multi-rank flow run on a single-GPU box for testing
    backend = os.environ.get("LK_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    group = None
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD

    cfg = datasets.CONFIGS[args.workload]
    W, K = args.warmup, args.steps
    T = W + K
    r0, r1 = shard_rows(cfg.n, ws, rank)
    if ws == 1:
        x_full = datasets.generate(args.workload)
        init = init_random(RunContext(seed=cfg.seed_init), x_full, cfg.k)
        x = x_full
    else:
        # each rank generates only its own shard (and the init rows)
        x_full = None
        x = datasets.generate_rows(args.workload, r0, r1)
        init = datasets.init_from_rows(args.workload)
    n, d, k = cfg.n, cfg.d, cfg.k
    strategy = args.strategy
    gpu_strat = strategy
    from paper_2010_06654_b200.pruners import gpu_groups
    n_groups = args.groups or gpu_groups(gpu_strat, n, k, d)
    eng = DeviceLloyd(x, k, gpu_strat, T, kernel=args.kernel, comm=group, n_total=n,
                      groups=n_groups, group_seed=cfg.seed_init, record_history=False)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def trajectory(profile: bool):
        eng.set_centroids(init)
        for t in range(1, W + 1):
            eng.step(t)
        torch.cuda.synchronize()
        # one captured iteration replays every later one (device-side
        # iteration index); the profiled pass runs eagerly for per-class events
        graphs = False if (profile or args.no_graph) else eng.capture(W + 1)
        launches_per_step = 0
        if graphs:
            l0 = eng.launch_count()
            eng.capture(W + 1)  # count the kernels one captured iteration holds
            launches_per_step = eng.launch_count() - l0
        if profile:
            eng.profile(True)
        barrier()
        torch.cuda.synchronize()
        launches0 = eng.launch_count()
        evs = []
        for t in range(W + 1, T + 1):
            flush.fill_(t & 0xFF)  # L2 flush between timed iterations (not timed)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if graphs:
                eng.replay()
            else:
                eng.step(t)
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        launched = eng.launch_count() - launches0 + launches_per_step * (T - W if graphs else 0)
        return ms, launched

    # untimed dry run (JIT / first-touch), then the timed trajectory
    trajectory(False)
    with ClockSampler(local) as clk:
        ms, launches = trajectory(False)
    ms_max = ms
    if ws > 1:
        import torch.distributed as dist
        t_ = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms_max = float(t_.item())
    stats = eng.stats[:T].to("cpu").numpy()
    chg = stats[:, 7]
    converged_in_window = bool(np.any(chg[W:T - 1] == 0))
    recs = [{"t": t + 1, "changed": int(stats[t, 0]), "flagged": int(stats[t, 1]),
             "candidate": int(stats[t, 6]), "ywl": int(stats[t, 9]), "pairs": int(stats[t, 10]),
             "group_dists": int(stats[t, 4]), "overflow": int(stats[t, 8]),
             "active": int(stats[t, 2]), "work": int(stats[t, 3])} for t in range(W, T)]

    # profiled pass over the same iterations: per-class device time
    _, _ = trajectory(True)
    cls_ms = {c: eng.profile_read(c)[0] for c in CLASS_NAMES}
    eng.profile(False)
    dom = max(cls_ms, key=lambda c: cls_ms[c])
    peaks = load_peaks()
    tiles = eng.group_cap == 128
    if tiles:
        n_groups = eng.group_count
    kind, units = algorithmic_work(dom, gpu_strat, x.shape[0], d, k, recs, False, n_groups, tiles)
    dom_s = cls_ms[dom] / 1e3
    uses_tc = args.kernel == "tc" or (args.kernel == "auto" and d >= 32)
    if kind == "flop":
        if dom in (2, 8):
            peak, pk_src, bound = 37.0, "nominal B200 FP64 (no measured figure)", "compute-fp64"
        elif uses_tc and dom in (0, 7):
            tf32 = measure_tf32_tflops()
            peak = tf32 / 3.0
            pk_src = (f"measured dense TF32 {tf32:.0f} TFLOP/s (torch.matmul fp32 8192^3, "
                      "allow_tf32, best of 12, this run) / 3 for the 3xTF32 split")
            bound = "tensor"
        else:
            peak = N_SMS * FP32_FLOP_PER_SM_CLK * peaks["sm_max_mhz"] * 1e6 / 1e12
            pk_src = f"FP32 SIMT = {N_SMS} SMs x 256 flop/clk x sm_max_mhz ({peaks['src']} clock)"
            bound = "compute-fp32"
        achieved = units / dom_s / 1e12 if dom_s > 0 else 0.0
        roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": None,
                "kernel": CLASS_NAMES[dom], "peak_source": pk_src}
    else:
        achieved = units / dom_s / 1e9 if dom_s > 0 else 0.0
        peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "kernel": CLASS_NAMES[dom],
                "peak_source": f"hbm_gbs ({peaks['src']})"}
    tot_cls = sum(cls_ms.values()) or 1.0
    roof["share_of_step"] = cls_ms[dom] / tot_cls
    roof["class_ms_per_step"] = {CLASS_NAMES[c]: cls_ms[c] / K for c in cls_ms}
    roof["traffic_note"] = ("null here: dram bytes of this kernel come from an ncu --set full "
                            "capture of the same command, profiles/r02/")
    eng.close()
    del eng, flush  # (the workspace is a torch tensor: free it before the e2e calls)
    torch.cuda.empty_cache()

    # e2e through the public API, pinned host input
    e2e = None
    if ws > 1:
        # multi-GPU public API (distributed.py): each rank binds its pinned host
        # shard, runs the sharded protocol (one NCCL all-reduce per iteration)
        # and reads its labels back; wall time max over ranks
        import torch.distributed as dist
        from paper_2010_06654_b200.distributed import DeviceEngine, ShardedLloyd
        xs = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()

        def sharded_call():
            dev = DeviceLloyd(xs, k, gpu_strat, T, kernel=args.kernel, comm=group, n_total=n,
                              groups=n_groups, group_seed=cfg.seed_init, record_history=False)
            drv = ShardedLloyd(DeviceEngine(dev), group)
            drv.bind()
            out = drv.run(init, T)
            dev.close()
            return out

        sharded_call()  # warm-up
        walls = []
        for _ in range(3):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = sharded_call()
            torch.cuda.synchronize()
            w = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            dist.all_reduce(w, op=dist.ReduceOp.MAX)
            walls.append(float(w.item()))
        wall = statistics.median(walls)
        its = res.iterations
        e2e = {"value": its / wall, "unit": "iterations/s",
               "h2d_bytes_per_step": int((n * d * 4 + ws * init.nbytes) / its),
               "d2h_bytes_per_step": int((8 * n + ws * k * d * 8) / its),
               "iterations": its, "wall_s": wall, "calls": 3, "statistic": "median",
               "includes": "per rank: context+workspace setup, H2D of its pinned shard, the "
                           "sharded iterations (one all-reduce of the int64 delta each), its "
                           "labels and the centroids D2H; wall time max over ranks"}
    if ws == 1:
        import paper_2010_06654_b200 as lk
        xp = torch.from_numpy(x).pin_memory()

        def api_call():
            if strategy == "lloyd":
                return lk.run_lloyd(xp, k, init=init, t_max=T)
            return lk.run_pruner(xp, k, strategy, init=init, t_max=T)

        api_call()  # warm-up call (module/attribute setup, allocator)
        walls = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = api_call()
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        wall = statistics.median(walls)
        its = len(res.iterations)
        e2e = {"value": its / wall, "unit": "iterations/s",
               "h2d_bytes_per_step": int((x.nbytes + init.nbytes) / its),
               "d2h_bytes_per_step": int((8 * n + k * d * 8 + 8 * its * (16 + 1)) / its),
               "iterations": its, "wall_s": wall, "calls": 3, "statistic": "median",
               "includes": "validation, H2D of the points from pinned memory (cached device "
                           "context), centroid grouping, iterations (CUDA-graph replay; one host sync "
                           "at the end, the device stops itself at convergence), per-iteration counters, "
                           "final int64 labels and centroids D2H; the label history stays on "
                           "the device until read (lazy RunResult.assign_history)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        rate, info = cpu_sample_rate(args.workload, strategy, W, K, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": "iterations/s", "cores": info["threads"], "kind": "port",
               "sample": f"oracle port ({info['strategy']}, fp64) over the first "
                         f"{info['n_sample']} of {n} rows, same k and init rule, "
                         f"iterations {W + 1}..{W + info['iterations']}, "
                         f"{info['seconds']} s; rate scaled by n_sample/n (extrapolated)"}

    if rank == 0:
        value = K / (ms_max / 1e3)
        line = {
            "metric": "Lloyd iterations/sec", "value": value, "unit": "iterations/s",
            "n_gpus": ws, "steps": K, "warmup": W, "ms_per_step": ms_max / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32 (certified; fp64 recheck)", "data": "synthetic",
            "config": workload_config(args, cfg),
            "strategy": f"{strategy} (GPU; kernel={args.kernel}, {n_groups} groups"
                        + (", group tiles" if tiles else "") + ")",
            "run": {"parallelism": f"dp{ws} (row shards, int64 delta all-reduce)",
                    "converged_in_window": converged_in_window,
                    "timed": "device events per iteration on the launching stream, max over ranks"},
            "effective_tflops": 2.0 * n * k * d * value / 1e12,
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "window_stats": {"changed": [r["changed"] for r in recs],
                             "rescanned": [r["work"] for r in recs],
                             "rechecked": [r["flagged"] for r in recs],
                             "candidate_rows": [r["candidate"] for r in recs],
                             "overflow_rows": [r["overflow"] for r in recs],
                             "group_rows": [r["ywl"] for r in recs],
                             "group_scans": [r["pairs"] for r in recs],
                             "group_dists": [r["group_dists"] for r in recs],
                             "active": [r["active"] for r in recs]},
        }
        print(json.dumps(line))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2010_06654_b200 import datasets
    cfg = datasets.CONFIGS[args.workload]
    rate, info = cpu_sample_rate(args.workload, args.strategy, args.warmup, args.steps,
                                 budget_s=args.cpu_budget)
    line = {
        "impl": "reference", "metric": "Lloyd iterations/sec", "value": rate,
        "unit": "iterations/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / rate if rate else None, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp64", "data": "synthetic",
        "config": workload_config(args, cfg),
        "strategy": f"{info['strategy']} (oracle C port of the reference's algorithm, fp64; "
                    "every exact strategy returns Lloyd's labels)",
        "cpu_baseline": {"value": rate, "unit": "iterations/s", "cores": info["threads"],
                         "kind": "port",
                         "sample": f"oracle port ({info['strategy']}, fp64, {info['threads']} "
                                   f"threads) over {info['n_sample']} of {cfg.n} rows, "
                                   f"{info['iterations']} timed iterations after "
                                   f"{args.warmup} warm-up, scaled by n_sample/n"},
        "e2e": {"value": rate, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def workload_config(args, cfg) -> dict:
    """The workload both arms run (identical dicts: strategy and machine details
    are reported beside it)."""
    return {"workload": args.workload, "n": cfg.n, "d": cfg.d, "k": cfg.k,
            "iterations": f"{args.warmup + 1}..{args.warmup + args.steps} of one trajectory from "
                          f"the reference's random init (seed {cfg.seed_init})",
            "l2": "GPU arm: 256 MB L2 flush between timed iterations (outside the events)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--strategy", default="yinyang",
                    choices=["lloyd", "hamerly", "yinyang", "elkan", "regroup"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--groups", type=int, default=0, help="Yinyang group count (0 = default)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches in the timed loop")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)  # contract: at least 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
