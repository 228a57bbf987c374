/*
 * lloydkit_b200.h -- C ABI of the B200-native exact-Lloyd hot path.
 *
 * The reference (lloydkit, pure Python + numpy) has no native boundary of its
 * own; its hot path is reached through three Python entry points:
 *
 *   run_lloyd(data, k, *, init, init_method, t_max, ctx)          lloyd.py:145-182
 *   run_pruner(data, k, strategy, *, init, ..., t_max, ctx)       pruners.py:862-923
 *   run_engine(data, k, KnobConfig(index_mode="none", ...), ...)  engine.py:828-853
 *
 * Each of those loops over  assign -> changed -> refine -> sse -> record.
 * The functions below replace the bodies of that loop one phase at a time, so
 * a ctypes binding (paper_2010_06654_b200/_native.py) can
 * drive it from the reference's own Python signatures:
 *
 *   lk_step_assign   replaces assign_full (lloyd.py:69-75) for Lloyd and
 *                    SequentialStrategy.seed / update_bounds / assign_pass
 *                    (pruners.py:83-87, :234-264 Hamerly, :418-497 Yinyang,
 *                    :128-174 Elkan) for the bounded strategies, plus the
 *                    changed count (lloyd.py:165 / pruners.py:903) and the
 *                    member-sum deltas that refine_full (lloyd.py:78-97) needs.
 *   lk_step_update   replaces the divide of refine_full (lloyd.py:94-96), the
 *                    centroid drifts (bounds.py:31-35), inter-centroid half
 *                    distances (bounds.py:38-47) and sse (core.py:172-179).
 *
 * Conventions (mirroring SPEC.md:104-109, one RunContext per run, single
 * writer): every call is stream-ordered on the caller's cudaStream_t, returns
 * an lk_status, never throws, and is NOT thread-safe on one context.  All
 * device memory lives in ONE caller-owned workspace (a torch uint8 tensor in
 * the Python host); lk_buffer() reports where each named buffer sits in it.
 * Points are bound once; centroids, labels and bounds stay resident in HBM.
 *
 * Multi-GPU (one process per GPU): rows are sharded, each rank has its own
 * context over its n_local rows, and the int64 delta buffer (LK_BUF_DELTA) is
 * summed across ranks (NCCL all-reduce) between lk_step_assign and
 * lk_step_update.  The sums are fixed-point integers, so the reduction is
 * exact and every rank computes bit-identical centroids.
 */
#ifndef LLOYDKIT_B200_H
#define LLOYDKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Every symbol declared here is exported even under -fvisibility=hidden. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
    LK_OK = 0,
    LK_ERR_ARG = 1,      /* bad argument; maps to ContractError / ValueError */
    LK_ERR_CUDA = 2,     /* CUDA runtime error; maps to RuntimeError */
    LK_ERR_STATE = 3,    /* call out of order (e.g. step before bind) */
    LK_ERR_UNSUPPORTED = 4
} lk_status;

/* Strategy ids (names of pruners.py:853-859 STRATEGIES that run on the GPU). */
typedef enum {
    LK_STRAT_LLOYD = 0,    /* run_lloyd: full n*k scan every iteration */
    LK_STRAT_HAMERLY = 1,  /* one upper + one global lower bound per point */
    LK_STRAT_YINYANG = 2,  /* upper bound + t group lower bounds per point */
    LK_STRAT_ELKAN = 3,    /* one lower bound per centroid while n_local * k <= 2^26
                              (SIMT); group bounds above that */
    LK_STRAT_REGROUP = 4   /* Yinyang with the group map rebuilt after every centroid update
                              and the bounds remapped (<= 32 groups) */
} lk_strategy;

/* Assignment-kernel selection. */
typedef enum {
    LK_KERNEL_AUTO = 0,    /* tcgen05 for d >= 32, SIMT otherwise */
    LK_KERNEL_SIMT = 1,    /* fp32 difference form on the CUDA cores */
    LK_KERNEL_TC = 2       /* tcgen05 3xTF32 dot-product form */
} lk_kernel;

typedef struct {
    int64_t n_local;       /* rows bound on this rank */
    int64_t n_total;       /* rows over all ranks (sizes the fixed-point scale) */
    int32_t d;
    int32_t k;
    int32_t strategy;      /* lk_strategy */
    int32_t groups;        /* Yinyang group count t (ignored otherwise) */
    int32_t t_max;         /* iterations that get a stats slot */
    int32_t kernel;        /* lk_kernel */
    int32_t has_x64;       /* 1: an fp64 copy of X is bound (input not fp32-exact) */
    int32_t device;        /* CUDA device ordinal */
    int64_t history_cap;   /* label-history log entries (0: no history log) */
    int32_t ranks;         /* ranks sharing the rows (0 or 1: single process);
                              informational, every delta of an iteration is
                              produced by lk_step_assign, before the caller's
                              all-reduce */
    int32_t reserved;
} lk_config;

/* Named buffers inside the workspace (byte offsets via lk_buffer). */
typedef enum {
    LK_BUF_X32 = 0,        /* float  [n_local, ldx]  points, fp32 (caller fills) */
    LK_BUF_X64 = 1,        /* double [n_local, d]    points, fp64 (if has_x64) */
    LK_BUF_C64 = 2,        /* double [k, d]          centroids (master copy) */
    LK_BUF_LABELS = 3,     /* int32  [n_local]       current labels */
    LK_BUF_UB = 4,         /* float  [n_local]       upper bounds */
    LK_BUF_LB = 5,         /* float  [nlb, n_local]  lower bounds (group-major) */
    LK_BUF_DELTA = 6,      /* int64  [delta_len]     all-reduce payload; accumulated by
                              lk_step_assign, consumed and zeroed by lk_step_update */
    LK_BUF_STATS = 7,      /* int64  [t_max, LK_NSTAT] per-iteration counters */
    LK_BUF_SSE = 8,        /* double [t_max]         per-iteration SSE */
    LK_BUF_GROUP_OF = 9,   /* int32  [k]             centroid -> group */
    LK_BUF_COUNTS = 10,    /* int64  [k]             cluster sizes */
    LK_BUF_QEXP = 11,      /* int32  [d + 1]         fixed-point exponents */
    LK_BUF_HLOG = 12,      /* int32x2 [history_cap]  (row, new label) of every moved row */
    LK_BUF_HLOG_OFF = 13,  /* int64  [t_max + 1]     log offset of each iteration (-1 overflow) */
    LK_BUF_TSTAMP = 14,    /* uint64 [t_max + 1, 2]  device clock (ns, %globaltimer): [t][0] update
                              start, [t][1] update end of iteration t; [0][1] iteration 1's
                              start (assign phase t = [t][0] - [t-1][1], also under graph replay) */
    LK_NBUF = 15
} lk_buffer_id;

/* Per-iteration counters (LK_BUF_STATS rows). */
enum {
    LK_STAT_CHANGED = 0,   /* points whose label changed (lloyd.py:165) */
    LK_STAT_FLAGGED = 1,   /* rows re-decided by the exact fp64 recheck */
    LK_STAT_ACTIVE = 2,    /* rows whose first bound test failed (tightened) */
    LK_STAT_WORK = 3,      /* rows rescanned against all / some centroids */
    LK_STAT_DIST = 4,      /* point-centroid distances evaluated (dist_comps) */
    LK_STAT_BOUND_UPD = 5, /* bound values rewritten (bound_updates) */
    LK_STAT_CANDIDATE = 6, /* rows re-decided in fp64 over <= 3 certified candidates */
    LK_STAT_CHANGED_GLOBAL = 7, /* changed summed over all ranks (stop rule) */
    LK_STAT_OVERFLOW = 8,  /* ambiguous rows with > LK_MAX_CAND candidates (fp32 rescan) */
    LK_STAT_YWL = 9,       /* Yinyang rows that reached the per-group scan */
    LK_STAT_PAIRS = 10,    /* Yinyang (row, group) scans */
    LK_STAT_REGROUPED = 11, /* Regroup: 1 if the group map was rebuilt before this iteration */
    LK_NSTAT = 16
};

int32_t lk_version(void);

/* k-means++ seeding (init_kmeanspp, core.py:192-217): one D^2 update over n
 * device rows (x32 fp32 [n, ldx], or x64 fp64 [n, ldx] when non-null),
 *   d2[i] = first ? s_i : min(d2[i], s_i),  s_i = sum_z (x_iz - c_z)^2
 * in fp64 with numpy's pairwise association over d -- the same values as the
 * reference's np.sum((data - data[j]) ** 2, axis=1), so the host-side draws
 * (rng.choice(n, p=d2 / d2.sum())) are the reference's.  No context needed;
 * c and d2 are device pointers; stream-ordered. */
lk_status lk_d2_update(const float *x32, const double *x64, int64_t n, int32_t d, int64_t ldx,
                       const double *c, double *d2, int32_t first, void *stream);
/* Last error message of the calling thread ("" if none). */
const char *lk_last_error(void);

/* Workspace size for a configuration (bytes, 256-aligned buffers inside). */
lk_status lk_workspace_bytes(const lk_config *cfg, uint64_t *bytes);

typedef struct lk_ctx lk_ctx;

/* Create a context over a caller-allocated device workspace of >= the size
 * lk_workspace_bytes reported.  The workspace must stay alive until destroy. */
lk_status lk_ctx_create(lk_ctx **out, const lk_config *cfg, void *workspace, uint64_t bytes);
lk_status lk_ctx_destroy(lk_ctx *ctx);

/* Byte offset and size of a named buffer inside the workspace.  (ids 1000 / 1001 report two
 * internal buffers of the group-tile worklist to tools/tile_stats.py: a debug aid, not part of
 * the interface.) */
lk_status lk_buffer(const lk_ctx *ctx, int32_t id, uint64_t *offset, uint64_t *bytes);
/* Row stride (floats) of LK_BUF_X32 and the length of LK_BUF_DELTA (int64s). */
lk_status lk_layout(const lk_ctx *ctx, int64_t *ldx, int64_t *delta_len, int32_t *nlb);

/* Group count t of a group-bound strategy and the most members a group may
 * have (0: not a group strategy).  On the block-sparse tensor-core path
 * (d <= 32, k <= 4096) every group is one 128-column tile: t = ceil(k / 128),
 * capacity 128; lk_set_groups rejects a larger group. */
lk_status lk_group_shape(const lk_ctx *ctx, int32_t *groups, int32_t *capacity);

/* After the caller has filled X32 (and X64): compute the per-dimension
 * max-|x| exponents of the local rows into LK_BUF_QEXP (device).  Multi-GPU
 * callers all-reduce(max) that int32 buffer before lk_set_quant. */
lk_status lk_scan_points(lk_ctx *ctx, void *stream);
/* Freeze the fixed-point scales from LK_BUF_QEXP.  Must follow lk_scan_points. */
lk_status lk_set_quant(lk_ctx *ctx, void *stream);

/* Yinyang / Elkan / Regroup: centroid -> group map (host int32 [k], values in
 * [0, groups)); the grouping only affects pruning power, never labels
 * (bounds.py:175-196 group_centroids is one way to build it). */
lk_status lk_set_groups(lk_ctx *ctx, const int32_t *group_of, void *stream);

/* Initial centroids: fp64 [k, d] device array (copied into LK_BUF_C64).
 * Resets labels to -1 (lloyd.py:159), sums, counts and stats. */
lk_status lk_set_centroids(lk_ctx *ctx, const double *c64, void *stream);

/* Iteration t (1-based): assignment (full scan or bound-filtered), exact fp64
 * recheck of ambiguous rows, changed count and member-sum deltas into
 * LK_BUF_DELTA.  Once an earlier iteration converged, kernels are no-ops.
 * The iteration index the kernels use lives on the device (advanced by
 * lk_step_update), so the launches of any t >= 2 are identical and a CUDA
 * graph captured from one iteration replays every later one; t only selects
 * the first-iteration (full scan) path. */
lk_status lk_step_assign(lk_ctx *ctx, int32_t t, void *stream);
/* Iteration t: apply the (reduced) deltas and zero them, new centroids (empty clusters keep
 * theirs), drifts, bound tables, SSE into LK_BUF_SSE[t-1], done flag. */
lk_status lk_step_update(lk_ctx *ctx, int32_t t, void *stream);

/* CUDA graph of one iteration t >= 2 (lk_step_assign + lk_step_update),
 * captured natively on a context-owned stream (the caller's stream may be the
 * legacy default stream, which cannot be captured; `stream` is unused) and
 * owned by the context; lk_graph_replay launches it on the caller's stream;
 * replays
 * are valid for every later iteration because the iteration index is
 * device-resident.  Single-process only (no collective inside). */
lk_status lk_graph_capture(lk_ctx *ctx, int32_t t, void *stream);
lk_status lk_graph_replay(lk_ctx *ctx, void *stream);

/* Debug shadow check of the stored bounds (validate_bounds, bounds.py:280-328;
 * run_pruner calls it when ctx.debug_validate, pruners.py:896-902): every
 * row's ub / global lower bound / group lower bounds against the exact fp64
 * distances to the current centroids, tolerance 1e-8 + 1e-9 |ref|.
 * decayed = 1: after lk_step_update (bounds decayed by the centroid drift, the
 * "iter{t}:decayed" point); 0: after lk_step_assign ("iter{t}:post").
 * out[0] = worst ub overshoot, out[1] = worst global lower-bound overshoot,
 * out[2 + g] = worst overshoot of group g (0: no violation); nout >= 2 + the
 * group count.  O(n k d) fp64 work; synchronizes the stream. */
lk_status lk_validate_bounds(lk_ctx *ctx, int32_t decayed, double *out, int32_t nout, void *stream);

/* Number of kernel launches issued by this context so far. */
int64_t lk_launch_count(const lk_ctx *ctx);

/* Timing helper for bench.py: total device time (ms) of the kernels of one
 * class recorded with events since the last reset (class: 0 assign/rescan,
 * 1 bound filter, 2 fp64 full recheck, 3 refine, 4 update, 5 group scans,
 * 6 group merge, 7 tensor-core candidate collection, 8 fp64 candidate
 * recheck, 9 fp32 rescan of candidate overflow).  Recording is enabled by
 * lk_profile(ctx, 1). */
lk_status lk_profile(lk_ctx *ctx, int32_t enable);
lk_status lk_profile_read(lk_ctx *ctx, int32_t cls, double *total_ms, int64_t *launches);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* LLOYDKIT_B200_H */
