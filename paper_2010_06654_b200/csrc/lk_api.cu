// lk_api.cu -- the extern "C" boundary declared in include/lloydkit_b200.h.
//
// A context owns no device memory of its own: every buffer is carved out of
// the caller's workspace at fixed, 256-byte aligned offsets, so the Python
// host (torch) accounts for all of HBM and can view any buffer as a tensor.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <stdlib.h>
#include <vector>

#include "lk_common.cuh"
#include "lk_internal.h"

namespace lkh {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

}  // namespace lkh

using lkh::set_error;

namespace {

enum InternalBuf {
    B_X32 = 0, B_X64, B_C64, B_LABELS, B_UB, B_LB, B_DELTA, B_STATS, B_SSE, B_GROUP_OF, B_COUNTS,
    B_QEXP, B_HLOG, B_HLOG_OFF, B_TSTAMP, B_CUR,
    // internal
    B_C64_PREV, B_C32, B_CNORM, B_DRIFT, B_SHALF, B_GDRIFT, B_SCAL, B_MOVED, B_FLAGGED, B_WORK,
    B_SUMS, B_QSUM, B_QSCALE, B_QINV, B_XSHIFT, B_DONE, B_SSE_PART, B_PW_PROG,
    B_XLO, B_XN2, B_CHI, B_CLO, B_CN2, B_XG_HI, B_XG_LO, B_CAND_ROWS, B_CAND_THR, B_CAND_LB, B_CAND_SLOTS, B_CAND_CNT, B_OVF,
    B_GPERM, B_GOFF, B_YWL, B_YPAIRS, B_YRES, B_GINV, B_CG, B_YLUN, B_YAUX, B_YPAIRS4, B_YBUCKET,
    B_SELF, B_DCUM, B_DGCUM, B_GLB, B_PTAB, B_PERM, B_LCUR, B_TILE_LAB, B_ROWR, B_ROWXO, B_ROWBV, B_ROWXN2, B_ROWLAB,
    B_YMASK, B_PMASK, B_SHIST, B_TMETA, B_VALID, B_CCH, B_RGSCR, B_RGMEANS, B_DCUMCOL,
    B_WORK2, B_YMASK2, B_YLUN2, B_GFREQ, B_GSEL, B_BHIST, B_BBASE, B_PINFO, B_COUNT_
};

struct Layout {
    uint64_t off[B_COUNT_];
    uint64_t size[B_COUNT_];
    uint64_t total;
    int64_t ldx, ldc, delta_len, pair_cap, bucket_cap;
    int32_t nlb, groups;
};

static bool is_group_strategy(int s);
static bool is_group_strategy(int s) {
    return s == LK_STRAT_YINYANG || s == LK_STRAT_ELKAN || s == LK_STRAT_REGROUP;
}

static uint64_t align256(uint64_t v) { return (v + 255) & ~uint64_t(255); }

static bool is_group_strategy(int s);
static bool tc_enabled(const lk_config& c);

// Elkan's per-centroid bounds (lk_elkan.cu) while the n x k bound table stays
// small (n * k <= 2^26: 256 MB); larger runs keep the grouped bounds.
// LK_ELKAN=0 (A/B knob) keeps the grouped path.
static bool elkan_mode(const lk_config& c) {
    static const int knob = [] {
        const char* e = getenv("LK_ELKAN");
        return e ? atoi(e) : 1;
    }();
    return knob != 0 && c.strategy == LK_STRAT_ELKAN && (int64_t)c.n_local * c.k <= (1LL << 26);
}

// the strategies that keep group bounds (lk_set_groups required)
static bool group_mode(const lk_config& c) { return is_group_strategy(c.strategy) && !elkan_mode(c); }

// Block-sparse Yinyang on the tensor cores (lk_tgy.cu): d <= 32 (one K chunk),
// groups = 128-column tiles of the B operand, at most 32 of them (k <= 4096).
// LK_TGY=0 (A/B knob) keeps the full-rescan tensor-core path.
static bool tgy_mode(const lk_config& c) {
    static const int knob = [] {
        const char* e = getenv("LK_TGY");
        return e ? atoi(e) : 1;
    }();
    const int G = (c.k + 127) / 128;
    // (Regroup rebuilds its groups every iteration; the tiles are fixed 128-column groups)
    return knob != 0 && is_group_strategy(c.strategy) && c.strategy != LK_STRAT_REGROUP &&
           tc_enabled(c) && c.d >= 8 && c.d <= 32 && G <= 32;
}

static int32_t nlb_for(const lk_config& c, int32_t* groups) {
    int32_t g = 1;
    switch (c.strategy) {
        case LK_STRAT_LLOYD: g = 0; break;
        case LK_STRAT_HAMERLY: g = 1; break;
        case LK_STRAT_ELKAN: g = c.groups > 0 ? c.groups : c.k; break;
        default: g = c.groups > 0 ? c.groups : (c.k + 9) / 10; break;
    }
    if (g > c.k) g = c.k;
    if (elkan_mode(c)) {
        *groups = 0;  // one bound per centroid, group-major [k, n]
        return c.k;
    }
    if (tgy_mode(c)) {
        // one group per 128-column tile; the row-major bound table is padded to
        // whole float4 loads (slots >= groups are never read)
        *groups = (c.k + 127) / 128;
        return (*groups + 3) / 4 * 4;
    }
    // the warp-per-row Yinyang path works on 8/16/32 group slots; extra slots
    // are empty groups (no members, never binding)
    if (group_mode(c) && g <= 32 && c.d <= 32)
        g = g <= 4 ? 4 : (g <= 8 ? 8 : (g <= 16 ? 16 : 32));
    *groups = g;
    return g < 1 ? 1 : g;
}

static bool tc_enabled(const lk_config& c) {
    if (elkan_mode(c)) return false;  // Elkan's per-centroid loop is SIMT
    return c.kernel == LK_KERNEL_TC || (c.kernel == LK_KERNEL_AUTO && c.d >= 32);
}

static bool make_layout(const lk_config& c, Layout* L) {
    if (c.n_local < 0 || c.d < 1 || c.k < 1 || c.t_max < 0 || c.n_total < c.n_local ||
        c.history_cap < 0)
        return false;
    if (c.n_local > 0x7fffffffLL) return false;  // row ids are int32 on device
    // k itself is unbounded (any 1 <= k <= n, core.py:186-187); the group
    // strategies pack (group, member position) into 16 + 16 bits, checked
    // per group in lk_set_groups
    if (is_group_strategy(c.strategy) && c.groups > 65535) return false;
    memset(L, 0, sizeof(*L));
    L->ldx = (c.d <= 2) ? c.d : ((c.d + 3) / 4) * 4;
    L->ldc = ((c.d + 3) / 4) * 4;
    L->nlb = nlb_for(c, &L->groups);
    L->delta_len = (int64_t)c.k * c.d + 2 * (int64_t)c.k + 8;
    const int64_t n = c.n_local, k = c.k, d = c.d;
    const int64_t tm = c.t_max > 0 ? c.t_max : 1;
    L->size[B_X32] = (uint64_t)n * L->ldx * 4;
    L->size[B_X64] = c.has_x64 ? (uint64_t)n * d * 8 : 0;
    L->size[B_C64] = (uint64_t)k * d * 8;
    L->size[B_LABELS] = (uint64_t)n * 4;
    L->size[B_UB] = c.strategy == LK_STRAT_LLOYD ? 0 : (uint64_t)n * 4;
    L->size[B_LB] = c.strategy == LK_STRAT_LLOYD ? 0 : (uint64_t)n * L->nlb * 4;
    L->size[B_DELTA] = (uint64_t)L->delta_len * 8;
    L->size[B_STATS] = (uint64_t)tm * LK_NSTAT * 8;
    L->size[B_SSE] = (uint64_t)tm * 8;
    L->size[B_GROUP_OF] = (uint64_t)k * 4;
    L->size[B_COUNTS] = (uint64_t)k * 8;
    L->size[B_QEXP] = (uint64_t)(3 * d + 1) * 4;
    L->size[B_HLOG] = c.history_cap > 0 ? (uint64_t)c.history_cap * 8 : 0;
    L->size[B_HLOG_OFF] = (uint64_t)(tm + 1) * 8;
    L->size[B_CUR] = (uint64_t)LK_NSTAT * 8;
    L->size[B_TSTAMP] = (uint64_t)(tm + 1) * 2 * 8;
    L->size[B_C64_PREV] = (uint64_t)k * d * 8;
    L->size[B_C32] = (uint64_t)k * L->ldc * 4;
    L->size[B_CNORM] = (uint64_t)k * 4;
    L->size[B_DRIFT] = (uint64_t)k * 4;
    L->size[B_SHALF] = (uint64_t)k * 4;
    L->size[B_GDRIFT] = (uint64_t)(L->groups > 0 ? L->groups : 1) * 4;
    L->size[B_SCAL] = 8 * 4;
    L->size[B_MOVED] = (uint64_t)n * 8;
    L->size[B_FLAGGED] = (uint64_t)n * 4;
    L->size[B_WORK] = c.strategy == LK_STRAT_LLOYD ? 0 : (uint64_t)n * 4;
    L->size[B_SUMS] = (uint64_t)k * d * 8;
    L->size[B_QSUM] = (uint64_t)k * 8;
    L->size[B_QSCALE] = (uint64_t)(d + 1) * 8;
    L->size[B_QINV] = (uint64_t)(d + 1) * 8;
    L->size[B_XSHIFT] = (uint64_t)d * 8;
    L->size[B_DONE] = 16;
    L->size[B_SSE_PART] = (uint64_t)k * 8;
    L->size[B_PW_PROG] = 4096 * 4;
    if (tc_enabled(c) && L->ldx % 4 == 0) {
        const int64_t kpad = (k + 255) / 256 * 256;
        L->size[B_XLO] = (uint64_t)n * L->ldx * 4;
        L->size[B_XN2] = (uint64_t)n * 4;
        L->size[B_CHI] = (uint64_t)kpad * L->ldc * 4;
        L->size[B_CLO] = (uint64_t)kpad * L->ldc * 4;
        L->size[B_CN2] = (uint64_t)kpad * 4;
        L->size[B_CAND_ROWS] = (uint64_t)n * 4;
        L->size[B_CAND_THR] = (uint64_t)n * 4;
        L->size[B_CAND_LB] = (uint64_t)n * 4;
        L->size[B_CAND_SLOTS] = (uint64_t)n * 4 * LK_MAX_CAND;
        L->size[B_CAND_CNT] = (uint64_t)n * 4;
        L->size[B_OVF] = (uint64_t)n * 4;
        L->size[B_XG_HI] = (uint64_t)n * L->ldx * 4;
        L->size[B_XG_LO] = (uint64_t)n * L->ldx * 4;
        // tile centering (rows sorted by label, tiles shifted by a centroid)
        L->size[B_PTAB] = (uint64_t)k * kpad * 4;
        L->size[B_PERM] = (uint64_t)n * 4;
        L->size[B_LCUR] = (uint64_t)(kpad + 1) * 4;  // (sort keys: B columns on the group-tile path)
        L->size[B_TILE_LAB] = (uint64_t)(n / 128 + 2) * 4;
        L->size[B_ROWR] = (uint64_t)n * 8;
        L->size[B_ROWXO] = (uint64_t)n * 4;
        L->size[B_ROWBV] = (uint64_t)n * 4;
        L->size[B_ROWXN2] = (uint64_t)n * 4;
        L->size[B_ROWLAB] = (uint64_t)n * 4;

    }
    if (tgy_mode(c)) {
        const int64_t kpad = (k + 255) / 256 * 256;
        L->size[B_GPERM] = (uint64_t)kpad * 4;     // column -> centroid (-1: padding)
        L->size[B_GOFF] = (uint64_t)(L->groups + 1) * 4;
        L->size[B_GINV] = (uint64_t)k * 4;         // centroid -> column
        L->size[B_YLUN] = (uint64_t)n * 8;
        L->size[B_YMASK] = (uint64_t)n * 4;
        L->size[B_TMETA] = (uint64_t)n * sizeof(lk::TgyMeta);
        L->size[B_PMASK] = (uint64_t)(n / 128 + 4) * 4;  // per 128-row tile
        L->size[B_SHIST] = (uint64_t)1536 * kpad * 4;  // (<= 1536 sort blocks)
        L->size[B_WORK2] = (uint64_t)n * 4;
        L->size[B_YMASK2] = (uint64_t)n * 4;
        L->size[B_YLUN2] = (uint64_t)n * 8;
        L->size[B_GFREQ] = (uint64_t)k * 32 * 4;
        L->size[B_GSEL] = (uint64_t)k * 4;
        L->size[B_BHIST] = (uint64_t)1536 * 64 * 4;
        L->size[B_BBASE] = 64 * 4;
        L->size[B_PINFO] = (uint64_t)(n / 256 + 2) * 16;
        L->size[B_DCUM] = (uint64_t)k * 4;
        L->size[B_DCUMCOL] = (uint64_t)kpad * 4;
        L->size[B_DGCUM] = (uint64_t)L->groups * 4;
        L->size[B_GLB] = (uint64_t)n * 4;
    } else if (group_mode(c)) {
        int64_t cap = n * (int64_t)L->groups;
        if (cap > (1LL << 30)) cap = 1LL << 30;  // result slots, <= 16 GB
        if (cap < 1) cap = 1;
        L->pair_cap = cap;
        L->size[B_GPERM] = (uint64_t)k * 4;
        L->size[B_GOFF] = (uint64_t)(L->groups + 1) * 4;
        L->size[B_YWL] = (uint64_t)n * 16;
        L->size[B_YPAIRS] = (uint64_t)cap * 8;
        L->size[B_YRES] = (uint64_t)cap * 16;
        L->size[B_GINV] = (uint64_t)k * 4;
        L->size[B_CG] = (uint64_t)k * L->ldc * 4;
        L->size[B_YLUN] = (uint64_t)n * 8;
        L->size[B_YAUX] = (uint64_t)n * 8;
        // group buckets: one slot per row per group (capped); overflow -> full rescan
        int64_t bcap = n;
        if (bcap * L->groups > (1LL << 31)) bcap = (1LL << 31) / L->groups;  // <= 16 GB
        if (bcap < 1) bcap = 1;
        L->bucket_cap = bcap;
        L->size[B_YPAIRS4] = (uint64_t)bcap * L->groups * 8;
        L->size[B_YBUCKET] = (uint64_t)(L->groups + 1) * 8;
        if (L->groups <= 32 && c.d <= 32 && !tc_enabled(c)) {
            // lazy (drift-offset) bounds of the fused path (SIMT group scans;
            // tensor-core runs rescan failing rows in full instead)
            L->size[B_DCUM] = (uint64_t)k * 4;
            L->size[B_DGCUM] = (uint64_t)L->groups * 4;
            L->size[B_GLB] = (uint64_t)n * 4;
        }
    }
    if (c.strategy == LK_STRAT_REGROUP && group_mode(c)) {
        L->size[B_RGSCR] = (uint64_t)(33 + k) * 4;
        L->size[B_RGMEANS] = (uint64_t)(L->groups > 0 ? L->groups : 1) * d * 8;
    }
    if (elkan_mode(c)) L->size[B_CCH] = (uint64_t)k * k * 4;  // half inter-centroid distances
    L->size[B_VALID] = (uint64_t)(2 + (L->groups > 0 ? L->groups : 1)) * 8;  // validator output
    L->size[B_SELF] = sizeof(lk::DevState);
    uint64_t off = 0;
    for (int b = 0; b < B_COUNT_; b++) {
        L->off[b] = off;
        off = align256(off + L->size[b]);
    }
    L->total = off;
    return true;
}

// numpy pairwise_sum association tree for a length-d reduction, as a postfix
// program: (0, start, len) = leaf, (1, 0, 0) = add the two top values.
static void build_pw(int start, int n, std::vector<int32_t>& prog) {
    if (n <= 128) {
        prog.push_back(0);
        prog.push_back(start);
        prog.push_back(n);
        return;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    build_pw(start, n2, prog);
    build_pw(start + n2, n - n2, prog);
    prog.push_back(1);
    prog.push_back(0);
    prog.push_back(0);
}

}  // namespace

struct lk_ctx {
    lk_config cfg;
    Layout L;
    uint8_t* ws;
    lk::DevState S;
    int sms;
    bool quant_set;
    bool centroids_set;
    bool groups_set;
    int64_t launches;
    // one-iteration CUDA graph (lk_graph_capture)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    // capture happens on a context-owned stream: the caller's stream may be
    // the legacy default stream, which cannot be captured
    cudaStream_t cap_stream = nullptr;
    // profiling
    bool profile;
    struct Rec { int cls; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
};

namespace {

template <typename T>
T* buf(lk_ctx* c, int b) {
    return c->L.size[b] ? reinterpret_cast<T*>(c->ws + c->L.off[b]) : nullptr;
}

cudaEvent_t take_event(lk_ctx* c) {
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    lk_ctx* c;
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(lk_ctx* c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
        if (c->profile) {
            a = take_event(c);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (c->profile) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, st);
            c->recs.push_back({cls, a, b});
        }
    }
};

}  // namespace

extern "C" {

int32_t lk_version(void) { return 1; }

lk_status lk_d2_update(const float* x32, const double* x64, int64_t n, int32_t d, int64_t ldx,
                       const double* c, double* d2, int32_t first, void* stream) {
    if ((!x32 && !x64) || !c || !d2 || n < 0 || d < 1 || ldx < d) {
        set_error("lk_d2_update: bad arguments");
        return LK_ERR_ARG;
    }
    std::vector<int32_t> prog;
    build_pw(0, d, prog);
    lk::PwProg pp;
    if (prog.size() > sizeof(pp.ops) / sizeof(pp.ops[0])) {
        set_error("lk_d2_update: d=%d too large for the pairwise program", d);
        return LK_ERR_UNSUPPORTED;
    }
    pp.len = (int32_t)prog.size();
    for (size_t i = 0; i < prog.size(); i++) pp.ops[i] = prog[i];
    return lkh::launch_d2_update(x32, x64, n, d, ldx, c, d2, first, pp, (cudaStream_t)stream);
}

const char* lk_last_error(void) { return lkh::g_err; }

lk_status lk_workspace_bytes(const lk_config* cfg, uint64_t* bytes) {
    if (!cfg || !bytes) return LK_ERR_ARG;
    Layout L;
    if (!make_layout(*cfg, &L)) {
        set_error("invalid configuration");
        return LK_ERR_ARG;
    }
    *bytes = L.total;
    return LK_OK;
}

lk_status lk_ctx_create(lk_ctx** out, const lk_config* cfg, void* workspace, uint64_t bytes) {
    if (!out || !cfg || !workspace) {
        set_error("null argument");
        return LK_ERR_ARG;
    }
    if (cfg->strategy < LK_STRAT_LLOYD || cfg->strategy > LK_STRAT_REGROUP) {
        set_error("unknown strategy id %d", cfg->strategy);
        return LK_ERR_ARG;
    }
    Layout L;
    if (!make_layout(*cfg, &L)) {
        set_error("invalid configuration (n=%lld d=%d k=%d)", (long long)cfg->n_local, cfg->d,
                  cfg->k);
        return LK_ERR_ARG;
    }
    if (bytes < L.total) {
        set_error("workspace too small: %llu < %llu", (unsigned long long)bytes,
                  (unsigned long long)L.total);
        return LK_ERR_ARG;
    }
    LK_CUDA_CHECK(cudaSetDevice(cfg->device));
    lk_ctx* c = new lk_ctx();
    c->cfg = *cfg;
    c->L = L;
    c->ws = reinterpret_cast<uint8_t*>(workspace);
    c->quant_set = false;
    c->centroids_set = false;
    c->groups_set = !group_mode(*cfg);
    c->launches = 0;
    c->profile = false;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
    c->sms = sms;

    lk::DevState& S = c->S;
    memset(&S, 0, sizeof(S));
    S.n = cfg->n_local;
    S.d = cfg->d;
    S.k = cfg->k;
    S.ldx = (int32_t)L.ldx;
    S.ldc = (int32_t)L.ldc;
    S.nlb = L.nlb;
    S.strategy = cfg->strategy;
    S.t_groups = L.groups;
    S.X32 = buf<float>(c, B_X32);
    S.X64 = buf<double>(c, B_X64);
    S.C64 = buf<double>(c, B_C64);
    S.C64_prev = buf<double>(c, B_C64_PREV);
    S.C32 = buf<float>(c, B_C32);
    S.cnorm = buf<float>(c, B_CNORM);
    S.drift = buf<float>(c, B_DRIFT);
    S.s_half = buf<float>(c, B_SHALF);
    S.gdrift = group_mode(*cfg) ? buf<float>(c, B_GDRIFT) : nullptr;  // (not Elkan's per-centroid bounds)
    S.scal = buf<float>(c, B_SCAL);
    S.group_of = buf<int32_t>(c, B_GROUP_OF);
    S.labels = buf<int32_t>(c, B_LABELS);
    S.ub = buf<float>(c, B_UB);
    S.lb = buf<float>(c, B_LB);
    S.moved = buf<int2>(c, B_MOVED);
    S.flagged = buf<int32_t>(c, B_FLAGGED);
    S.work = buf<int32_t>(c, B_WORK);
    S.delta = buf<int64_t>(c, B_DELTA);
    S.sums = buf<int64_t>(c, B_SUMS);
    S.counts = buf<int64_t>(c, B_COUNTS);
    S.qsum = buf<int64_t>(c, B_QSUM);
    S.qexp = buf<int32_t>(c, B_QEXP);
    S.xshift = buf<double>(c, B_XSHIFT);
    S.done = buf<int32_t>(c, B_DONE);
    S.iter = S.done + 1;
    S.cur = buf<int64_t>(c, B_CUR);
    S.t_max = cfg->t_max;
    S.hlog = buf<int2>(c, B_HLOG);
    S.hlog_off = buf<int64_t>(c, B_HLOG_OFF);
    S.tstamp = buf<uint64_t>(c, B_TSTAMP);
    S.hlog_cap = cfg->history_cap;
    S.stats = buf<int64_t>(c, B_STATS);
    S.sse = buf<double>(c, B_SSE);
    S.pw_prog = buf<int32_t>(c, B_PW_PROG);
    S.Xlo = buf<float>(c, B_XLO);
    S.xn2 = buf<float>(c, B_XN2);
    S.Chi = buf<float>(c, B_CHI);
    S.Clo = buf<float>(c, B_CLO);
    S.cn2 = buf<float>(c, B_CN2);
    S.Xg_hi = buf<float>(c, B_XG_HI);
    S.Xg_lo = buf<float>(c, B_XG_LO);
    S.ptab = buf<float>(c, B_PTAB);
    S.perm = buf<int32_t>(c, B_PERM);
    S.lcur = buf<int32_t>(c, B_LCUR);
    S.tile_lab = buf<int32_t>(c, B_TILE_LAB);
    S.rowR = buf<double>(c, B_ROWR);
    S.rowxo = buf<float>(c, B_ROWXO);
    S.rowbv = buf<float>(c, B_ROWBV);
    S.rowxn2 = buf<float>(c, B_ROWXN2);
    S.rowlab = buf<int32_t>(c, B_ROWLAB);
    S.kpad = (int32_t)((cfg->k + 255) / 256 * 256);
    {
        const char* e = getenv("LK_TC_CENTER");  // A/B knob for the tile centering
        // measured: pays at d <= 32 (one K chunk, resident A tiles; cfg5 138 -> 121
        // ms), not at d = 128 / 784 where few rows are ambiguous anyway
        S.center = (S.ptab != nullptr && (e ? atoi(e) != 0 : cfg->d <= 32)) ? 1 : 0;
    }
    S.cand_rows = buf<int32_t>(c, B_CAND_ROWS);
    S.cand_thr = buf<float>(c, B_CAND_THR);
    S.cand_lb = buf<float>(c, B_CAND_LB);
    S.cand_slots = buf<int32_t>(c, B_CAND_SLOTS);
    S.cand_cnt = buf<int32_t>(c, B_CAND_CNT);
    S.ovf = buf<int32_t>(c, B_OVF);
    S.gperm = buf<int32_t>(c, B_GPERM);
    S.goff = buf<int32_t>(c, B_GOFF);
    S.ywl = buf<int4>(c, B_YWL);
    S.ypairs = buf<int2>(c, B_YPAIRS);
    S.yres = buf<float4>(c, B_YRES);
    S.ginv = buf<int32_t>(c, B_GINV);
    S.Cg = buf<float>(c, B_CG);
    S.ylun = buf<float2>(c, B_YLUN);
    S.yaux = buf<int2>(c, B_YAUX);
    S.ypairs2 = buf<int2>(c, B_YPAIRS4);
    S.ybucket = buf<int64_t>(c, B_YBUCKET);
    S.bucket_cap = L.bucket_cap;
    S.pair_cap = L.pair_cap;

    std::vector<int32_t> prog;
    build_pw(0, cfg->d, prog);
    if (prog.size() > 4096) {
        delete c;
        set_error("pairwise program too long for d=%d", cfg->d);
        return LK_ERR_UNSUPPORTED;
    }
    S.pw_len = (int32_t)prog.size();
    LK_CUDA_CHECK(cudaMemcpy(S.pw_prog, prog.data(), prog.size() * 4, cudaMemcpyHostToDevice));
    LK_CUDA_CHECK(cudaMemset(S.done, 0, 16));
    S.lazy = L.size[B_GLB] > 0 ? 1 : 0;
    S.tgy = tgy_mode(*cfg) ? 1 : 0;
    S.elkan = elkan_mode(*cfg) ? 1 : 0;
    S.cch = buf<float>(c, B_CCH);
    S.kcols = S.tgy ? 128 * L.groups : cfg->k;
    S.colperm = S.tgy ? buf<int32_t>(c, B_GPERM) : nullptr;
    S.ymask = buf<uint32_t>(c, B_YMASK);
    S.pmask = buf<uint32_t>(c, B_PMASK);
    S.shist = buf<int32_t>(c, B_SHIST);
    S.tmeta = buf<lk::TgyMeta>(c, B_TMETA);
    S.work2 = buf<int32_t>(c, B_WORK2);
    S.ymask2 = buf<uint32_t>(c, B_YMASK2);
    S.ylun2 = buf<float2>(c, B_YLUN2);
    S.gfreq = buf<int32_t>(c, B_GFREQ);
    S.gsel = buf<uint32_t>(c, B_GSEL);
    S.bhist = buf<int32_t>(c, B_BHIST);
    S.bbase = buf<int32_t>(c, B_BBASE);
    S.pinfo = buf<int4>(c, B_PINFO);
    S.hlog_inline = (S.lazy && S.hlog != nullptr && S.hlog_cap > 0) ? 1 : 0;
    {
        const char* e = getenv("LK_SGATE");  // A/B knob for the centroid-separation gate
        S.sgate = e ? (atoi(e) != 0) : 1;
    }
    S.dcum = buf<float>(c, B_DCUM);
    S.dcum_col = buf<float>(c, B_DCUMCOL);
    S.dgcum = buf<float>(c, B_DGCUM);
    S.glb = buf<float>(c, B_GLB);
    S.self = buf<lk::DevState>(c, B_SELF);
    LK_CUDA_CHECK(cudaMemcpy((void*)S.self, &S, sizeof(S), cudaMemcpyHostToDevice));
    // every kernel attribute is set here, never inside a (possibly captured) step
    lk_status as = lkh::init_simt_attributes();
    if (as == LK_OK && S.Xlo) as = lkh::init_tc_attributes();
    if (as == LK_OK && S.Cg) as = lkh::init_yy_attributes();
    if (as == LK_OK && S.Cg) as = lkh::init_fused_attributes();
    if (as != LK_OK) {
        delete c;
        return as;
    }
    *out = c;
    return LK_OK;
}

lk_status lk_ctx_destroy(lk_ctx* c) {
    if (!c) return LK_OK;
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    if (c->graph) cudaGraphDestroy(c->graph);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    for (auto& r : c->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->pool) cudaEventDestroy(e);
    delete c;
    return LK_OK;
}

lk_status lk_buffer(const lk_ctx* c, int32_t id, uint64_t* offset, uint64_t* bytes) {
    // (debug tools: 1000 the group-tile worklist records, 1001 the tile labels;
    // internal layout, not part of the interface)
    if (c && (id == 1000 || id == 1001)) id = id == 1000 ? B_TMETA : B_TILE_LAB;
    else
    if (!c || id < 0 || id >= LK_NBUF) {
        set_error("bad buffer id %d", id);
        return LK_ERR_ARG;
    }
    if (offset) *offset = c->L.off[id];
    if (bytes) *bytes = c->L.size[id];
    return LK_OK;
}

lk_status lk_group_shape(const lk_ctx* c, int32_t* groups, int32_t* capacity) {
    if (!c) return LK_ERR_ARG;
    if (groups) *groups = c->L.groups;
    // (Elkan's per-centroid bounds: k singleton groups, capacity 1; no lk_set_groups)
    if (groups && c->S.elkan) *groups = c->cfg.k;
    if (capacity) *capacity = c->S.elkan ? 1 : c->S.tgy ? 128 : (group_mode(c->cfg) ? 32767 : 0);
    return LK_OK;
}

lk_status lk_layout(const lk_ctx* c, int64_t* ldx, int64_t* delta_len, int32_t* nlb) {
    if (!c) return LK_ERR_ARG;
    if (ldx) *ldx = c->L.ldx;
    if (delta_len) *delta_len = c->L.delta_len;
    if (nlb) *nlb = c->L.nlb;
    return LK_OK;
}

static __global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

lk_status lk_scan_points(lk_ctx* c, void* stream) {
    if (!c) return LK_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    k_fill_i32<<<1, 256, 0, st>>>(c->S.qexp, 3 * (int64_t)c->cfg.d + 1, INT32_MIN);
    LK_LAUNCH_CHECK();
    c->launches += 2;
    lk_status s = lkh::launch_scan_exp(c->S, c->sms, st);
    if (s != LK_OK) return s;
    if (c->S.Xlo) {
        c->launches += 1;
        return lkh::launch_tc_prep_points(c->S, c->sms, st);
    }
    return LK_OK;
}

// Fixed-point scales from the scanned ranges, on the device (no host round
// trip).  Per dimension the shift m_z is the middle of [min x_z, max x_z] and
// r_z >= |x_z - m_z| its half range; the scale is 2^(B - e_z) with
// 2^e_z > r_z, B = 62 - ceil(log2(n_total + 1)), so a sum of n_total
// quantized values stays below 2^62; qexp[d] covers
// ||x - m||^2 <= sum_z r_z^2.
__device__ __forceinline__ float unkey(int k) { return __int_as_float(k >= 0 ? k : (k ^ 0x7fffffff)); }

__device__ __forceinline__ void range_of(const int32_t* qexp, int d, int z, double* m, double* r) {
    const int kh = qexp[d + 1 + z], kl = qexp[2 * d + 1 + z];
    if (kh == INT32_MIN || kl == INT32_MIN) {  // no rows anywhere
        *m = 0.0;
        *r = 0.0;
        return;
    }
    const double hi = (double)unkey(kh), lo = -(double)unkey(kl);
    const double mm = 0.5 * hi + 0.5 * lo;
    *m = mm;
    *r = fmax(hi - mm, mm - lo) * (1.0 + 1e-12);
}

static __global__ void k_set_quant(int32_t* qexp, double* qscale, double* qinv, double* xshift, int d,
                                   int B) {
    for (int z = threadIdx.x; z < d; z += blockDim.x) {
        double m, r;
        range_of(qexp, d, z, &m, &r);
        int ez = 0;
        if (r > 0.0) frexp(r, &ez);
        xshift[z] = m;
        qexp[z] = ez;
        qscale[z] = ldexp(1.0, B - ez);
        qinv[z] = ldexp(1.0, ez - B);
    }
    if (threadIdx.x == 0) {
        double r2 = 0.0;
        for (int z = 0; z < d; z++) {
            double m, r;
            range_of(qexp, d, z, &m, &r);
            r2 = fma(r, r, r2);
        }
        int e2 = 0;
        if (r2 > 0.0) frexp(r2 * (1.0 + 1e-9), &e2);
        qexp[d] = e2;
        qscale[d] = ldexp(1.0, B - e2);
        qinv[d] = ldexp(1.0, e2 - B);
    }
}

lk_status lk_set_quant(lk_ctx* c, void* stream) {
    if (!c) return LK_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int d = c->cfg.d;
    // Sum of n_total values each < 2^B in magnitude must stay below 2^62.
    int lg = 0;
    while ((1LL << lg) <= c->cfg.n_total) lg++;
    const int B = 62 - lg;
    k_set_quant<<<1, 128, 0, st>>>(c->S.qexp, buf<double>(c, B_QSCALE), buf<double>(c, B_QINV),
                                   c->S.xshift, d, B);
    LK_LAUNCH_CHECK();
    c->launches += 1;
    c->quant_set = true;
    return LK_OK;
}

static __global__ void k_init_centroids(lk::DevState S, int kpad) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x / 32) + warp;
    if (S.colperm && j < kpad && S.colperm[j] < 0) {
        // a padding column of the group tiles: never a candidate
        if (lane == 0) S.cn2[j] = INFINITY;
        for (int z = lane; z < S.ldc; z += 32) {
            S.Chi[(int64_t)j * S.ldc + z] = 0.f;
            S.Clo[(int64_t)j * S.ldc + z] = 0.f;
        }
    }
    if (j >= S.k) {
        if (!S.colperm && j < kpad && S.cn2 && lane == 0) S.cn2[j] = INFINITY;
        return;
    }
    // B-operand column of centroid j (group order on the group-tile path)
    const int64_t cj = S.colperm ? S.ginv[j] : j;
    double cn2 = 0.0, c2 = 0.0;
    for (int z = lane; z < S.ldc; z += 32) {
        double c = z < S.d ? S.C64[(int64_t)j * S.d + z] : 0.0;
        float v = (float)c;
        S.C32[(int64_t)j * S.ldc + z] = v;
        if (S.Cg) S.Cg[(int64_t)S.ginv[j] * S.ldc + z] = v;
        if (z < S.d) S.C64_prev[(int64_t)j * S.d + z] = c;
        cn2 = fma((double)v, (double)v, cn2);
        c2 = fma(c, c, c2);
        if (S.Chi) {
            float hi = lk::tf32_trunc(v);
            S.Chi[cj * S.ldc + z] = hi;
            S.Clo[cj * S.ldc + z] = v - hi;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        cn2 += __shfl_xor_sync(LK_FULL_MASK, cn2, o);
        c2 += __shfl_xor_sync(LK_FULL_MASK, c2, o);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *S.iter = 1;
    if (lane == 0) {
        if (S.cn2) S.cn2[cj] = (float)c2;
        float cn = __double2float_ru(sqrt(cn2) * (1.0 + 1e-12));
        S.cnorm[j] = cn;
        S.drift[j] = 0.f;
        S.s_half[j] = 0.f;
        lk::atomic_max_pos(S.scal, cn);
    }
}

lk_status lk_set_groups(lk_ctx* c, const int32_t* group_of, void* stream) {
    if (!c || !group_of) return LK_ERR_ARG;
    if (!group_mode(c->cfg)) {
        set_error("lk_set_groups: strategy %d keeps no group bounds", c->cfg.strategy);
        return LK_ERR_STATE;
    }
    const int k = c->cfg.k, t = c->L.groups;
    const int cap = c->S.tgy ? 128 : 32767;  // group-tile path: one 128-column tile per group
    std::vector<int32_t> cnt(t + 1, 0), perm(k), off(t + 1, 0);
    for (int j = 0; j < k; j++) {
        if (group_of[j] < 0 || group_of[j] >= t) {
            set_error("group_of[%d] = %d outside [0, %d)", j, group_of[j], t);
            return LK_ERR_ARG;
        }
        cnt[group_of[j]]++;
    }
    for (int g = 0; g < t; g++) {
        if (cnt[g] > cap) {
            set_error("lk_set_groups: group %d has %d members (at most %d)", g, cnt[g], cap);
            return LK_ERR_ARG;
        }
        off[g + 1] = c->S.tgy ? 128 * (g + 1) : off[g] + cnt[g];
    }
    std::vector<int32_t> fill(off.begin(), off.end()), inv(k);
    if (c->S.tgy) perm.assign((size_t)c->S.kpad, -1);  // column -> centroid, padding -1
    for (int j = 0; j < k; j++) {
        inv[j] = fill[group_of[j]];
        perm[fill[group_of[j]]++] = j;  // ascending j within a group
    }
    cudaStream_t st = (cudaStream_t)stream;
    LK_CUDA_CHECK(cudaMemcpyAsync(c->S.group_of, group_of, k * 4, cudaMemcpyHostToDevice, st));
    LK_CUDA_CHECK(cudaMemcpyAsync(c->S.gperm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, st));
    LK_CUDA_CHECK(cudaMemcpyAsync(c->S.goff, off.data(), (t + 1) * 4, cudaMemcpyHostToDevice, st));
    LK_CUDA_CHECK(cudaMemcpyAsync(c->S.ginv, inv.data(), k * 4, cudaMemcpyHostToDevice, st));
    LK_CUDA_CHECK(cudaStreamSynchronize(st));
    c->groups_set = true;
    return LK_OK;
}

lk_status lk_set_centroids(lk_ctx* c, const double* c64, void* stream) {
    if (!c || !c64) return LK_ERR_ARG;
    if (!c->groups_set) {
        set_error("lk_set_centroids: call lk_set_groups first for group-bound strategies");
        return LK_ERR_STATE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    lk::DevState& S = c->S;
    const int64_t k = c->cfg.k, d = c->cfg.d;
    if ((const void*)c64 != (const void*)S.C64)
        LK_CUDA_CHECK(cudaMemcpyAsync(S.C64, c64, k * d * 8, cudaMemcpyDeviceToDevice, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.scal, 0, 8 * 4, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.labels, 0xff, (size_t)c->cfg.n_local * 4, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.sums, 0, k * d * 8, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.counts, 0, k * 8, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.qsum, 0, k * 8, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.done, 0, 16, st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.stats, 0, c->L.size[B_STATS], st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.cur, 0, c->L.size[B_CUR], st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.hlog_off, 0, c->L.size[B_HLOG_OFF], st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.tstamp, 0xff, c->L.size[B_TSTAMP], st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.sse, 0, c->L.size[B_SSE], st));
    LK_CUDA_CHECK(cudaMemsetAsync(S.delta, 0, c->L.size[B_DELTA], st));
    if (S.tgy || S.elkan) LK_CUDA_CHECK(cudaMemsetAsync(S.lb, 0, c->L.size[B_LB], st));  // bounds >= 0
    if (S.dcum_col) LK_CUDA_CHECK(cudaMemsetAsync(S.dcum_col, 0, c->L.size[B_DCUMCOL], st));
    if (S.gsel) {
        // no bucket key before the first listing
        LK_CUDA_CHECK(cudaMemsetAsync(S.gsel, 0, c->L.size[B_GSEL], st));
        LK_CUDA_CHECK(cudaMemsetAsync(S.gfreq, 0, c->L.size[B_GFREQ], st));
    }
    if (S.lazy) {
        LK_CUDA_CHECK(cudaMemsetAsync(S.dcum, 0, c->L.size[B_DCUM], st));
        LK_CUDA_CHECK(cudaMemsetAsync(S.dgcum, 0, c->L.size[B_DGCUM], st));
    }
    const int kpad = (int)((k + 255) / 256 * 256);
    k_init_centroids<<<(kpad + 7) / 8, 256, 0, st>>>(S, kpad);
    LK_LAUNCH_CHECK();
    c->launches += 1;
    c->centroids_set = true;
    return LK_OK;
}

// Device-clock stamp of iteration 1's start (tstamp[0][1]); the update kernel
// stamps every iteration's update start / end (tstamp[t][0..1]), so the
// assign / refine split survives CUDA-graph replay.
static __global__ void k_stamp_start(lk::DevState S) {
    if (threadIdx.x == 0) {
        uint64_t g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        S.tstamp[1] = g;
    }
}

lk_status lk_step_assign(lk_ctx* c, int32_t t, void* stream) {
    if (!c) return LK_ERR_ARG;
    if (!c->quant_set || !c->centroids_set || !c->groups_set) {
        set_error("lk_step_assign before lk_set_quant / lk_set_centroids / lk_set_groups");
        return LK_ERR_STATE;
    }
    if (t < 1 || t > c->cfg.t_max) {
        set_error("iteration %d outside [1, %d]", t, c->cfg.t_max);
        return LK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    lk::DevState& S = c->S;
    int64_t* stat = S.cur;  // counters of the iteration in flight (copied out by the update)
    // the delta payload is zeroed by the update that consumes it (and at
    // lk_set_centroids); the bucket counters only by the multi-kernel path
    if (S.ybucket && !lkh::yy_fused_ok(S))
        LK_CUDA_CHECK(cudaMemsetAsync(S.ybucket, 0, c->L.size[B_YBUCKET], st));
    const int64_t n = c->cfg.n_local;
    const bool use_tc = lkh::tc_supported(S);
    lk_status s;
    if (t == 1) {
        // the iteration's start on the device clock (later iterations start
        // where the previous update ended: lk_step_update stamps it)
        k_stamp_start<<<1, 32, 0, st>>>(S);
        LK_LAUNCH_CHECK();
        c->launches += 1;
    }
    if (n > 0) {
        if (S.elkan) {
            // per-centroid bounds, every iteration (iteration 1 seeds them exactly)
            ProfScope p(c, 1, st);
            s = lkh::launch_elkan(S, stat, c->sms, st);
            if (s != LK_OK) return s;
            c->launches += 2;
        } else if (t == 1 && group_mode(c->cfg) && lkh::yy_masked(S) && !use_tc) {
            // group-order full scan that also seeds exact per-group bounds
            ProfScope p(c, 0, st);
            s = lkh::launch_yy_seed(S, stat, c->sms, st);
            if (s != LK_OK) return s;
            c->launches += 1;
        } else if (c->cfg.strategy == LK_STRAT_LLOYD || t == 1) {
            ProfScope p(c, 0, st);
            // iteration >= 2 on the tensor cores: label-sorted, centroid-shifted tiles
            s = (use_tc && t >= 2) ? lkh::launch_assign_tc_centered(S, nullptr, nullptr, stat, n,
                                                                     c->cfg.n_total == n, c->sms, st)
                : use_tc ? lkh::launch_assign_tc(S, nullptr, nullptr, stat, n, c->sms, st)
                         : lkh::launch_assign_simt(S, nullptr, nullptr, stat, n, c->sms, st);
            if (s != LK_OK) return s;
            c->launches += 1;
        } else if (S.tgy) {
            // block-sparse Yinyang on the tensor cores: filter -> label-sorted
            // worklist -> (row-tile pair x failing group tile) MMAs (lk_tgy.cu)
            {
                ProfScope p(c, 1, st);
                s = lkh::launch_filter_tgy(S, stat, c->sms, st);
                if (s != LK_OK) return s;
            }
            {
                ProfScope p(c, 10, st);
                s = lkh::launch_sort_tgy(S, stat, c->sms, st);
                if (s != LK_OK) return s;
            }
            ProfScope p(c, 0, st);
            s = lkh::launch_assign_tgy(S, stat, n, c->sms, st);
            if (s != LK_OK) return s;
            c->launches += lkh::tgy_bucket_on(S) ? 13 : 9;
        } else if (group_mode(c->cfg)) {
            // tensor-core runs: every row failing the bounds is rescanned in full
            const bool full_only = use_tc;
            if (lkh::yy_fused_ok(S)) {
                // one kernel: filter, group scans, certified merge, the fp64
                // recheck of the rows the merge leaves ambiguous, refinement
                // deltas (lk_yy_fused.cu)
                {
                    ProfScope p(c, 1, st);
                    s = lkh::launch_yy_fused(S, stat, buf<double>(c, B_QSCALE), c->sms, st);
                    if (s != LK_OK) return s;
                }
                c->launches += 1;
                if (S.hlog && !S.hlog_inline) {
                    ProfScope p(c, 3, st);
                    s = lkh::launch_log_history(S, c->sms, st);
                    if (s != LK_OK) return s;
                    c->launches += 1;
                }
                return LK_OK;
            } else {
            {
                ProfScope p(c, 1, st);
                s = lkh::launch_yy_filter(S, stat, c->sms, st, full_only);
                if (s != LK_OK) return s;
            }
            {
                ProfScope p(c, 5, st);
                s = lkh::launch_yy_pairs(S, stat, c->sms, st, full_only);
                if (s != LK_OK) return s;
            }
            {
                ProfScope p(c, 6, st);
                s = lkh::launch_yy_merge(S, stat, c->sms, st, full_only);
                if (s != LK_OK) return s;
            }
            ProfScope p(c, 0, st);
            // full rescans: capacity overflow, or every failing row when full_only
            s = (use_tc && !S.center) ? lkh::launch_assign_tc_adaptive(S, S.work, stat + LK_STAT_WORK, stat,
                                                                     n, c->sms, st)
                : use_tc ? lkh::launch_assign_tc_centered(S, S.work, stat + LK_STAT_WORK, stat, n,
                                                        false, c->sms, st)
                       : lkh::launch_assign_simt(S, S.work, stat + LK_STAT_WORK, stat, n, c->sms, st);
            if (s != LK_OK) return s;
            c->launches += 4;
            }
        } else {
            {
                ProfScope p(c, 1, st);
                s = lkh::launch_filter_hamerly(S, stat, c->sms, st);
                if (s != LK_OK) return s;
            }
            ProfScope p(c, 0, st);
            s = (use_tc && !S.center) ? lkh::launch_assign_tc_adaptive(S, S.work, stat + LK_STAT_WORK, stat,
                                                                     n, c->sms, st)
                : use_tc ? lkh::launch_assign_tc_centered(S, S.work, stat + LK_STAT_WORK, stat, n,
                                                        false, c->sms, st)
                       : lkh::launch_assign_simt(S, S.work, stat + LK_STAT_WORK, stat, n, c->sms, st);
            if (s != LK_OK) return s;
            c->launches += 2;
        }
        if (use_tc) {
            {
                ProfScope p(c, 7, st);
                s = lkh::launch_collect_tc(S, stat, n, c->sms, st);
                if (s != LK_OK) return s;
            }
            {
                ProfScope p(c, 8, st);
                s = lkh::launch_recheck_cand(S, stat, n, c->sms, st);
                if (s != LK_OK) return s;
            }
            {
                ProfScope p(c, 9, st);
                s = lkh::launch_assign_short(S, S.ovf, stat + LK_STAT_OVERFLOW, stat, n, c->sms, st);
                if (s != LK_OK) return s;
            }
            c->launches += 4;
        }
        {
            ProfScope p(c, 2, st);
            s = lkh::launch_recheck(S, stat, n, c->sms, st);
            if (s != LK_OK) return s;
        }
        {
            ProfScope p(c, 3, st);
            s = lkh::launch_refine(S, stat, buf<double>(c, B_QSCALE), n, c->sms, st);
            if (s != LK_OK) return s;
            s = lkh::launch_log_history(S, c->sms, st);
            if (s != LK_OK) return s;
        }
        c->launches += S.hlog ? 3 : 2;
    }
    return LK_OK;
}

lk_status lk_step_update(lk_ctx* c, int32_t t, void* stream) {
    if (!c) return LK_ERR_ARG;
    if (t < 1 || t > c->cfg.t_max) {
        set_error("iteration %d outside [1, %d]", t, c->cfg.t_max);
        return LK_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    ProfScope p(c, 4, st);
    const bool need_half = c->cfg.strategy != LK_STRAT_LLOYD && c->S.sgate;
    lk_status s = lkh::launch_update(c->S, buf<double>(c, B_QSCALE), buf<double>(c, B_QINV),
                                     buf<double>(c, B_SSE_PART), need_half, st);
    c->launches += need_half ? 2 : 1;
    if (s == LK_OK && c->S.center) {
        s = lkh::launch_pair_table(c->S, st);  // centering offsets of the next iteration
        c->launches += 1;
    }
    if (s == LK_OK && c->cfg.strategy == LK_STRAT_REGROUP && group_mode(c->cfg)) {
        // Regroup: the group map rebuilt from the new centroids, bounds remapped
        s = lkh::launch_regroup(c->S, buf<int32_t>(c, B_RGSCR), buf<double>(c, B_RGMEANS), c->sms, st);
        c->launches += 3;
    }
    return s;
}

lk_status lk_graph_capture(lk_ctx* c, int32_t t, void* stream) {
    if (!c) return LK_ERR_ARG;
    if (t < 2) {
        set_error("lk_graph_capture: iteration 1 takes the first-iteration path; capture t >= 2");
        return LK_ERR_ARG;
    }
    (void)stream;  // nothing executes during capture; replay uses the caller's stream
    if (!c->cap_stream) LK_CUDA_CHECK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaStream_t st = c->cap_stream;
    if (c->graph_exec) {
        cudaGraphExecDestroy(c->graph_exec);
        c->graph_exec = nullptr;
    }
    if (c->graph) {
        cudaGraphDestroy(c->graph);
        c->graph = nullptr;
    }
    const bool prof = c->profile;
    c->profile = false;  // no event records inside the graph
    LK_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    lk_status s1 = lk_step_assign(c, t, (void*)st);
    lk_status s2 = s1 == LK_OK ? lk_step_update(c, t, (void*)st) : s1;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(st, &g);
    c->profile = prof;
    if (s2 != LK_OK) {
        if (g) cudaGraphDestroy(g);
        return s2;
    }
    if (e != cudaSuccess) {
        set_error("cudaStreamEndCapture: %s", cudaGetErrorString(e));
        return LK_ERR_CUDA;
    }
    c->graph = g;
    LK_CUDA_CHECK(cudaGraphInstantiate(&c->graph_exec, g, 0));
    return LK_OK;
}

lk_status lk_graph_replay(lk_ctx* c, void* stream) {
    if (!c || !c->graph_exec) {
        set_error("lk_graph_replay before lk_graph_capture");
        return LK_ERR_STATE;
    }
    LK_CUDA_CHECK(cudaGraphLaunch(c->graph_exec, (cudaStream_t)stream));
    return LK_OK;
}

lk_status lk_validate_bounds(lk_ctx* c, int32_t decayed, double* out, int32_t nout, void* stream) {
    if (!c || !out) return LK_ERR_ARG;
    const int need = 2 + (c->L.groups > 0 ? c->L.groups : 1);
    if (nout < need) {
        set_error("lk_validate_bounds: %d output slots, need %d", nout, need);
        return LK_ERR_ARG;
    }
    for (int i = 0; i < nout; i++) out[i] = 0.0;
    return lkh::launch_validate(c->S, decayed != 0, out, need, buf<double>(c, B_VALID),
                                (cudaStream_t)stream);
}

int64_t lk_launch_count(const lk_ctx* c) { return c ? c->launches : 0; }

lk_status lk_profile(lk_ctx* c, int32_t enable) {
    if (!c) return LK_ERR_ARG;
    c->profile = enable != 0;
    LK_CUDA_CHECK(cudaDeviceSynchronize());
    for (auto& r : c->recs) {
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->recs.clear();
    return LK_OK;
}

lk_status lk_profile_read(lk_ctx* c, int32_t cls, double* total_ms, int64_t* launches) {
    if (!c) return LK_ERR_ARG;
    double tot = 0.0;
    int64_t nl = 0;
    for (auto& r : c->recs) {
        if (r.cls != cls) continue;
        LK_CUDA_CHECK(cudaEventSynchronize(r.b));
        float ms = 0.f;
        LK_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
        tot += ms;
        nl++;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = nl;
    return LK_OK;
}

}  // extern "C"
