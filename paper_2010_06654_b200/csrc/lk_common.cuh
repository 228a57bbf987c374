// lk_common.cuh -- shared device helpers and the parameter block every kernel
// of the exact-Lloyd path receives.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/lloydkit_b200.h"

#define LK_FULL_MASK 0xffffffffu
#define LK_MAX_CAND 16

namespace lk {

constexpr int kWarp = 32;
constexpr float kU32 = 5.9604644775390625e-08f;  // 2^-24, fp32 unit roundoff

// Per sorted position of the group-tile worklist: everything the certification
// of k_assign_tgy needs, in one 32-byte record (one full sector per row; the
// sort writes it at a scattered position).
struct __align__(16) TgyMeta {
    double R;      // ||x'||^2 + 2 x'.o (x' = x - o, o the tile's centroid)
    float xo;      // ||x'|| rounded up
    float bv;      // search threshold (upper bound on the TC value of the row's label column)
    float xn2;     // ||x||^2
    float lun;     // lower bound over the groups the row does not scan
    int32_t row;   // global row id
    uint32_t mask; // the row's groups to scan
};

// Everything the hot kernels need, passed by value (fits the 4 KB param space).
struct DevState {
    int64_t n;        // local rows
    int32_t d, k;
    int32_t ldx;      // X32 row stride (floats)
    int32_t ldc;      // C32 row stride (floats)
    int32_t nlb;      // lower bounds per row (1 Hamerly, t Yinyang, k Elkan)
    int32_t strategy;
    int32_t t_groups; // group count
    const float* X32;
    const double* X64;      // nullable
    double* C64;            // [k, d] master centroids
    double* C64_prev;       // [k, d] previous centroids (for drift)
    float* C32;             // [k, ldc] fp32 copy
    float* cnorm;           // [k] ||c32|| rounded up
    float* drift;           // [k] centroid drift rounded up
    float* s_half;          // [k] 1/2 min distance to another centroid, rounded down
    float* gdrift;          // [t] max drift inside each group
    float* scal;            // [8] scalars: 0 cmax, 1 drift max1, 2 drift max2, 3 (int) argmax
    int32_t* group_of;      // [k]
    int32_t* labels;        // [n]
    float* ub;              // [n]
    float* lb;              // [nlb, n] (group-major)
    int2* moved;            // [n] (row, old label)
    int32_t* flagged;       // [n]
    int32_t* work;          // [n]
    int64_t* delta;         // [k*d | k | k | 1]
    int64_t* sums;          // [k, d] fixed-point member sums
    int64_t* counts;        // [k]
    int64_t* qsum;          // [k] fixed-point sum of ||x||^2 per cluster
    int32_t* qexp;          // [3d+1]: exponents (|x_z - m_z| < 2^qexp[z]; qexp[d] for
                            // ||x - m||^2), then the order keys of max x_z and of max -x_z
    double* xshift;         // [d] m: the fixed-point sums are of x - m
    int32_t* done;          // [1] set once an iteration had changed == 0
    int32_t* iter;          // [1] current iteration (1-based), advanced by the update
    int64_t* cur;           // [LK_NSTAT] counters of the iteration in flight
    int64_t* stats;         // [t_max, LK_NSTAT]
    uint64_t* tstamp;       // [t_max + 1][2] device clock (ns): [t][0] update start, [t][1] update end
                            // of iteration t; [0][1] the start of iteration 1
    int32_t t_max;
    int2* hlog;             // [hlog_cap] label-history log: (row, new label) of moved rows
    int64_t* hlog_off;      // [t_max + 1] log offsets per iteration (-1: overflow)
    int64_t hlog_cap;
    int32_t hlog_inline;    // the fused Yinyang path writes the log itself (no k_log_history)
    double* sse;            // [t_max]
    int32_t* pw_prog;       // numpy pairwise-sum program for the fp64 recheck
    int32_t pw_len;
    // tensor-core (3xTF32) path; null when disabled
    float* Xlo;             // [n, ldx] x - trunc_tf32(x)
    float* xn2;             // [n] ||x||^2 (fp64 rounded to fp32)
    float* Chi;             // [k, ldc] trunc_tf32(c32)
    float* Clo;             // [k, ldc] c32 - Chi
    float* cn2;             // [k_pad] ||c||^2, +inf beyond k
    float* Xg_hi;           // [n, ldx] gathered rescan rows
    float* Xg_lo;           // [n, ldx]
    int32_t* cand_rows;     // [n] ambiguous rows of the tensor-core pass
    float* cand_thr;        // [n] D' threshold containing every possible winner
    float* cand_lb;         // [n] certified lower bound on every non-candidate distance
    int32_t* cand_slots;    // [n, LK_MAX_CAND] collected candidates
    int32_t* cand_cnt;      // [n] candidates found (> LK_MAX_CAND: overflow)
    int32_t* ovf;           // [n] overflow rows (fp32 difference-form rescan)
    // tile centering of the tensor-core pass (rows sorted by label; each
    // 128-row tile shifted by its first row's label centroid)
    int32_t center;         // 1: full passes and rescans run centered
    int32_t kpad;           // row stride of ptab (k rounded up to 256)
    float* ptab;            // [k, kpad] ||c_a - c_j||^2 (fp32 difference form), +inf pad
    int32_t* perm;          // [n] rows sorted by label
    int32_t* lcur;          // [k + 1] per-label histogram / cursors
    int32_t* tile_lab;      // [n / 128 + 1] label whose centroid a tile is centered on (-1: none)
    double* rowR;           // [n] ||x'||^2 + 2 x'.o of each gathered row (x' = x - o)
    float* rowxo;           // [n] ||x'|| rounded up
    float* rowbv;           // [n] search threshold of a gathered row (k_assign_tc2; +inf: none)
    float* rowxn2;          // [n] ||x||^2 of each gathered row (contiguous copy for the certification)
    int32_t* rowlab;        // [n] label of each gathered row before the pass
    // Yinyang group bounds
    int32_t* gperm;         // [k] centroid ids sorted by group
    int32_t* ginv;          // [k] position of centroid j in gperm
    int32_t* goff;          // [t + 1] group ranges in gperm
    float* Cg;              // [k, ldc] fp32 centroids in group order (gperm)
    float2* ylun;           // [n] per worklist row: (min bound over unscanned groups, the label's bits on the group tiles)
    int4* ywl;              // [n] worklist: (row, pair offset, pair count, bits of D~_a)
    int2* ypairs;           // [pair_cap] (row, group | label position << 16)
    float4* yres;           // [pair_cap] (bits of best j, best D~, second D~, -)
    int64_t pair_cap;
    int2* yaux;             // [n] per worklist row: (first result slot or -1, label position)
    int2* ypairs2;          // [t, bucket_cap] scans bucketed by group: (row, result slot)
    int64_t* ybucket;       // [t] bucket fill counts
    int64_t bucket_cap;
    // drift-offset ("lazy") bound encoding of the fused Yinyang path
    // (lk_yy_fused.cu): bounds are stored against cumulative drifts, so a row
    // whose bounds still prune is never rewritten
    int32_t lazy;
    int32_t sgate;          // Hamerly's centroid-separation gate on (s_half maintained)
    float* dcum;            // [k] cumulative centroid drift (rounded up)
    float* dgcum;           // [t] cumulative group drift (rounded up); scal[4] = cumulative max drift
    float* glb;             // [n] stored global lower bound (min over the groups)
    float* dcum_col;        // [kpad] group tiles: dcum of each B column (the pass's ub store)
    // block-sparse Yinyang on the tensor cores (lk_tgy.cu, k_assign_tgy):
    // groups are 128-column tiles of the B operand (centroids in group order)
    int32_t tgy;            // 1: the group-tile path is on
    int32_t kcols;          // B-operand columns (128 * groups with the group tiles, else k)
    const int32_t* colperm; // [kpad] centroid id of each B column (-1: padding); null = identity
    uint32_t* ymask;        // [n] per worklist entry: groups the row must scan
    uint32_t* pmask;        // [n / 128 + 4] per 128-row tile: union of its rows' masks
    int32_t* shist;         // [tgy_sort_blocks, kcols] worklist sort: per-block key counts
    struct TgyMeta* tmeta;  // [n] per sorted position of the group-tile worklist (32 B)
    // second sort key of the group-tile worklist (rows of one label ordered by
    // the groups they scan, so a 128-row tile's union of masks stays small)
    int32_t* work2;         // [n] the worklist partitioned by mask bucket: rows,
    uint32_t* ymask2;       // [n]   masks,
    float2* ylun2;          // [n]   (bound over the unscanned groups, label)
    int32_t* gfreq;         // [k, 32] listed rows of a label that scan group g (this iteration)
    uint32_t* gsel;         // [k] the groups whose mask bits form a label's bucket key
    int32_t* bhist;         // [tgy_sort_blocks, 64] per-block bucket counts / offsets
    int32_t* bbase;         // [64] bucket bases
    int4* pinfo;            // [n / 256 + 2] per row-tile pair of the sorted worklist (k_pair_info)
    // Elkan's per-centroid bounds (lk_elkan.cu): lb is [k, n]
    int32_t elkan;
    float* cch;             // [k, k] certified lower bound of 1/2 ||c_a - c_j||
    // a copy of this struct in device memory, for out-of-line device
    // functions (a reference to the kernel parameter would copy it to the stack)
    const DevState* self;
};

// Stored form of a certified upper bound U on d(x, c_label): in the lazy
// encoding ub_s = U - Dc[label] rounded up, so that at any later iteration
// ub_s + Dc_now[label] (rounded up) >= U + the label's drift since (Dc only
// grows, by rounded-up drifts).
__device__ __forceinline__ float store_ub(const DevState& S, float U, int label) {
    return S.lazy ? __fsub_ru(U, S.dcum[label]) : U;
}

// Blocks of the group-tile worklist sort (lk_tc.cu k_sort_*): three per SM (one wave at 72 registers).
inline int tgy_sort_blocks(int sms) {
    // four resident blocks per SM (k_sort_gather: 64 registers, 40 KB of shared memory)
    const int nb = 4 * (sms > 0 ? sms : 148);
    return nb > 1536 ? 1536 : nb;
}

// numpy pairwise-sum association program passed by value (k-means++ D^2
// updates): (0, start, len) = leaf, (1, 0, 0) = add the two top values.
struct PwProg {
    int32_t len;
    int32_t ops[189];
};

// Finalize a row's lower bounds from one certified bound on every non-winning
// centroid (Hamerly: the single slot; Yinyang: every group slot).  Lazy
// encoding: lb_s[g] = v + Dg[g] and glb_s = v + Dm, rounded down.
// Index of (row, group g) in the bound table: group-major [nlb, n] (a warp's
// loads of one group coalesce), except in the lazy encoding, which is
// row-major [n, nlb] (only failing rows read their groups: one contiguous
// 16-128 B row, no sectors fetched for rows that prune).
__device__ __forceinline__ int64_t lb_index(const DevState& S, int64_t row, int g) {
    return S.lazy ? row * S.nlb + g : (int64_t)g * S.n + row;
}

__device__ __forceinline__ void write_lb_all(const DevState& S, int64_t row, float v) {
    if (S.tgy) {
        // group tiles: the row's scanned groups already hold their own bounds
        // (k_assign_tgy writes them for ambiguous rows too; the table starts at
        // 0), so a re-decision only sets the global bound
        S.glb[row] = __fadd_rd(v, S.scal[4]);
        return;
    }
    if (S.lazy) {
        for (int g = 0; g < S.nlb; g++) S.lb[row * S.nlb + g] = __fadd_rd(v, S.dgcum[g]);
        S.glb[row] = __fadd_rd(v, S.scal[4]);
        return;
    }
    for (int g = 0; g < S.nlb; g++) S.lb[(int64_t)g * S.n + row] = v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    return g;
}

__device__ __forceinline__ float tf32_trunc(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ unsigned lane_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Warp-aggregated append to a device worklist: one atomic per warp.  Every
// lane of the (converged) warp must call it.
__device__ __forceinline__ int64_t warp_append(bool pred, unsigned long long* counter) {
    unsigned m = __ballot_sync(LK_FULL_MASK, pred);
    if (m == 0) return -1;
    int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
    base = __shfl_sync(LK_FULL_MASK, base, leader);
    return pred ? (int64_t)(base + __popc(m & lanemask_lt())) : -1;
}

__device__ __forceinline__ void warp_count(bool pred, int64_t* counter) {
    unsigned m = __ballot_sync(LK_FULL_MASK, pred);
    if (m && lane_id() == (unsigned)(__ffs(m) - 1))
        atomicAdd((unsigned long long*)counter, (unsigned long long)__popc(m));
}

__device__ __forceinline__ void warp_add(int64_t v, int64_t* counter) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(LK_FULL_MASK, v, o);
    if (lane_id() == 0 && v) atomicAdd((unsigned long long*)counter, (unsigned long long)v);
}

// Block-aggregated append: one global atomic per block per call.  Every
// thread of the block must call it (block-uniform control flow); scratch is
// >= (blockDim/32 + 1) ints of shared memory.  Returns the slot (or -1).
__device__ __forceinline__ int64_t block_append(bool pred, unsigned long long* counter,
                                                unsigned long long* scratch) {
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned m = __ballot_sync(LK_FULL_MASK, pred);
    if (lane_id() == 0) scratch[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < nw; w++) {
            unsigned long long c = scratch[w];
            scratch[w] = tot;
            tot += c;
        }
        scratch[nw] = tot ? atomicAdd(counter, tot) : 0ull;
    }
    __syncthreads();
    int64_t pos = pred ? (int64_t)(scratch[nw] + scratch[warp] + __popc(m & lanemask_lt())) : -1;
    __syncthreads();  // scratch reusable by the next call
    return pos;
}

// Block-aggregated counter increment (block-uniform).
__device__ __forceinline__ void block_count(bool pred, int64_t* counter,
                                            unsigned long long* scratch) {
    block_append(pred, (unsigned long long*)counter, scratch);
}

// Nonnegative-float atomic max via integer ordering.
__device__ __forceinline__ void atomic_max_pos(float* addr, float v) {
    atomicMax((int*)addr, __float_as_int(v));
}

// Relative error (in units of the computed distance) of the fp32
// difference-form distance sqrt(sum_z fl(x_z - c_z)^2) against the exact
// distance of the fp32 operands, plus the fp64 oracle's own error.  Generous
// (d + 8) u; see DESIGN.md "certifying labels".
__device__ __forceinline__ float simt_rel_err(int d) { return (float)(d + 8) * kU32; }

}  // namespace lk

// Host-side error plumbing shared by the launchers.
namespace lkh {
void set_error(const char* fmt, ...);
}

#define LK_CUDA_CHECK(expr)                                                          \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            lkh::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                \
                           cudaGetErrorString(_e));                                  \
            return LK_ERR_CUDA;                                                      \
        }                                                                            \
    } while (0)

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its predecessor in the stream drains; pdl_wait() blocks until
// the predecessor has completed and its writes are visible (a no-op for a plain
// launch).  pdl_trigger() lets the successor be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

namespace lk {
inline bool pdl_enabled() {
    static const int v = [] {
        const char* e = getenv("LK_PDL");  // A/B knob (measured neutral on cfg1 / cfg2: off)
        return e ? atoi(e) : 0;
    }();
    return v != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, args...);
}
}  // namespace lk

#define LK_LAUNCH_CHECK()                                                            \
    do {                                                                             \
        cudaError_t _e = cudaGetLastError();                                         \
        if (_e != cudaSuccess) {                                                     \
            lkh::set_error("%s:%d launch: %s", __FILE__, __LINE__,                   \
                           cudaGetErrorString(_e));                                  \
            return LK_ERR_CUDA;                                                      \
        }                                                                            \
    } while (0)
