// lk_tgy.cu -- the bound filter of the block-sparse Yinyang pass on the tensor
// cores (group tiles, d <= 32; the pass itself is k_assign_tgy in lk_tc.cu).
//
// Reference: Yinyang.update_bounds (pruners.py:418-436) and the gates of
// assign_pass (pruners.py:445-456): decay ub by the label's drift and every
// group bound by its group's largest drift, the global gate, the tighten of ub
// to the point's distance from its own centroid, then the per-group gate.
// Bounds are stored against cumulative drifts, so the decay is
// free and a row that still prunes costs its label, ub and global bound (12 B).
//
// A row that fails a group gate goes to the worklist with the bitmask of its
// failing groups plus the group of its label (the label's own column must be
// in the scan: the pass certifies the winner against it) and the smallest
// decayed bound over the groups it does not scan.
#include <math.h>
#include <stdlib.h>

#include "lk_async.cuh"
#include "lk_common.cuh"
#include "lk_internal.h"

namespace lk {
namespace tgy {

constexpr int kThreads = 256;

// One row of the filter: the gates, the tighten, the group mask.  Returns
// whether the row goes to the worklist (mask, lun set).  a / ub_s / glb_s are
// the row's label and stored bounds (loaded by the caller, one row ahead).
template <int DP>
__device__ __forceinline__ bool tgy_row(const DevState& S, int64_t i, int a, float ub_s, float glb_s,
                                        const float* dg, float dm, float rho, int64_t& n_active,
                                        int64_t& n_pairs, uint32_t& mask, float& lun) {
    const int G = S.t_groups;
    bool need = false;
    mask = 0;
    lun = INFINITY;
    float u = __fadd_ru(ub_s, __ldg(S.dcum + a));
    const float sa = __ldg(S.s_half + a);
    const float gate = fmaxf(__fsub_rd(glb_s, dm), sa);
    if (!(gate > u)) {
        n_active++;
        // tighten: fp32 difference-form distance to the own centroid,
        // certified upper bound
        float xr[DP];
        const float4* xp = reinterpret_cast<const float4*>(S.X32 + i * S.ldx);
#pragma unroll
        for (int z4 = 0; z4 < DP / 4; z4++) {
            const float4 v = 4 * z4 < S.d ? __ldg(xp + z4) : make_float4(0.f, 0.f, 0.f, 0.f);
            xr[4 * z4] = v.x;
            xr[4 * z4 + 1] = v.y;
            xr[4 * z4 + 2] = v.z;
            xr[4 * z4 + 3] = v.w;
        }
        // the group table is loaded with the point (one memory round trip
        // instead of two; most rows that fail the global gate need it)
        float v[32];
        const float4* lp = reinterpret_cast<const float4*>(S.lb + i * S.nlb);
#pragma unroll
        for (int g4 = 0; g4 < 8; g4++) {
            if (4 * g4 < G) {
                const float4 q = __ldcs(lp + g4);
                v[4 * g4] = q.x;
                v[4 * g4 + 1] = q.y;
                v[4 * g4 + 2] = q.z;
                v[4 * g4 + 3] = q.w;
            } else {
                v[4 * g4] = v[4 * g4 + 1] = v[4 * g4 + 2] = v[4 * g4 + 3] = INFINITY;
            }
        }
        const float4* cp = reinterpret_cast<const float4*>(S.C32 + (int64_t)a * S.ldc);
        float acc = 0.f, xn2 = 0.f;
#pragma unroll
        for (int z4 = 0; z4 < DP / 4; z4++) {
            if (4 * z4 < S.d) {
                const float4 c = __ldg(cp + z4);
                const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    // (padding dimensions are zero in both rows)
                    const float t = xr[4 * z4 + e] - cv[e];
                    acc = fmaf(t, t, acc);
                    xn2 = fmaf(xr[4 * z4 + e], xr[4 * z4 + e], xn2);
                }
            }
        }
        const float U = (sqrtf(acc) + kU32 * (sqrtf(xn2) + __ldg(S.cnorm + a))) * (1.0f + rho);
        const bool tight = U < u;
        u = fminf(u, U);
        if (!(gate > u)) {
            float gmin = INFINITY;
#pragma unroll
            for (int g = 0; g < 32; g++) {
                v[g] = g < G ? __fsub_rd(v[g], dg[g]) : INFINITY;
                gmin = fminf(gmin, v[g]);
            }
            need = !(fmaxf(gmin, sa) > u);
            if (need) {
                const int ga = __ldg(S.group_of + a);
#pragma unroll
                for (int g = 0; g < 32; g++) {
                    const bool scan = !(v[g] > u) || g == ga;
                    if (g < G && scan) mask |= 1u << g;
                    else lun = fminf(lun, v[g]);
                }
                n_pairs += __popc(mask);
            } else {
                // every group prunes: their (tighter) minimum becomes the global bound
                S.glb[i] = __fadd_rd(gmin, dm);
            }
        }
        if (tight && !need) S.ub[i] = __fsub_ru(u, __ldg(S.dcum + a));
    }
    return need;
}

// Variant 0: a thread per row, block-aggregated appends.
template <int DP>
__global__ void __launch_bounds__(kThreads) k_filter_tgy(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    __shared__ float dg[32];
    const int G = S.t_groups;
    if (threadIdx.x < 32) dg[threadIdx.x] = threadIdx.x < G ? S.dgcum[threadIdx.x] : 0.f;
    __syncthreads();
    const float dm = S.scal[4];
    const float rho = simt_rel_err(S.d);
    int64_t n_active = 0, n_pairs = 0;
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < S.n; base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + threadIdx.x;
        bool need = false;
        uint32_t mask = 0;
        float lun = INFINITY;
        int a = 0;
        if (i < S.n) {
            a = __ldcs(S.labels + i);
            need = tgy_row<DP>(S, i, a, __ldcs(S.ub + i), __ldcs(S.glb + i), dg, dm, rho,
                               n_active, n_pairs, mask, lun);
        }
        const int64_t pos = block_append(need, (unsigned long long*)(stat + LK_STAT_WORK), scr);
        if (need) {
            // (the label rides along: the sort keys on it without a gather)
            S.work[pos] = (int)i;
            S.ymask[pos] = mask;
            S.ylun[pos] = make_float2(lun, __int_as_float(a));
        }
    }
    warp_add(n_active, stat + LK_STAT_ACTIVE);
    warp_add(n_pairs, stat + LK_STAT_PAIRS);
}

// Variant 3: no block barriers.  Each warp appends its listed rows
// to its own shared-memory queue and flushes it with one global atomic when
// it is nearly full (one atomic per ~kQ rows, coalesced worklist stores), so
// a warp waiting on its rows' loads never holds up the block's other warps;
// the next row's label and stored bounds are loaded one row ahead.
constexpr int kQ = 128;
template <int DP>
__global__ void __launch_bounds__(kThreads, 4) k_filter_tgy_wq(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ int qrow[kThreads / 32][kQ];
    __shared__ uint32_t qmask[kThreads / 32][kQ];
    __shared__ float qlun[kThreads / 32][kQ];
    __shared__ int qlab[kThreads / 32][kQ];
    __shared__ float dg[32];
    const int G = S.t_groups;
    if (threadIdx.x < 32) dg[threadIdx.x] = threadIdx.x < G ? S.dgcum[threadIdx.x] : 0.f;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float dm = S.scal[4];
    const float rho = simt_rel_err(S.d);
    int64_t n_active = 0, n_pairs = 0;
    int qn = 0;  // (warp-uniform)
    auto flush = [&]() {
        __syncwarp();
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd((unsigned long long*)(stat + LK_STAT_WORK), (unsigned long long)qn);
        b = __shfl_sync(LK_FULL_MASK, b, 0);
        for (int e = lane; e < qn; e += 32) {
            S.work[b + e] = qrow[w][e];
            S.ymask[b + e] = qmask[w][e];
            S.ylun[b + e] = make_float2(qlun[w][e], __int_as_float(qlab[w][e]));
        }
        __syncwarp();
        qn = 0;
    };
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    int a_n = 0;
    float ub_n = 0.f, glb_n = 0.f;
    if (i < S.n) {
        a_n = __ldcs(S.labels + i);
        ub_n = __ldcs(S.ub + i);
        glb_n = __ldcs(S.glb + i);
    }
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < S.n; base += stride, i += stride) {
        const int a = a_n;
        const float ub_s = ub_n, glb_s = glb_n;
        if (i + stride < S.n) {
            a_n = __ldcs(S.labels + i + stride);
            ub_n = __ldcs(S.ub + i + stride);
            glb_n = __ldcs(S.glb + i + stride);
        }
        bool need = false;
        uint32_t mask = 0;
        float lun = INFINITY;
        if (i < S.n) need = tgy_row<DP>(S, i, a, ub_s, glb_s, dg, dm, rho, n_active, n_pairs, mask, lun);
        const unsigned bal = __ballot_sync(LK_FULL_MASK, need);
        if (need) {
            const int off = qn + __popc(bal & lanemask_lt());
            qrow[w][off] = (int)i;
            qmask[w][off] = mask;
            qlun[w][off] = lun;
            qlab[w][off] = a;
        }
        qn += __popc(bal);
        if (qn > kQ - 32) flush();
    }
    if (qn) flush();
    warp_add(n_active, stat + LK_STAT_ACTIVE);
    warp_add(n_pairs, stat + LK_STAT_PAIRS);
}


// Variant 2: a streaming pipeline, 8 lanes per row.  Each CTA walks
// 128-row tiles of the row range; one thread stages a tile's labels, stored
// bounds, points and group tables with 1-D bulk copies (3 stages, ~34 KB each
// at d = 32, 32 groups) -- every byte of the row range streams in whether the
// row fails its global gate or not (84% do at cfg5), so HBM sees long
// sequential reads with ~20 MB in flight instead of one thread's dependent
// gathers.  8 lanes per row (one float4 of the point and of the group table
// each, reductions by shuffles), 4 rows per lane group, the label-indexed
// loads of all 4 rows issued before any of them is used.  Rows past the last
// full tile take the one-thread-per-row path (tgy_row).
constexpr int kTR = 128;   // rows per tile
constexpr int kST = 3;     // stages
constexpr int kQB = 64;    // worklist queue per warp
__host__ __device__ inline int tgy_bulk_stage_bytes(int ldx, int nlb) { return kTR * (12 + 4 * ldx + 4 * nlb); }

template <int DP>
__global__ void __launch_bounds__(kThreads, 2) k_filter_tgy_bulk(DevState S, int64_t* stat) {
    if (*S.done) return;
    extern __shared__ __align__(128) uint8_t fsm[];
    __shared__ uint64_t fbar[kST];
    __shared__ int qrow[kThreads / 32][kQB];
    __shared__ uint32_t qmask[kThreads / 32][kQB];
    __shared__ float qlun[kThreads / 32][kQB];
    __shared__ int qlab[kThreads / 32][kQB];
    __shared__ float dg[32];
    const int G = S.t_groups;
    const int ldx = S.ldx, nlb = S.nlb;
    const int SB = tgy_bulk_stage_bytes(ldx, nlb);
    const int64_t n_full = S.n / kTR;  // full tiles
    const int64_t n_my = n_full > blockIdx.x ? (n_full - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, sub = lane & 7, rg = tid >> 3;
    if (tid < 32) dg[tid] = tid < G ? S.dgcum[tid] : 0.f;
    auto stage_ptr = [&](int st_) { return fsm + (size_t)st_ * SB; };
    auto issue = [&](int64_t j, int st_) {
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)kTR;
        uint8_t* b = stage_ptr(st_);
        mbar_expect_tx(&fbar[st_], (uint32_t)SB);
        bulk_load(b, S.labels + r0, kTR * 4, &fbar[st_]);
        bulk_load(b + kTR * 4, S.ub + r0, kTR * 4, &fbar[st_]);
        bulk_load(b + kTR * 8, S.glb + r0, kTR * 4, &fbar[st_]);
        bulk_load(b + kTR * 12, S.X32 + r0 * ldx, (uint32_t)(kTR * ldx * 4), &fbar[st_]);
        bulk_load(b + kTR * (12 + 4 * ldx), S.lb + r0 * nlb, (uint32_t)(kTR * nlb * 4), &fbar[st_]);
    };
    if (tid == 0) {
        for (int e = 0; e < kST; e++) mbar_init(&fbar[e], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int e = 0; e < kST && e < n_my; e++) issue(e, e);
    }
    __syncthreads();
    const float dm = S.scal[4];
    const float rho = simt_rel_err(S.d);
    const int c4n = ldx / 4;
    int64_t n_active = 0, n_pairs = 0;
    int qn = 0;  // (warp-uniform)
    auto flush = [&]() {
        __syncwarp();
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd((unsigned long long*)(stat + LK_STAT_WORK), (unsigned long long)qn);
        b = __shfl_sync(LK_FULL_MASK, b, 0);
        for (int e = lane; e < qn; e += 32) {
            S.work[b + e] = qrow[w][e];
            S.ymask[b + e] = qmask[w][e];
            S.ylun[b + e] = make_float2(qlun[w][e], __int_as_float(qlab[w][e]));
        }
        __syncwarp();
        qn = 0;
    };
    // append the rows whose lane group leader (sub == 0) has need set
    auto append = [&](bool need, int64_t i, uint32_t mask, float lun, int lab) {
        const unsigned bal = __ballot_sync(LK_FULL_MASK, need);
        if (need) {
            const int off = qn + __popc(bal & lanemask_lt());
            qrow[w][off] = (int)i;
            qmask[w][off] = mask;
            qlun[w][off] = lun;
            qlab[w][off] = lab;
        }
        qn += __popc(bal);
        if (qn > kQB - 32) flush();
    };
    for (int64_t j = 0; j < n_my; j++) {
        const int st_ = (int)(j % kST);
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)kTR;
        mbar_wait(&fbar[st_], (uint32_t)((j / kST) & 1));
        const uint8_t* b = stage_ptr(st_);
        const int* slab = reinterpret_cast<const int*>(b);
        const float* sub_s = reinterpret_cast<const float*>(b + kTR * 4);
        const float* sglb = reinterpret_cast<const float*>(b + kTR * 8);
        const float4* spt = reinterpret_cast<const float4*>(b + kTR * 12);
        const float4* slb = reinterpret_cast<const float4*>(b + kTR * (12 + 4 * ldx));
        // the label-indexed loads of the lane group's 4 rows first
        int a[4], ga[4];
        float dca[4], sa[4], cna[4];
        float4 cv[4];
#pragma unroll
        for (int rr = 0; rr < 4; rr++) {
            const int r = rg + 32 * rr;
            a[rr] = slab[r];
            dca[rr] = __ldg(S.dcum + a[rr]);
            sa[rr] = __ldg(S.s_half + a[rr]);
            cna[rr] = __ldg(S.cnorm + a[rr]);
            ga[rr] = __ldg(S.group_of + a[rr]);
            cv[rr] = sub < c4n ? __ldg(reinterpret_cast<const float4*>(S.C32 + (int64_t)a[rr] * S.ldc) + sub)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int rr = 0; rr < 4; rr++) {
            const int r = rg + 32 * rr;
            const int64_t i = r0 + r;
            const float u0 = __fadd_ru(sub_s[r], dca[rr]);
            const float gate = fmaxf(__fsub_rd(sglb[r], dm), sa[rr]);
            const bool active = !(gate > u0);
            // tighten (fp32 difference form, certified)
            const float4 x = sub < c4n ? spt[r * c4n + sub] : make_float4(0.f, 0.f, 0.f, 0.f);
            float acc, xn2;
            {
                const float t0 = x.x - cv[rr].x, t1 = x.y - cv[rr].y, t2 = x.z - cv[rr].z, t3 = x.w - cv[rr].w;
                acc = fmaf(t3, t3, fmaf(t2, t2, fmaf(t1, t1, t0 * t0)));
                xn2 = fmaf(x.w, x.w, fmaf(x.z, x.z, fmaf(x.y, x.y, x.x * x.x)));
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                acc += __shfl_xor_sync(LK_FULL_MASK, acc, o, 8);
                xn2 += __shfl_xor_sync(LK_FULL_MASK, xn2, o, 8);
            }
            const float U = (sqrtf(acc) + kU32 * (sqrtf(xn2) + cna[rr])) * (1.0f + rho);
            const bool tight = U < u0;
            const float u = fminf(u0, U);
            const bool fail = active && !(gate > u);
            // the lane's four groups
            float v[4];
            {
                const float4 q = 4 * sub < G ? slb[r * (nlb / 4) + sub] : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
                v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
            }
            float gmin = INFINITY;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int g = 4 * sub + e;
                v[e] = g < G ? __fsub_rd(v[e], dg[g]) : INFINITY;
                gmin = fminf(gmin, v[e]);
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) gmin = fminf(gmin, __shfl_xor_sync(LK_FULL_MASK, gmin, o, 8));
            const bool need = fail && !(fmaxf(gmin, sa[rr]) > u);
            uint32_t mask = 0;
            float lun = INFINITY;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int g = 4 * sub + e;
                const bool scan = !(v[e] > u) || g == ga[rr];
                if (g < G && scan) mask |= 1u << g;
                else lun = fminf(lun, v[e]);
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                mask |= __shfl_xor_sync(LK_FULL_MASK, mask, o, 8);
                lun = fminf(lun, __shfl_xor_sync(LK_FULL_MASK, lun, o, 8));
            }
            if (sub == 0) {
                if (fail && !need) S.glb[i] = __fadd_rd(gmin, dm);  // every group prunes
                if (active && tight && !need) S.ub[i] = __fsub_ru(u, dca[rr]);
                n_active += active;
                if (need) n_pairs += __popc(mask);
            }
            append(need && sub == 0, i, mask, lun, a[rr]);
        }
        __syncthreads();  // stage st_ consumed
        if (tid == 0 && j + kST < n_my) issue(j + kST, st_);
    }
    // rows past the last full tile: one thread per row
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t i0 = n_full * kTR; i0 < S.n; i0 += kThreads) {
            const int64_t i = i0 + tid;
            bool need = false;
            uint32_t mask = 0;
            float lun = INFINITY;
            int la = 0;
            if (i < S.n) {
                int64_t na = 0, np = 0;
                la = S.labels[i];
                need = tgy_row<DP>(S, i, la, S.ub[i], S.glb[i], dg, dm, rho, na, np, mask, lun);
                n_active += na;
                n_pairs += np;
            }
            append(need, i, mask, lun, la);
        }
    }
    if (qn) flush();
    warp_add(n_active, stat + LK_STAT_ACTIVE);
    warp_add(n_pairs, stat + LK_STAT_PAIRS);
}

// Variant 4 (default for 16 < d <= 32): the streaming pipeline of variant 1
// with a thread per row.  The 8-lanes-per-row form issues ~1800 thread
// instructions per row (every lane repeats the row's scalar work and 15
// shuffles; ncu: issue-active 51% at 16 warps per SM, DRAM 35%), so it is
// bound by instruction issue, not by HBM.  Here a tile's 128 rows are staged
// the same way (1-D bulk copies; stages and CTAs per SM: see NST below) and thread r
// walks row r's point and group table in shared memory, the float4 columns
// rotated by r so that a quarter-warp's eight threads read eight different
// bank groups (conflict-free at 128-byte rows); the own centroid's row comes
// through L1/L2 in the same rotated order.
constexpr int kSR = 128;   // rows per tile = threads per CTA

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// NST = 2: two stages per CTA, three CTAs per SM, a tile's label-indexed loads
// requested at its start.  NST = 3: three stages, two CTAs per SM, and the
// next tile's label-indexed loads (its stage has landed while the previous
// tile ran) requested before this tile's math, so no tile starts with an L2
// round trip.
template <int DP, int NST>
__global__ void __launch_bounds__(kSR, NST == 2 ? 3 : 2) k_filter_tgy_srow(DevState S, int64_t* stat) {
    if (*S.done) return;
    constexpr int kSS = NST;
    extern __shared__ __align__(128) uint8_t fsm[];
    __shared__ uint64_t fbar[kSS];
    __shared__ int qrow[kSR / 32][kQB];
    __shared__ uint32_t qmask[kSR / 32][kQB];
    __shared__ float qlun[kSR / 32][kQB];
    __shared__ int qlab[kSR / 32][kQB];
    __shared__ __align__(16) float dg[32];
    const int G = S.t_groups;
    const int ldx = S.ldx, nlb = S.nlb;  // (both 32: the launcher checks)
    const int SB = kSR * (12 + 4 * ldx + 4 * nlb);
    const int64_t n_full = S.n / kSR;  // full tiles
    const int64_t n_my = n_full > blockIdx.x ? (n_full - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    if (tid < 32) dg[tid] = tid < G ? S.dgcum[tid] : 0.f;
    auto issue = [&](int64_t j, int st_) {
        const int64_t r0 = (blockIdx.x + j * gridDim.x) * (int64_t)kSR;
        uint8_t* b = fsm + (size_t)st_ * SB;
        mbar_expect_tx(&fbar[st_], (uint32_t)SB);
        bulk_load(b, S.labels + r0, kSR * 4, &fbar[st_]);
        bulk_load(b + kSR * 4, S.ub + r0, kSR * 4, &fbar[st_]);
        bulk_load(b + kSR * 8, S.glb + r0, kSR * 4, &fbar[st_]);
        bulk_load(b + kSR * 12, S.X32 + r0 * ldx, (uint32_t)(kSR * ldx * 4), &fbar[st_]);
        bulk_load(b + kSR * (12 + 4 * ldx), S.lb + r0 * nlb, (uint32_t)(kSR * nlb * 4), &fbar[st_]);
    };
    if (tid == 0) {
        for (int e = 0; e < kSS; e++) mbar_init(&fbar[e], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int e = 0; e < kSS && e < n_my; e++) issue(e, e);
    }
    __syncthreads();
    const float dm = S.scal[4];
    const float rho = simt_rel_err(S.d);
    int64_t n_active = 0, n_pairs = 0;
    int qn = 0;  // (warp-uniform)
    auto flush = [&]() {
        __syncwarp();
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd((unsigned long long*)(stat + LK_STAT_WORK), (unsigned long long)qn);
        b = __shfl_sync(LK_FULL_MASK, b, 0);
        for (int e = lane; e < qn; e += 32) {
            S.work[b + e] = qrow[w][e];
            S.ymask[b + e] = qmask[w][e];
            S.ylun[b + e] = make_float2(qlun[w][e], __int_as_float(qlab[w][e]));
        }
        __syncwarp();
        qn = 0;
    };
    auto append = [&](bool need, int64_t i, uint32_t mask, float lun, int lab) {
        const unsigned bal = __ballot_sync(LK_FULL_MASK, need);
        if (need) {
            const int off = qn + __popc(bal & lanemask_lt());
            qrow[w][off] = (int)i;
            qmask[w][off] = mask;
            qlun[w][off] = lun;
            qlab[w][off] = lab;
        }
        qn += __popc(bal);
        if (qn > kQB - 32) flush();
    };
    // groups past G never scan and never bound: v = lb - (-inf) = +inf
    if (tid < 32 && tid >= G) dg[tid] = -INFINITY;
    __syncthreads();
    const float rho1 = 1.0f + rho + 4.76837158203125e-07f;  // (+ 2^-21: the approximate square roots)
    // everything indexed by a row's label, requested at once (one L2 round
    // trip); rows that pass the global gate (16% at cfg5) load it in vain
    struct ByLabel {
        float4 cv[8];
        float dca, sa, cna;
        int ga, a;
    };
    auto by_label = [&](int a_, ByLabel& L) {
        const float4* cp = reinterpret_cast<const float4*>(S.C32 + (int64_t)a_ * S.ldc);
#pragma unroll
        for (int c = 0; c < 8; c++) L.cv[c] = __ldg(cp + ((c + tid) & 7));
        L.dca = __ldg(S.dcum + a_);
        L.sa = __ldg(S.s_half + a_);
        L.cna = __ldg(S.cnorm + a_);
        L.ga = __ldg(S.group_of + a_);
        L.a = a_;
    };
    ByLabel cur, nxt;
    if (NST >= 3 && n_my > 0) {
        mbar_wait(&fbar[0], 0);
        by_label(reinterpret_cast<const int*>(fsm)[tid], cur);
    }
    for (int64_t j = 0; j < n_my; j++) {
        const int st_ = (int)(j % kSS);
        const int64_t i = (blockIdx.x + j * gridDim.x) * (int64_t)kSR + tid;
        if (NST >= 3) {
            if (j + 1 < n_my) {
                const int s1 = (int)((j + 1) % kSS);
                mbar_wait(&fbar[s1], (uint32_t)(((j + 1) / kSS) & 1));
                by_label(reinterpret_cast<const int*>(fsm + (size_t)s1 * SB)[tid], nxt);
            }
        } else {
            mbar_wait(&fbar[st_], (uint32_t)((j / kSS) & 1));
        }
        const uint8_t* b = fsm + (size_t)st_ * SB;
        if (NST < 3) by_label(reinterpret_cast<const int*>(b)[tid], cur);
        const int a = cur.a;
        const float ub_s = reinterpret_cast<const float*>(b + kSR * 4)[tid];
        const float glb_s = reinterpret_cast<const float*>(b + kSR * 8)[tid];
        const float4* spt = reinterpret_cast<const float4*>(b + kSR * 12) + tid * 8;
        const float4* slb = reinterpret_cast<const float4*>(b + kSR * (12 + 4 * 32)) + tid * 8;
        const float4 (&cv)[8] = cur.cv;
        const float dca = cur.dca, sa = cur.sa, cna = cur.cna;
        const int ga = cur.ga;
        // tighten (fp32 difference form, certified)
        float acc = 0.f, xn2 = 0.f;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const float4 x = spt[(c + tid) & 7];
            const float t0 = x.x - cv[c].x, t1 = x.y - cv[c].y, t2 = x.z - cv[c].z, t3 = x.w - cv[c].w;
            acc = fmaf(t3, t3, fmaf(t2, t2, fmaf(t1, t1, fmaf(t0, t0, acc))));
            xn2 = fmaf(x.w, x.w, fmaf(x.z, x.z, fmaf(x.y, x.y, fmaf(x.x, x.x, xn2))));
        }
        const float u0 = __fadd_ru(ub_s, dca);
        const float gate = fmaxf(__fsub_rd(glb_s, dm), sa);
        const bool active = !(gate > u0);
        // (sqrt.approx: relative error <= 2^-23, covered by rho1)
        const float U = (sqrt_approx(acc) + kU32 * (sqrt_approx(xn2) + cna)) * rho1;
        const bool tight = U < u0;
        const float u = fminf(u0, U);
        const bool fail = active && !(gate > u);
        // the group gate, branch-free: the mask of the groups to scan (the
        // label's own group included) and the bound over the others
        float gmin = INFINITY, lun = INFINITY;
        uint32_t mask = 0;
        const unsigned gac = (unsigned)ga >> 2, gab = 1u << (ga & 3);
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int cc = (c + tid) & 7;
            const float4 q = slb[cc];
            const float4 dq = reinterpret_cast<const float4*>(dg)[cc];
            const unsigned ob = (unsigned)cc == gac ? gab : 0u;
            const float v0 = __fsub_rd(q.x, dq.x), v1 = __fsub_rd(q.y, dq.y);  // (a negative lower bound is still valid)
            const float v2 = __fsub_rd(q.z, dq.z), v3 = __fsub_rd(q.w, dq.w);
            gmin = fminf(gmin, fminf(fminf(v0, v1), fminf(v2, v3)));
            const bool s0 = !(v0 > u) || (ob & 1u), s1 = !(v1 > u) || (ob & 2u);
            const bool s2 = !(v2 > u) || (ob & 4u), s3 = !(v3 > u) || (ob & 8u);
            const unsigned nib = (s0 ? 1u : 0u) | (s1 ? 2u : 0u) | (s2 ? 4u : 0u) | (s3 ? 8u : 0u);
            mask |= nib << (4 * cc);
            lun = fminf(lun, fminf(fminf(s0 ? INFINITY : v0, s1 ? INFINITY : v1),
                                   fminf(s2 ? INFINITY : v2, s3 ? INFINITY : v3)));
        }
        const bool need = fail && !(fmaxf(gmin, sa) > u);
        if (fail && !need) S.glb[i] = __fadd_rd(gmin, dm);  // every group prunes: their minimum is the global bound
        if (active && tight && !need) S.ub[i] = __fsub_ru(u, dca);
        n_active += active;
        if (need) n_pairs += __popc(mask);
        append(need, i, mask, lun, a);
        __syncthreads();  // stage st_ consumed
        if (tid == 0 && j + kSS < n_my) issue(j + kSS, st_);
        if (NST >= 3) cur = nxt;
    }
    // rows past the last full tile: one thread per row from global memory
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t i0 = n_full * kSR; i0 < S.n; i0 += kSR) {
            const int64_t i = i0 + tid;
            bool need = false;
            uint32_t mask = 0;
            float lun = INFINITY;
            int la = 0;
            if (i < S.n) {
                int64_t na = 0, np = 0;
                la = S.labels[i];
                need = tgy_row<DP>(S, i, la, S.ub[i], S.glb[i], dg, dm, rho, na, np, mask, lun);
                n_active += na;
                n_pairs += np;
            }
            append(need, i, mask, lun, la);
        }
    }
    if (qn) flush();
    warp_add(n_active, stat + LK_STAT_ACTIVE);
    warp_add(n_pairs, stat + LK_STAT_PAIRS);
}

}  // namespace tgy
}  // namespace lk

namespace lkh {

lk_status launch_filter_tgy(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st) {
    int64_t blocks = (S.n + lk::tgy::kThreads - 1) / lk::tgy::kThreads;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    if (blocks < 1) blocks = 1;
    // LK_TGY_FILTER (A/B knob): 1 (default) the streaming pipeline with a
    // thread per row where it applies (128-byte points and group tables:
    // 28 < d <= 32, 29..32 groups), else 0; 0 a thread per row from global
    // memory with block-aggregated appends; 2 the streaming pipeline with 8
    // lanes per row; 3 a thread per row with warp queues
    static const int variant = [] {
        const char* e = getenv("LK_TGY_FILTER");
        return e ? atoi(e) : 1;
    }();
    const bool bulk_ok = S.nlb % 4 == 0 && S.ldx % 4 == 0;
    if (bulk_ok && S.nlb == 32 && S.ldx == 32 && (variant == 4 || variant == 1)) {
        // the streaming pipeline, a thread per row (LK_TGY_STAGES, A/B knob: 2
        // stages and three CTAs per SM -- the default: 3.7 ms on cfg5 -- or 3
        // stages and two CTAs per SM with the next tile's label-indexed loads
        // prefetched: 4.2 ms, eight warps per SM hide less than the prefetch saves)
        static const int nst = [] {
            const char* e = getenv("LK_TGY_STAGES");
            return (e && atoi(e) == 3) ? 3 : 2;
        }();
        const int smem = nst * lk::tgy::kSR * (12 + 4 * S.ldx + 4 * S.nlb);
        static bool attr4 = false;
        if (!attr4) {
            LK_CUDA_CHECK(cudaFuncSetAttribute(lk::tgy::k_filter_tgy_srow<32, 2>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 72 * 1024));
            LK_CUDA_CHECK(cudaFuncSetAttribute(lk::tgy::k_filter_tgy_srow<32, 3>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 108 * 1024));
            attr4 = true;
        }
        if (nst == 2)
            lk::tgy::k_filter_tgy_srow<32, 2><<<(unsigned)(sms * 3), lk::tgy::kSR, smem, st>>>(S, stat);
        else
            lk::tgy::k_filter_tgy_srow<32, 3><<<(unsigned)(sms * 2), lk::tgy::kSR, smem, st>>>(S, stat);
    } else if (bulk_ok && (variant == 2 || variant == 5)) {
        // the streaming pipeline: one wave of two CTAs per SM
        constexpr int kMaxSmem = 110 * 1024;
        const int smem = lk::tgy::kST * lk::tgy::tgy_bulk_stage_bytes(S.ldx, S.nlb);
        static bool attr_set = false;
        if (!attr_set) {
            LK_CUDA_CHECK(cudaFuncSetAttribute(lk::tgy::k_filter_tgy_bulk<32>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
            attr_set = true;
        }
        if (smem > kMaxSmem) {
            lkh::set_error("filter: %d B of staging per CTA", smem);
            return LK_ERR_UNSUPPORTED;
        }
        lk::tgy::k_filter_tgy_bulk<32><<<(unsigned)(sms * 2), lk::tgy::kThreads, smem, st>>>(S, stat);
    } else if (variant == 3) {
        // (four resident blocks per SM at 64 registers: one wave)
        if (blocks > (int64_t)sms * 4) blocks = (int64_t)sms * 4;
        if (S.d <= 8)
            lk::tgy::k_filter_tgy_wq<8><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
        else if (S.d <= 16)
            lk::tgy::k_filter_tgy_wq<16><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
        else
            lk::tgy::k_filter_tgy_wq<32><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
    } else {
        if (S.d <= 8)
            lk::tgy::k_filter_tgy<8><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
        else if (S.d <= 16)
            lk::tgy::k_filter_tgy<16><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
        else
            lk::tgy::k_filter_tgy<32><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
    }
    LK_LAUNCH_CHECK();
    return LK_OK;
}

}  // namespace lkh
