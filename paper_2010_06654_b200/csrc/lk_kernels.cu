// lk_kernels.cu -- the SIMT kernels of the exact-Lloyd iteration on sm_100a.
//
//   K1  k_assign_reg / k_assign_gen   fused fp32 difference-form distance +
//       per-row top-2 (replaces assign_full, lloyd.py:69-75 and
//       SequentialStrategy.seed, pruners.py:83-87 + _two_smallest :44-50).
//       Rows whose top-2 gap is inside the certified error bound are not
//       decided here; they go to K1x.
//   K1x k_recheck_fp64  exact re-decision of ambiguous rows in fp64 with
//       numpy's pairwise association order (core.py:98-108), so the label is
//       the oracle's label bit for bit, ties to the lowest index.
//   K2  k_filter_hamerly  drift decay of ub/lb + gate + tighten + compaction
//       (Hamerly.update_bounds pruners.py:234-239, assign_pass :244-254).
//   K4  k_refine_moved  fixed-point member-sum deltas of moved points
//       (refine_full lloyd.py:78-97, incrementally as in engine.py:134-172).
//   K5  k_update_centroids (+ its last block: global scalars) / k_half_sep  centroid divide with
//       the empty-cluster rule (lloyd.py:94-96), drifts (bounds.py:31-35),
//       s = half nearest-other distance (bounds.py:38-47), SSE (core.py:172).
#include <float.h>
#include <limits.h>
#include <math.h>

#include "lk_common.cuh"
#include "lk_exact.cuh"
#include "lk_internal.h"


namespace lk {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// shared epilogue: certify or flag one row, write label / bounds / worklists

// U1: certified upper bound on the true distance to candidate j1.
// L2: certified lower bound on the true distance to every other centroid.
// Must be called by every thread of the block (valid=false threads just vote).
__device__ __forceinline__ void row_finish(const DevState& S, bool valid, int64_t row, int j1,
                                           float U1, float L2, int64_t* stat) {
    bool certain = valid && (L2 > U1);
    bool flag = valid && !certain;
    int old = 0;
    bool moved = false;
    if (certain) {
        old = S.labels[row];
        moved = (old != j1);
        S.labels[row] = j1;
        if (S.strategy != LK_STRAT_LLOYD) {
            S.ub[row] = store_ub(S, U1, j1);
            write_lb_all(S, row, fmaxf(L2, 0.0f));
        }
    }
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    int64_t pos = block_append(moved, (unsigned long long*)(stat + LK_STAT_CHANGED), scr);
    if (moved) S.moved[pos] = make_int2((int)row, old);
    int64_t fpos = block_append(flag, (unsigned long long*)(stat + LK_STAT_FLAGGED), scr);
    if (flag) S.flagged[fpos] = (int)row;
}

__device__ __forceinline__ void top2_push(float D, int j, float& b1, int& j1, float& b2) {
    if (D < b1) {
        b2 = b1;
        b1 = D;
        j1 = j;
    } else {
        b2 = fminf(b2, D);
    }
}

// Certified bounds from fp32 difference-form squared distances b1 (label j1)
// and b2 (best other): see DESIGN.md "certifying labels".
__device__ __forceinline__ void simt_bounds(const DevState& S, float b1, int j1, float b2,
                                            float xnorm, float& U1, float& L2) {
    const float rho = simt_rel_err(S.d);
    const float cmax = S.scal[0];
    float a1 = kU32 * (xnorm + S.cnorm[j1]);
    float a2 = kU32 * (xnorm + cmax);
    U1 = (sqrtf(b1) + a1) * (1.0f + rho);
    L2 = isinf(b2) ? INFINITY : (sqrtf(b2) - a2) * (1.0f - rho);
}

// ---------------------------------------------------------------------------
// K1 (d <= 32): point rows in registers, centroid tiles in shared memory

template <int DP, int RPT>
__global__ void __launch_bounds__(kThreads) k_assign_reg(DevState S, const int32_t* rowlist,
                                                         const int64_t* rowcount, int64_t* stat,
                                                         int tile_k) {
    if (*S.done) return;
    extern __shared__ __align__(16) float csm[];  // [tile_k][DP]
    const int64_t m = rowlist ? *rowcount : S.n;
    const int ntiles = (S.k + tile_k - 1) / tile_k;
    const int64_t rpb = (int64_t)kThreads * RPT;
    int loaded = -1;
    for (int64_t base = (int64_t)blockIdx.x * rpb; base < m; base += (int64_t)gridDim.x * rpb) {
        float x[RPT][DP];
        float xn2[RPT];
        int64_t row[RPT];
        bool valid[RPT];
#pragma unroll
        for (int q = 0; q < RPT; q++) {
            int64_t r = base + threadIdx.x + (int64_t)q * kThreads;
            valid[q] = r < m;
            row[q] = valid[q] ? (rowlist ? (int64_t)rowlist[r] : r) : 0;
            const float* xp = S.X32 + row[q] * S.ldx;
            xn2[q] = 0.f;
#pragma unroll
            for (int z = 0; z < DP; z++) {
                float v = (valid[q] && z < S.d) ? __ldg(xp + z) : 0.f;
                x[q][z] = v;
                xn2[q] = fmaf(v, v, xn2[q]);
            }
        }
        float b1[RPT], b2[RPT];
        int j1[RPT];
#pragma unroll
        for (int q = 0; q < RPT; q++) { b1[q] = INFINITY; b2[q] = INFINITY; j1[q] = 0; }

        for (int tile = 0; tile < ntiles; tile++) {
            const int j0 = tile * tile_k;
            const int nj = min(tile_k, S.k - j0);
            if (loaded != tile) {
                __syncthreads();
                for (int e = threadIdx.x; e < nj * DP; e += kThreads) {
                    int jj = e / DP, z = e - jj * DP;
                    csm[e] = z < S.d ? S.C32[(int64_t)(j0 + jj) * S.ldc + z] : 0.f;
                }
                __syncthreads();
                loaded = tile;
            }
            for (int jj = 0; jj < nj; jj++) {
                float c[DP];
                if constexpr (DP % 4 == 0) {
#pragma unroll
                    for (int z = 0; z < DP; z += 4) {
                        float4 v = *reinterpret_cast<const float4*>(csm + jj * DP + z);
                        c[z] = v.x; c[z + 1] = v.y; c[z + 2] = v.z; c[z + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int z = 0; z < DP; z++) c[z] = csm[jj * DP + z];
                }
#pragma unroll
                for (int q = 0; q < RPT; q++) {
                    float acc = 0.f;
#pragma unroll
                    for (int z = 0; z < DP; z++) {
                        float t = x[q][z] - c[z];
                        acc = fmaf(t, t, acc);
                    }
                    top2_push(acc, j0 + jj, b1[q], j1[q], b2[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPT; q++) {
            float U1 = 0.f, L2 = 0.f;
            if (valid[q]) simt_bounds(S, b1[q], j1[q], b2[q], sqrtf(xn2[q]), U1, L2);
            row_finish(S, valid[q], row[q], j1[q], U1, L2, stat);
        }
    }
}

// ---------------------------------------------------------------------------
// K1 (d > 32): 256 rows x 32 centroids per pass, d streamed in chunks of 32

constexpr int kGenTJ = 32;
constexpr int kGenDC = 32;

__global__ void __launch_bounds__(kThreads) k_assign_gen(DevState S, const int32_t* rowlist,
                                                         const int64_t* rowcount, int64_t* stat) {
    if (*S.done) return;
    __shared__ float xs[kGenDC][kThreads + 1];
    __shared__ __align__(16) float cs[kGenDC][kGenTJ];
    __shared__ int64_t rows_s[kThreads];
    const int64_t m = rowlist ? *rowcount : S.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < m;
         base += (int64_t)gridDim.x * kThreads) {
        __syncthreads();
        {
            int64_t r = base + threadIdx.x;
            rows_s[threadIdx.x] = r < m ? (rowlist ? (int64_t)rowlist[r] : r) : -1;
        }
        __syncthreads();
        const bool valid = rows_s[threadIdx.x] >= 0;
        float b1 = INFINITY, b2 = INFINITY, xn2 = 0.f;
        int j1 = 0;
        for (int j0 = 0; j0 < S.k; j0 += kGenTJ) {
            float acc[kGenTJ];
#pragma unroll
            for (int c = 0; c < kGenTJ; c++) acc[c] = 0.f;
            for (int z0 = 0; z0 < S.d; z0 += kGenDC) {
                __syncthreads();
                // X chunk: warp w loads rows w*32 .. w*32+31, lane = dimension
                for (int rr = 0; rr < 32; rr++) {
                    int r = warp * 32 + rr;
                    int64_t gr = rows_s[r];
                    int z = z0 + lane;
                    xs[lane][r] = (gr >= 0 && z < S.d) ? __ldg(S.X32 + gr * S.ldx + z) : 0.f;
                }
                for (int e = threadIdx.x; e < kGenDC * kGenTJ; e += kThreads) {
                    int jj = e / kGenDC, z = e - jj * kGenDC;
                    int j = j0 + jj, zz = z0 + z;
                    cs[z][jj] = (j < S.k && zz < S.d) ? S.C32[(int64_t)j * S.ldc + zz] : 0.f;
                }
                __syncthreads();
#pragma unroll 4
                for (int z = 0; z < kGenDC; z++) {
                    float xv = xs[z][threadIdx.x];
                    if (j0 == 0) xn2 = fmaf(xv, xv, xn2);
#pragma unroll
                    for (int c4 = 0; c4 < kGenTJ; c4 += 4) {
                        float4 cv = *reinterpret_cast<const float4*>(&cs[z][c4]);
                        float t0 = xv - cv.x, t1 = xv - cv.y, t2 = xv - cv.z, t3 = xv - cv.w;
                        acc[c4] = fmaf(t0, t0, acc[c4]);
                        acc[c4 + 1] = fmaf(t1, t1, acc[c4 + 1]);
                        acc[c4 + 2] = fmaf(t2, t2, acc[c4 + 2]);
                        acc[c4 + 3] = fmaf(t3, t3, acc[c4 + 3]);
                    }
                }
            }
            const int nj = min(kGenTJ, S.k - j0);
#pragma unroll
            for (int c = 0; c < kGenTJ; c++)
                if (c < nj) top2_push(acc[c], j0 + c, b1, j1, b2);
        }
        float U1 = 0.f, L2 = 0.f;
        if (valid) simt_bounds(S, b1, j1, b2, sqrtf(xn2), U1, L2);
        row_finish(S, valid, valid ? rows_s[threadIdx.x] : 0, j1, U1, L2, stat);
    }
}

// ---------------------------------------------------------------------------
// K1x: exact fp64 recheck, numpy pairwise order (one block per flagged row)

// qscale_inline != nullptr: the assignment kernel already refined its own
// moved rows (lk_yy_fused.cu), so the rows moved here add their fixed-point
// deltas and changed count directly.
__global__ void __launch_bounds__(kThreads) k_recheck_fp64(DevState S, int64_t* stat,
                                                           const double* qscale_inline) {
    if (*S.done) return;
    extern __shared__ double xr[];  // [d]
    const int64_t m = stat[LK_STAT_FLAGGED];
    for (int64_t f = blockIdx.x; f < m; f += gridDim.x)
        recheck_row_block<kThreads>(S, stat, qscale_inline, S.flagged[f], xr);
}

// K1c: exact fp64 re-decision of the tensor-core pass's ambiguous rows over
// their collected candidates.  Every centroid outside the candidate set is
// provably strictly farther than the best candidate's upper bound, so the
// oracle's argmin lies in the set; the candidates' distances are computed
// exactly as the oracle computes them (numpy order, fp64), ties to the lowest
// index.  Rows whose set overflowed LK_MAX_CAND go to the fp32
// difference-form rescan (tight error bound), and from there to fp64 if needed.
// 16 lanes per ambiguous row (two rows per warp): lane i computes candidate
// slot i exactly (fp64, numpy's pairwise order), a 16-lane (value, index)
// top-2 merge picks the winner.
// numpy's pairwise leaf (pw_leaf) for len <= 32 with the row and the centroid
// in registers (compile-time indices): the same association and roundings.
__device__ __forceinline__ double pw_leaf32r(const float (&x)[32], const double (&c)[32], int len) {
    auto t2 = [&](int z) {
        const double t = __dsub_rn((double)x[z], c[z]);
        return __dmul_rn(t, t);
    };
    if (len < 8) {
        double res = 0.0;
#pragma unroll
        for (int z = 0; z < 8; z++)
            if (z < len) res = __dadd_rn(res, t2(z));
        return res;
    }
    const int main_end = len - (len % 8);
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = t2(j);
#pragma unroll
    for (int i = 1; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (8 * i < main_end) r[j] = __dadd_rn(r[j], t2(8 * i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll
    for (int z = 8; z < 32; z++)
        if (z >= main_end && z < len) res = __dadd_rn(res, t2(z));
    return res;
}

template <int kL>  // lanes per row; lane i takes candidate slots i, i + kL, ...
__global__ void __launch_bounds__(kThreads) k_recheck_cand(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    constexpr int kRows = kThreads / kL;
    const int sub = threadIdx.x & (kL - 1);
    const int64_t m = stat[LK_STAT_CANDIDATE];
    for (int64_t base = (int64_t)blockIdx.x * kRows; base < m; base += (int64_t)gridDim.x * kRows) {
        const int64_t e = base + threadIdx.x / kL;
        const bool ok = e < m;
        int64_t row = 0;
        int cnt = 0;
        if (ok) {
            row = S.cand_rows[e];
            cnt = S.cand_cnt[e];
        }
        const bool over_row = ok && (cnt < 1 || cnt > LK_MAX_CAND);
        double b1 = INFINITY, b2 = INFINITY;
        int j1 = 0x7fffffff;
        // d <= 32, fp32 rows, even d: the row and each candidate in registers
        // (vector loads: a thread reads whole rows, no 8x sector amplification)
        const bool regs = kL == 1 && S.d <= 32 && !S.X64 && (S.d & 1) == 0 && S.pw_len == 3 &&
                          (S.ldx & 3) == 0;
        if (ok && !over_row && regs) {
            float xr[32];
            const float4* xp = reinterpret_cast<const float4*>(S.X32 + row * S.ldx);
#pragma unroll
            for (int z4 = 0; z4 < 8; z4++) {
                const float4 v = 4 * z4 < S.d ? __ldg(xp + z4) : make_float4(0.f, 0.f, 0.f, 0.f);
                xr[4 * z4] = v.x; xr[4 * z4 + 1] = v.y; xr[4 * z4 + 2] = v.z; xr[4 * z4 + 3] = v.w;
            }
#pragma unroll
            for (int z = 0; z < 32; z++)
                if (z >= S.d) xr[z] = 0.f;
            for (int i = 0; i < cnt; i++) {
                const int j = S.cand_slots[e * LK_MAX_CAND + i];
                const double2* cp = reinterpret_cast<const double2*>(S.C64 + (int64_t)j * S.d);
                double c[32];
#pragma unroll
                for (int z2 = 0; z2 < 16; z2++) {
                    const double2 v = 2 * z2 < S.d ? __ldg(cp + z2) : make_double2(0.0, 0.0);
                    c[2 * z2] = v.x;
                    c[2 * z2 + 1] = v.y;
                }
                const double dd = __dsqrt_rn(pw_leaf32r(xr, c, S.d));
                merge_top2(b1, j1, b2, dd, j, INFINITY);
            }
        } else if (ok && !over_row) {
            for (int i = sub; i < cnt; i += kL) {
                const int j = S.cand_slots[e * LK_MAX_CAND + i];
                const double* cp = S.C64 + (int64_t)j * S.d;
                const double dd = __dsqrt_rn(S.X64 ? pw_dist2(S.X64 + row * S.d, cp, S.pw_prog, S.pw_len)
                                                   : pw_dist2(S.X32 + row * S.ldx, cp, S.pw_prog, S.pw_len));
                merge_top2(b1, j1, b2, dd, j, INFINITY);
            }
        }
#pragma unroll
        for (int o = kL / 2; o > 0; o >>= 1)
            merge_top2(b1, j1, b2, __shfl_xor_sync(LK_FULL_MASK, b1, o, kL),
                       __shfl_xor_sync(LK_FULL_MASK, j1, o, kL), __shfl_xor_sync(LK_FULL_MASK, b2, o, kL));
        const bool lead = ok && sub == 0;
        bool mv = false;
        int old = 0;
        if (lead && !over_row) {
            old = S.labels[row];
            mv = old != j1;
            S.labels[row] = j1;
            if (S.strategy != LK_STRAT_LLOYD) {
                S.ub[row] = store_ub(S, __double2float_ru(b1 * (1.0 + 1e-12)), j1);
                const float l2 = isinf(b2) ? INFINITY : __double2float_rd(b2 * (1.0 - 1e-12));
                write_lb_all(S, row, fminf(l2, S.cand_lb[e]));
            }
        }
        const bool over = lead && over_row;
        int64_t pos = block_append(mv, (unsigned long long*)(stat + LK_STAT_CHANGED), scr);
        if (mv) S.moved[pos] = make_int2((int)row, old);
        int64_t fpos = block_append(over, (unsigned long long*)(stat + LK_STAT_OVERFLOW), scr);
        if (over) S.ovf[fpos] = (int)row;
    }
}

// K2 on the tensor-core path (d >= 32: no tighten, the rescan decides): a pure
// streaming pass.  Four rows per thread (int4 / float4 loads and stores), one
// block-level scan and one global atomic per 1024 rows for the rescan list
// (one atomic per warp measured slower: 0.29 -> 0.45 ms on cfg5, the counter
// serializes), the active count accumulated locally.  20 B per row + 4 B per
// listed row.
__global__ void __launch_bounds__(kThreads) k_filter_hamerly_tc(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ int wsum[kThreads / 32 + 1];
    __shared__ unsigned long long sbase;
    const float dmax1 = S.scal[1], dmax2 = S.scal[2];
    const int amax = __float_as_int(S.scal[3]);
    const int64_t n = S.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t n_active = 0;
    // software pipeline: the next chunk's labels and bounds are requested
    // before this chunk's scan (two barriers and an atomic round trip), so the
    // block never waits on HBM and on the list slot one after the other
    const int64_t cstep = (int64_t)gridDim.x * kThreads * 4;
    int4 a4n = make_int4(0, 0, 0, 0);
    float4 u4n = make_float4(0.f, 0.f, 0.f, 0.f), l4n = u4n;
    {
        const int64_t i0 = (int64_t)blockIdx.x * kThreads * 4 + 4 * (int64_t)threadIdx.x;
        if (i0 + 3 < n) {
            a4n = __ldcs(reinterpret_cast<const int4*>(S.labels + i0));
            u4n = __ldcs(reinterpret_cast<const float4*>(S.ub + i0));
            l4n = __ldcs(reinterpret_cast<const float4*>(S.lb + i0));
        }
    }
    for (int64_t base = (int64_t)blockIdx.x * kThreads * 4; base < n; base += cstep) {
        const int64_t i0 = base + 4 * (int64_t)threadIdx.x;
        int a[4];
        float ub[4], lb[4];
        bool need[4];
        const bool full4 = i0 + 3 < n;
        if (full4) {
            const int4 a4 = a4n;
            const float4 u4 = u4n, l4 = l4n;
            if (i0 + cstep + 3 < n) {
                a4n = __ldcs(reinterpret_cast<const int4*>(S.labels + i0 + cstep));
                u4n = __ldcs(reinterpret_cast<const float4*>(S.ub + i0 + cstep));
                l4n = __ldcs(reinterpret_cast<const float4*>(S.lb + i0 + cstep));
            }
            a[0] = a4.x; a[1] = a4.y; a[2] = a4.z; a[3] = a4.w;
            ub[0] = u4.x; ub[1] = u4.y; ub[2] = u4.z; ub[3] = u4.w;
            lb[0] = l4.x; lb[1] = l4.y; lb[2] = l4.z; lb[3] = l4.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const bool ok = i0 + e < n;
                a[e] = ok ? S.labels[i0 + e] : 0;
                ub[e] = ok ? S.ub[i0 + e] : 0.f;
                lb[e] = ok ? S.lb[i0 + e] : 0.f;
            }
        }
        int cnt = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const bool ok = i0 + e < n;
            const float u = __fadd_ru(ub[e], __ldg(S.drift + a[e]));
            const float l = fmaxf(__fsub_rd(lb[e], a[e] == amax ? dmax2 : dmax1), 0.f);
            const float gate = fmaxf(l, __ldg(S.s_half + a[e]));
            need[e] = ok && !(gate > u);
            cnt += need[e];
            ub[e] = u;
            lb[e] = l;
        }
        if (full4) {
            __stcs(reinterpret_cast<float4*>(S.ub + i0), make_float4(ub[0], ub[1], ub[2], ub[3]));
            __stcs(reinterpret_cast<float4*>(S.lb + i0), make_float4(lb[0], lb[1], lb[2], lb[3]));
        } else {
#pragma unroll
            for (int e = 0; e < 4; e++)
                if (i0 + e < n) {
                    S.ub[i0 + e] = ub[e];
                    S.lb[i0 + e] = lb[e];
                }
        }
        n_active += cnt;
        // block exclusive scan of the counts, one atomic for the block's slots
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(LK_FULL_MASK, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < kThreads / 32; w++) {
                const int c = wsum[w];
                wsum[w] = tot;
                tot += c;
            }
            sbase = tot ? atomicAdd((unsigned long long*)(stat + LK_STAT_WORK), (unsigned long long)tot) : 0ull;
        }
        __syncthreads();
        int64_t pos = (int64_t)sbase + wsum[warp] + incl - cnt;
#pragma unroll
        for (int e = 0; e < 4; e++)
            if (need[e]) S.work[pos++] = (int)(i0 + e);
        __syncthreads();  // wsum / sbase reusable
    }
    warp_add(n_active, stat + LK_STAT_ACTIVE);
}

// ---------------------------------------------------------------------------
// K2: Hamerly bound decay + gate + tighten + compaction of the rows to rescan

__global__ void __launch_bounds__(kThreads) k_filter_hamerly(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    const float dmax1 = S.scal[1], dmax2 = S.scal[2];
    const int amax = __float_as_int(S.scal[3]);
    const float rho = simt_rel_err(S.d);
    const int64_t n = S.n;
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < n;
         base += (int64_t)gridDim.x * kThreads) {
        int64_t i = base + threadIdx.x;
        bool valid = i < n;
        bool active = false, need = false;
        if (valid) {
            int a = S.labels[i];
            float u = __fadd_ru(S.ub[i], S.drift[a]);
            float l = fmaxf(__fsub_rd(S.lb[i], a == amax ? dmax2 : dmax1), 0.f);
            float gate = fmaxf(l, S.s_half[a]);
            if (!(gate > u) && S.Xlo != nullptr && S.d >= 32) {
                // long rows on the tensor cores: skip the 2d-load tighten, the
                // full rescan decides the row anyway
                active = true;
                need = true;
            } else if (!(gate > u)) {
                active = true;
                const float* xp = S.X32 + i * S.ldx;
                const float* cp = S.C32 + (int64_t)a * S.ldc;
                float acc = 0.f, xn2 = 0.f;
                for (int z = 0; z < S.d; z++) {
                    float xv = __ldg(xp + z);
                    float t = xv - __ldg(cp + z);
                    acc = fmaf(t, t, acc);
                    xn2 = fmaf(xv, xv, xn2);
                }
                float U = (sqrtf(acc) + kU32 * (sqrtf(xn2) + S.cnorm[a])) * (1.0f + rho);
                u = fminf(u, U);
                need = !(gate > u);
            }
            S.ub[i] = u;
            S.lb[i] = l;
        }
        block_count(active, stat + LK_STAT_ACTIVE, scr);
        int64_t pos = block_append(need, (unsigned long long*)(stat + LK_STAT_WORK), scr);
        if (need) S.work[pos] = (int)i;
    }
}

// ---------------------------------------------------------------------------
// K4: fixed-point member-sum deltas of the moved rows


// G lanes per moved row (G = power of two >= min(d, 32)); warp-uniform loop.
// d in 17..32 (one lane per dimension): a warp takes 8 consecutive moved rows.
// The moved list of a centered tensor-core pass is in label-sorted order, so
// consecutive rows mostly leave the same cluster: the old-label side is summed
// in registers along a run of equal old labels and added once per run (integer
// sums: the result is the same in any order); the new side per row.
__device__ __forceinline__ void refine_batch32(const DevState& S, const double* qscale, int64_t e0,
                                               int64_t m) {
    constexpr int B = 8;
    const int lane = threadIdx.x & 31;
    int64_t* dS = S.delta;
    int64_t* dN = S.delta + (int64_t)S.k * S.d;
    int64_t* dQ = dN + S.k;
    int row[B], old[B], nw[B];
    double v[B];
#pragma unroll
    for (int b = 0; b < B; b++) {
        row[b] = -1;
        old[b] = -1;
        if (e0 + b < m) {
            const int2 mv = S.moved[e0 + b];
            row[b] = mv.x;
            old[b] = mv.y;
        }
    }
    const double sc = lane < S.d ? qscale[lane] : 0.0;
#pragma unroll
    for (int b = 0; b < B; b++) {
        nw[b] = row[b] >= 0 ? S.labels[row[b]] : 0;
        v[b] = (row[b] >= 0 && lane < S.d) ? load_xs(S, row[b], lane) : 0.0;
    }
    const double scq = qscale[S.d];
    long long run_q = 0, run_qq = 0;
    int run_old = -1, run_n = 0;
#pragma unroll
    for (int b = 0; b < B; b++) {
        if (row[b] < 0) continue;  // (warp-uniform)
        const long long q = lane < S.d ? __double2ll_rn(v[b] * sc) : 0;
        double x2 = v[b] * v[b];
        // ||x||^2 as k_refine_moved<32> forms it: lane z holds x_z^2 (one term per
        // lane), then the fixed xor tree
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x2 += __shfl_xor_sync(LK_FULL_MASK, x2, o);
        const long long qq = __double2ll_rn(x2 * scq);
        if (q) atomicAdd((unsigned long long*)(dS + (int64_t)nw[b] * S.d + lane), (unsigned long long)q);
        if (lane == 0) {
            atomicAdd((unsigned long long*)(dN + nw[b]), 1ull);
            atomicAdd((unsigned long long*)(dQ + nw[b]), (unsigned long long)qq);
        }
        if (old[b] != run_old) {
            if (run_old >= 0) {
                if (run_q) atomicAdd((unsigned long long*)(dS + (int64_t)run_old * S.d + lane), (unsigned long long)(-run_q));
                if (lane == 0) {
                    atomicAdd((unsigned long long*)(dN + run_old), (unsigned long long)(-(long long)run_n));
                    atomicAdd((unsigned long long*)(dQ + run_old), (unsigned long long)(-run_qq));
                }
            }
            run_old = old[b];
            run_q = 0;
            run_qq = 0;
            run_n = 0;
        }
        run_q += q;
        run_qq += qq;
        run_n++;
    }
    if (run_old >= 0) {
        if (run_q) atomicAdd((unsigned long long*)(dS + (int64_t)run_old * S.d + lane), (unsigned long long)(-run_q));
        if (lane == 0) {
            atomicAdd((unsigned long long*)(dN + run_old), (unsigned long long)(-(long long)run_n));
            atomicAdd((unsigned long long*)(dQ + run_old), (unsigned long long)(-run_qq));
        }
    }
}

// (its own kernel: the batched registers must not lower the occupancy of the
// one-row-per-warp kernel used for longer rows)
__global__ void __launch_bounds__(kThreads) k_refine_moved_b32(DevState S, int64_t* stat,
                                                               const double* qscale) {
    if (*S.done) return;
    const int64_t m = stat[LK_STAT_CHANGED];
    const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (kThreads / 32);
    for (int64_t e0 = gw * 8; e0 < m; e0 += nwarps * 8) refine_batch32(S, qscale, e0, m);
    if (blockIdx.x == 0 && threadIdx.x == 0) S.delta[(int64_t)S.k * S.d + 2 * S.k] = m;
}

template <int G>
__global__ void __launch_bounds__(kThreads) k_refine_moved(DevState S, int64_t* stat,
                                                           const double* qscale) {
    if (*S.done) return;
    const int64_t m = stat[LK_STAT_CHANGED];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % G;
    constexpr int kGroupsPerWarp = 32 / G;
    int64_t* dS = S.delta;
    int64_t* dN = S.delta + (int64_t)S.k * S.d;
    int64_t* dQ = dN + S.k;
    const int64_t stride = (int64_t)gridDim.x * (kThreads / 32) * kGroupsPerWarp;
    for (int64_t wb = ((int64_t)blockIdx.x * (kThreads / 32) + warp) * kGroupsPerWarp; wb < m;
         wb += stride) {
        const int64_t e = wb + lane / G;
        const bool ok = e < m;
        double x2 = 0.0;
        int64_t row = 0;
        int old = -1, nw = 0;
        if (ok) {
            int2 mv = S.moved[e];
            row = mv.x;
            old = mv.y;
            nw = S.labels[row];
            for (int z = sub; z < S.d; z += G) {
                double v = load_xs(S, row, z);
                x2 = fma(v, v, x2);
                long long q = __double2ll_rn(v * qscale[z]);
                if (q) {
                    atomicAdd((unsigned long long*)(dS + (int64_t)nw * S.d + z),
                              (unsigned long long)q);
                    if (old >= 0)
                        atomicAdd((unsigned long long*)(dS + (int64_t)old * S.d + z),
                                  (unsigned long long)(-q));
                }
            }
        }
        // deterministic group reduction of ||x||^2 (fixed xor tree)
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) x2 += __shfl_xor_sync(LK_FULL_MASK, x2, o, G);
        if (ok && sub == 0) {
            long long qq = __double2ll_rn(x2 * qscale[S.d]);
            atomicAdd((unsigned long long*)(dN + nw), 1ull);
            atomicAdd((unsigned long long*)(dQ + nw), (unsigned long long)qq);
            if (old >= 0) {
                atomicAdd((unsigned long long*)(dN + old), (unsigned long long)(-1ll));
                atomicAdd((unsigned long long*)(dQ + old), (unsigned long long)(-qq));
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // local changed count rides along in the all-reduce payload
        S.delta[(int64_t)S.k * S.d + 2 * S.k] = m;
    }
}

// ---------------------------------------------------------------------------
// K5: centroid update (one warp per centroid) and global scalars

// One block (the last of k_update_centroids): SSE (fixed reduction order),
// max ||c||, top-2 drift, group drifts, done flag.
__device__ __forceinline__ void update_global_block(const DevState& S, const double* sse_part) {
    const int t = *S.iter;
    __shared__ double ssum[kThreads / 32];
    __shared__ float smax[kThreads / 32], sd1[kThreads / 32], sd2[kThreads / 32];
    __shared__ int sarg[kThreads / 32];
    __shared__ float sg[1024];  // group drift maxima (t <= 1024)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const bool sg_ok = S.gdrift && S.t_groups > 0 && S.t_groups <= 1024;
    // everything the block reads is issued up front (one dependent L2 round
    // trip instead of one per phase): the changed count, the counters of the
    // iteration, the cumulative group drifts
    int64_t changed = 0, curv = 0;
    if (tid == 0) changed = __ldcg(S.delta + (int64_t)S.k * S.d + 2 * S.k);
    if (tid < LK_NSTAT) curv = __ldcg(S.cur + tid);
    float dgc = 0.f;
    if (S.gdrift && S.lazy && tid < S.t_groups) dgc = __ldcg(S.dgcum + tid);
    for (int g = tid; g < S.t_groups && g < 1024; g += blockDim.x) sg[g] = 0.f;
    __syncthreads();
    double acc = 0.0;
    float cm = 0.f, d1 = -1.f, d2 = -1.f;
    int a1 = -1;
    for (int j = tid; j < S.k; j += blockDim.x) {
        acc += __ldcg(sse_part + j);
        cm = fmaxf(cm, __ldcg(S.cnorm + j));
        float dj = __ldcg(S.drift + j);
        if (dj > d1) { d2 = d1; d1 = dj; a1 = j; }
        else d2 = fmaxf(d2, dj);
        // group drifts (Yinyang): max drift over each group's members
        if (sg_ok) atomicMax(reinterpret_cast<int*>(sg + __ldg(S.group_of + j)), __float_as_int(dj));
    }
    // fixed-order reductions: xor butterflies in each warp, then the warps in order
    auto merge_d = [](float& x1, float& x2, int& xa, float o1, float o2, int oa) {
        if (o1 > x1 || (o1 == x1 && oa >= 0 && (xa < 0 || oa < xa))) {
            x2 = fmaxf(x1, o2);
            x1 = o1;
            xa = oa;
        } else {
            x2 = fmaxf(x2, o1);
        }
    };
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(LK_FULL_MASK, acc, o);
        cm = fmaxf(cm, __shfl_xor_sync(LK_FULL_MASK, cm, o));
        const float o1 = __shfl_xor_sync(LK_FULL_MASK, d1, o), o2 = __shfl_xor_sync(LK_FULL_MASK, d2, o);
        const int oa = __shfl_xor_sync(LK_FULL_MASK, a1, o);
        merge_d(d1, d2, a1, o1, o2, oa);
    }
    if (lane == 0) { ssum[wid] = acc; smax[wid] = cm; sd1[wid] = d1; sd2[wid] = d2; sarg[wid] = a1; }
    __syncthreads();
    if (tid == 0) {
        double ss = ssum[0];
        float mx = smax[0], x1 = sd1[0], x2 = sd2[0];
        int xa = sarg[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
            ss += ssum[w];
            mx = fmaxf(mx, smax[w]);
            merge_d(x1, x2, xa, sd1[w], sd2[w], sarg[w]);
        }
        ssum[0] = ss;
        smax[0] = fmaxf(x1, 0.f);  // (the max drift, for the cumulative offset below)
        S.scal[0] = mx;
        S.scal[1] = fmaxf(x1, 0.f);
        S.scal[2] = fmaxf(x2, 0.f);
        S.scal[3] = __int_as_float(xa);
        S.delta[(int64_t)S.k * S.d + 2 * S.k] = 0;
        if (t >= 1 && t <= S.t_max) S.sse[t - 1] = ss;
        if (t >= 1 && t <= S.t_max) S.tstamp[2 * t + 1] = globaltimer_ns();  // the update's end
        if (S.hlog_inline && t >= 1 && t <= S.t_max) {
            // close the iteration's label-history segment (k_log_history's job on
            // the other paths); curv = this thread's cur[LK_STAT_CHANGED] (slot 0)
            const int64_t base = __ldcg(S.hlog_off + (t - 1));
            const int64_t mlog = curv;
            S.hlog_off[t] = (base >= 0 && base + mlog <= S.hlog_cap) ? base + mlog : -1;
        }
        *S.iter = t + 1;
        if (changed == 0) *S.done = 1;
    }
    const int64_t chg0 = __shfl_sync(LK_FULL_MASK, changed, 0);  // (warp 0: thread 0's load)
    if (tid < LK_NSTAT) {
        // the iteration's counters (the global changed count in its slot) into
        // the stats row, then cleared for the next iteration
        const int64_t v = tid == LK_STAT_CHANGED_GLOBAL ? chg0 : curv;
        if (t >= 1 && t <= S.t_max) S.stats[(int64_t)(t - 1) * LK_NSTAT + tid] = v;
        S.cur[tid] = 0;
    }
    // s_half is rebuilt by k_half_sep's atomicMin: start from +inf
    // (gate off: s = 0 never prunes)
    for (int j = tid; j < S.k; j += blockDim.x) S.s_half[j] = S.sgate ? INFINITY : 0.f;
    if (S.gdrift) {
        if (sg_ok) {
            __syncthreads();
            for (int g = tid; g < S.t_groups; g += blockDim.x) S.gdrift[g] = sg[g];
            if (S.lazy)
                for (int g = tid; g < S.t_groups; g += blockDim.x)
                    S.dgcum[g] = __fadd_ru(g == tid ? dgc : __ldcg(S.dgcum + g), sg[g]);
            if (S.lazy && tid == 0) S.scal[4] = __fadd_ru(__ldcg(S.scal + 4), smax[0]);
        } else {
            __syncthreads();
            for (int g = tid; g < S.t_groups; g += blockDim.x) S.gdrift[g] = 0.f;
            __syncthreads();
            for (int j = tid; j < S.k; j += blockDim.x) atomic_max_pos(S.gdrift + S.group_of[j], __ldcg(S.drift + j));
            if (S.lazy) {
                __syncthreads();
                for (int g = tid; g < S.t_groups; g += blockDim.x)
                    S.dgcum[g] = __fadd_ru(S.dgcum[g], S.gdrift[g]);
                if (tid == 0) S.scal[4] = __fadd_ru(S.scal[4], smax[0]);
            }
        }
    }
}

// One centroid j per warp (warp-uniform call): divide with the empty rule,
// drift (+ cumulative drift), fp32 / tf32 copies, norms, SSE part; zeroes the
// consumed delta payload of j.
__device__ __forceinline__ void update_centroid_warp(const DevState& S, int j, const double* qinv,
                                                     double* sse_part) {
    const int lane = threadIdx.x & 31;
    int64_t* dS = S.delta;
    int64_t* dN = S.delta + (int64_t)S.k * S.d;
    int64_t* dQ = dN + S.k;
    if (j < S.k) {
    // (body indented one level less than its scope, to keep the diff small)
    int64_t cnt = S.counts[j] + dN[j];
    int64_t qs = S.qsum[j] + dQ[j];
    const int64_t cj = S.colperm ? S.ginv[j] : j;  // B-operand column of centroid j
    double s2 = 0.0, drift2 = 0.0, cn2 = 0.0, c2 = 0.0;
    for (int z = lane; z < S.d; z += 32) {
        int64_t sv = S.sums[(int64_t)j * S.d + z] + dS[(int64_t)j * S.d + z];
        S.sums[(int64_t)j * S.d + z] = sv;
        double old = S.C64[(int64_t)j * S.d + z];
        double c = old;
        if (cnt > 0) {
            // (sums are of x - m: sr / cnt is the mean's offset from m)
            double sr = (double)sv * qinv[z];
            c = __ldg(S.xshift + z) + sr / (double)cnt;
            s2 = fma(sr, sr, s2);
        }
        S.C64_prev[(int64_t)j * S.d + z] = old;
        S.C64[(int64_t)j * S.d + z] = c;
        double dd = c - old;
        drift2 = fma(dd, dd, drift2);
        float c32 = (float)c;
        S.C32[(int64_t)j * S.ldc + z] = c32;
        if (S.Cg) S.Cg[(int64_t)S.ginv[j] * S.ldc + z] = c32;
        cn2 = fma((double)c32, (double)c32, cn2);
        if (S.Chi) {
            float hi = tf32_trunc(c32);
            S.Chi[cj * S.ldc + z] = hi;
            S.Clo[cj * S.ldc + z] = c32 - hi;
            c2 = fma(c, c, c2);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        s2 += __shfl_xor_sync(LK_FULL_MASK, s2, o);
        drift2 += __shfl_xor_sync(LK_FULL_MASK, drift2, o);
        cn2 += __shfl_xor_sync(LK_FULL_MASK, cn2, o);
        c2 += __shfl_xor_sync(LK_FULL_MASK, c2, o);
    }
    if (lane == 0) {
        if (S.cn2) S.cn2[cj] = (float)c2;
        S.counts[j] = cnt;
        S.qsum[j] = qs;
        const float dj = drift2 > 0.0 ? __double2float_ru(sqrt(drift2) * (1.0 + 1e-12)) : 0.f;
        S.drift[j] = dj;
        if (S.lazy) {
            const float dc = __fadd_ru(S.dcum[j], dj);
            S.dcum[j] = dc;
            if (S.dcum_col) S.dcum_col[cj] = dc;
        }
        S.cnorm[j] = __double2float_ru(sqrt(cn2) * (1.0 + 1e-12));
        sse_part[j] = cnt > 0 ? ((double)qs * qinv[S.d] - s2 / (double)cnt) : 0.0;
        // the delta payload is consumed: zero it for the next iteration
        dN[j] = 0;
        dQ[j] = 0;
    }
    for (int z = lane; z < S.d; z += 32) dS[(int64_t)j * S.d + z] = 0;
    }
}

__global__ void __launch_bounds__(kThreads) k_update_centroids(DevState S, const double* qscale,
                                                               const double* qinv,
                                                               double* sse_part) {
    pdl_wait();
    pdl_trigger();
    if (*S.done) return;
    if (threadIdx.x == 0) {
        // the update phase's start on the device clock (earliest block)
        const int t = *S.iter;
        if (t >= 1 && t <= S.t_max)
            atomicMin(reinterpret_cast<unsigned long long*>(S.tstamp + 2 * t), globaltimer_ns());
    }
    const int warp = threadIdx.x >> 5;
    const int j = blockIdx.x * (kThreads / 32) + warp;
    update_centroid_warp(S, j, qinv, sse_part);
    // the last block to finish reduces the per-centroid results (threadfence
    // reduction: its reads see every block's writes)
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned tk = atomicAdd((unsigned*)(S.done + 2), 1u);
        last = tk == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        update_global_block(S, sse_part);
        if (threadIdx.x == 0) S.done[2] = 0;
    }
}

// s_j = 1/2 min_{j' != j} |c_j - c_j'|, certified lower bound (fp32 diff form).
// 64 x 64 (j, j') tiles per block, 4 x 4 pairs per thread, d streamed in
// chunks of 32 through shared memory; per-j minima combined with atomicMin
// on the (nonnegative) float bits.  s_half must be +inf-filled beforehand.
constexpr int kHsDC = 32;

// P x P pairs per thread: tiles of T = 16 P centroids (P = 4: 64 x 64 tiles; small k
// takes smaller tiles so that the grid still fills the GPU -- k = 256 is 16
// blocks of 64 x 64 but 256 of 16 x 16).  The sum over d of a pair runs in the
// same order whatever P, so s_half does not depend on it.
template <int P>
__device__ __forceinline__ void half_sep_tile(const DevState& S, int tj, int tjp) {
    constexpr int T = 16 * P;
    __shared__ float ta[kHsDC][T + 4];
    __shared__ float tb[kHsDC][T + 4];
    const int j0 = tj * T, jp0 = tjp * T;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads
    float acc[P][P];
#pragma unroll
    for (int a = 0; a < P; a++)
#pragma unroll
        for (int b = 0; b < P; b++) acc[a][b] = 0.f;
    for (int z0 = 0; z0 < S.d; z0 += kHsDC) {
        const int zn = min(kHsDC, S.d - z0);  // (short rows: only the real dimensions)
        __syncthreads();
        for (int e = threadIdx.x; e < T * zn; e += kThreads) {
            int r = e / zn, z = e % zn;
            int zz = z0 + z;
            ta[z][r] = (j0 + r < S.k) ? S.C32[(int64_t)(j0 + r) * S.ldc + zz] : 0.f;
            tb[z][r] = (jp0 + r < S.k) ? S.C32[(int64_t)(jp0 + r) * S.ldc + zz] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int z = 0; z < zn; z++) {
            float av[P], bv[P];
#pragma unroll
            for (int a = 0; a < P; a++) av[a] = ta[z][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < P; b++) bv[b] = tb[z][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < P; a++)
#pragma unroll
                for (int b = 0; b < P; b++) {
                    float t = av[a] - bv[b];
                    acc[a][b] = fmaf(t, t, acc[a][b]);
                }
        }
    }
    const float rho = simt_rel_err(S.d);
#pragma unroll
    for (int a = 0; a < P; a++) {
        const int j = j0 + ty + 16 * a;
        float best = INFINITY;
        if (j < S.k) {
            const float cj = S.cnorm[j];
#pragma unroll
            for (int b = 0; b < P; b++) {
                const int jp = jp0 + tx + 16 * b;
                if (jp < S.k && jp != j) {
                    float lbd = (sqrtf(acc[a][b]) - kU32 * (cj + S.cnorm[jp])) * (1.0f - rho);
                    best = fminf(best, fmaxf(0.5f * lbd * (1.0f - 4.0f * kU32), 0.f));
                }
            }
        }
        // min over the 16 threads sharing row j (same ty, lanes tx 0..15)
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) best = fminf(best, __shfl_xor_sync(LK_FULL_MASK, best, o, 16));
        if (tx == 0 && j < S.k && best < INFINITY) atomicMin((int*)(S.s_half + j), __float_as_int(best));
    }
}

template <int P>
__global__ void __launch_bounds__(kThreads) k_half_sep(DevState S) {
    pdl_wait();
    pdl_trigger();
    if (*S.done) return;
    half_sep_tile<P>(S, blockIdx.y, blockIdx.x);
}

// Label history as a log: the moved rows of iteration t with their new label
// (iteration 1 moves every row off -1).  The host rebuilds per-iteration label
// vectors from it (lloyd.py:140 assign_history) without copying n labels per
// iteration.  Runs after the refine kernel, before the update.
__device__ __forceinline__ void log_history_grid(const DevState& S) {
    const int t = *S.iter;
    if (t < 1 || t > S.t_max) return;
    const int64_t m = S.cur[LK_STAT_CHANGED];
    const int64_t base = S.hlog_off[t - 1];
    const bool ok = base >= 0 && base + m <= S.hlog_cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) S.hlog_off[t] = ok ? base + m : -1;
    if (!ok) return;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int row = S.moved[e].x;
        S.hlog[base + e] = make_int2(row, S.labels[row]);
    }
}

__global__ void k_log_history(DevState S) {
    pdl_wait();
    pdl_trigger();
    if (*S.done) return;
    log_history_grid(S);
}

__global__ void k_fill_inf(DevState S) {
    if (*S.done) return;
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < S.k) S.s_half[j] = INFINITY;
}

// Per-dimension range of the local rows as order keys (fkey: the int32 order
// of the fp32 values): qexp[d + 1 + z] = max key of x_z, qexp[2d + 1 + z] =
// max key of -x_z (fp64 input: rounded outward to fp32).  Multi-GPU callers
// all-reduce(max) the whole qexp buffer before lk_set_quant.  For d <= 1024
// each thread owns one dimension (blockDim a multiple of d), block maxima in
// shared memory, then one global atomic per block and key.
__device__ __forceinline__ int fkey(float f) {
    const int b = __float_as_int(f);
    return b >= 0 ? b : (b ^ 0x7fffffff);
}

__global__ void __launch_bounds__(1024) k_scan_range(DevState S) {
    extern __shared__ int skey[];  // [2d]
    const int d = S.d;
    for (int z = threadIdx.x; z < 2 * d; z += blockDim.x) skey[z] = INT_MIN;
    __syncthreads();
    const auto val = [&](int64_t row, int z, float& hi, float& lo) {
        if (S.X64) {
            const double v = S.X64[row * d + z];
            hi = fmaxf(hi, __double2float_ru(v));
            lo = fminf(lo, __double2float_rd(v));
        } else {
            const float v = __ldg(S.X32 + row * S.ldx + z);
            hi = fmaxf(hi, v);
            lo = fminf(lo, v);
        }
    };
    if (d <= 1024) {
        const int per = blockDim.x / d;
        if ((int)threadIdx.x < per * d) {
            const int z = threadIdx.x % d, r0 = threadIdx.x / d;
            float hi = -INFINITY, lo = INFINITY;
            for (int64_t row = (int64_t)blockIdx.x * per + r0; row < S.n;
                 row += (int64_t)gridDim.x * per)
                val(row, z, hi, lo);
            if (hi >= lo) {
                atomicMax(skey + z, fkey(hi));
                atomicMax(skey + d + z, fkey(-lo));
            }
        }
    } else {
        for (int64_t row = blockIdx.x; row < S.n; row += gridDim.x)
            for (int z = threadIdx.x; z < d; z += blockDim.x) {
                float hi = -INFINITY, lo = INFINITY;
                val(row, z, hi, lo);
                atomicMax(skey + z, fkey(hi));
                atomicMax(skey + d + z, fkey(-lo));
            }
    }
    __syncthreads();
    for (int z = threadIdx.x; z < 2 * d; z += blockDim.x)
        if (skey[z] != INT_MIN) atomicMax(S.qexp + d + 1 + z, skey[z]);
}

}  // namespace lk

// ---------------------------------------------------------------------------
// launchers

namespace lkh {

using namespace lk;

static int grid_for(int64_t work_items, int per_block, int max_blocks) {
    int64_t b = (work_items + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

// A short row list (the tensor-core pass's candidate overflow: ~0.003% of the
// rows) with d <= 32: one warp per row, lane L scans centroids L, L + 32, ...
// with k_assign_reg's arithmetic (difference form, fmaf chain in dimension
// order, first minimum kept), then a (value, index) warp merge and the same
// certification; a block-per-256-rows scan would leave all but a few SMs idle.
template <int DP>
__global__ void __launch_bounds__(kThreads) k_assign_warp(DevState S, const int32_t* rowlist,
                                                          const int64_t* rowcount, int64_t* stat) {
    if (*S.done) return;
    const int64_t m = *rowcount;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t e = gw; e < m; e += nw) {
        const int64_t row = rowlist[e];
        const float* xp = S.X32 + row * S.ldx;
        float x[DP];
        float xn2 = 0.f;
#pragma unroll
        for (int z = 0; z < DP; z++) {
            x[z] = z < S.d ? __ldg(xp + z) : 0.f;
            xn2 = fmaf(x[z], x[z], xn2);
        }
        float b1 = INFINITY, b2 = INFINITY;
        int j1 = 0;
        for (int j = lane; j < S.k; j += 32) {
            const float* cp = S.C32 + (int64_t)j * S.ldc;
            float c[DP];
            if (DP >= 4 && (S.ldc & 3) == 0) {
                // the lane's centroid row as float4 (rows are zero-padded to ldc)
#pragma unroll
                for (int z = 0; z < DP; z += 4) {
                    const float4 v = (z < S.ldc) ? __ldg(reinterpret_cast<const float4*>(cp + z))
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
                    c[z] = v.x; c[z + 1] = v.y; c[z + 2] = v.z; c[z + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int z = 0; z < DP; z++) c[z] = z < S.d ? __ldg(cp + z) : 0.f;
            }
            float acc = 0.f;
#pragma unroll
            for (int z = 0; z < DP; z++) {
                const float t = x[z] - (z < S.d ? c[z] : 0.f);
                acc = fmaf(t, t, acc);
            }
            top2_push(acc, j, b1, j1, b2);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ob1 = __shfl_xor_sync(LK_FULL_MASK, b1, o), ob2 = __shfl_xor_sync(LK_FULL_MASK, b2, o);
            const int oj1 = __shfl_xor_sync(LK_FULL_MASK, j1, o);
            if (ob1 < b1 || (ob1 == b1 && oj1 < j1)) {
                b2 = fminf(b1, ob2);
                b1 = ob1;
                j1 = oj1;
            } else {
                b2 = fminf(b2, ob1);
            }
        }
        if (lane == 0) {
            float U1, L2;
            simt_bounds(S, b1, j1, b2, sqrtf(xn2), U1, L2);
            if (L2 > U1) {
                const int old = S.labels[row];
                S.labels[row] = j1;
                if (S.strategy != LK_STRAT_LLOYD) {
                    S.ub[row] = store_ub(S, U1, j1);
                    write_lb_all(S, row, fmaxf(L2, 0.0f));
                }
                if (old != j1) {
                    const unsigned long long p = atomicAdd((unsigned long long*)(stat + LK_STAT_CHANGED), 1ull);
                    S.moved[p] = make_int2((int)row, old);
                }
            } else {
                const unsigned long long p = atomicAdd((unsigned long long*)(stat + LK_STAT_FLAGGED), 1ull);
                S.flagged[p] = (int)row;
            }
        }
    }
}

template <int DP, int RPT>
static lk_status launch_reg(const DevState& S, const int32_t* rowlist, const int64_t* rowcount,
                            int64_t* stat, int64_t max_rows, int sms, cudaStream_t st) {
    int tile_k = S.k;
    const int smem_cap = 96 * 1024;
    if ((int64_t)tile_k * DP * 4 > smem_cap) tile_k = smem_cap / (DP * 4);
    size_t smem = (size_t)tile_k * DP * 4;
    int grid = grid_for(max_rows, kThreads * RPT, sms * 6);
    k_assign_reg<DP, RPT><<<grid, kThreads, smem, st>>>(S, rowlist, rowcount, stat, tile_k);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

// A short device-counted row list (the candidate overflow), warp per row for d <= 32.
lk_status launch_assign_short(const DevState& S, const int32_t* rowlist, const int64_t* rowcount,
                              int64_t* stat, int64_t max_rows, int sms, cudaStream_t st) {
    const int d = S.d;
    if (d > 32) return launch_assign_simt(S, rowlist, rowcount, stat, max_rows, sms, st);
    const int grid = grid_for(max_rows, kThreads / 32, sms * 4);
    if (d <= 2) k_assign_warp<2><<<grid, kThreads, 0, st>>>(S, rowlist, rowcount, stat);
    else if (d <= 4) k_assign_warp<4><<<grid, kThreads, 0, st>>>(S, rowlist, rowcount, stat);
    else if (d <= 8) k_assign_warp<8><<<grid, kThreads, 0, st>>>(S, rowlist, rowcount, stat);
    else if (d <= 16) k_assign_warp<16><<<grid, kThreads, 0, st>>>(S, rowlist, rowcount, stat);
    else k_assign_warp<32><<<grid, kThreads, 0, st>>>(S, rowlist, rowcount, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_assign_simt(const DevState& S, const int32_t* rowlist, const int64_t* rowcount,
                             int64_t* stat, int64_t max_rows, int sms, cudaStream_t st) {
    const int d = S.d;
    if (d <= 2) return launch_reg<2, 2>(S, rowlist, rowcount, stat, max_rows, sms, st);
    if (d <= 4) return launch_reg<4, 2>(S, rowlist, rowcount, stat, max_rows, sms, st);
    if (d <= 8) return launch_reg<8, 2>(S, rowlist, rowcount, stat, max_rows, sms, st);
    if (d <= 16) return launch_reg<16, 2>(S, rowlist, rowcount, stat, max_rows, sms, st);
    if (d <= 32) return launch_reg<32, 1>(S, rowlist, rowcount, stat, max_rows, sms, st);
    int grid = grid_for(max_rows, kThreads, sms * 4);
    k_assign_gen<<<grid, kThreads, 0, st>>>(S, rowlist, rowcount, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_recheck(const DevState& S, int64_t* stat, int64_t max_rows, int sms,
                         cudaStream_t st, const double* qscale_inline) {
    size_t smem = (size_t)S.d * sizeof(double);  // <= 48 KB for d <= 6144
    int grid = grid_for(max_rows, 1, sms * 2);
    k_recheck_fp64<<<grid, kThreads, smem, st>>>(S, stat, qscale_inline);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_recheck_cand(const DevState& S, int64_t* stat, int64_t max_rows, int sms,
                              cudaStream_t st) {
    // long rows: one candidate per lane (cfg4: 0.39 -> 0.19 ms); short rows
    // (few candidates, cheap distances): one thread per row is fastest
    if (S.d > 64) {
        k_recheck_cand<LK_MAX_CAND><<<grid_for(max_rows, kThreads / LK_MAX_CAND, sms * 8), kThreads, 0, st>>>(S, stat);
    } else {
        k_recheck_cand<1><<<grid_for(max_rows, kThreads, sms * 4), kThreads, 0, st>>>(S, stat);
    }
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_filter_hamerly(const DevState& S, int64_t* stat, int sms, cudaStream_t st) {
    if (S.Xlo != nullptr && S.d >= 32 && (reinterpret_cast<uintptr_t>(S.labels) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(S.ub) & 15) == 0 && (reinterpret_cast<uintptr_t>(S.lb) & 15) == 0) {
        k_filter_hamerly_tc<<<grid_for(S.n, kThreads * 4, sms * 8), kThreads, 0, st>>>(S, stat);
        LK_LAUNCH_CHECK();
        return LK_OK;
    }
    int grid = grid_for(S.n, kThreads, sms * 8);
    k_filter_hamerly<<<grid, kThreads, 0, st>>>(S, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_refine(const DevState& S, int64_t* stat, const double* qscale, int64_t max_rows,
                        int sms, cudaStream_t st) {
    int g = 32;
    if (S.d <= 1) g = 1;
    else if (S.d <= 2) g = 2;
    else if (S.d <= 4) g = 4;
    else if (S.d <= 8) g = 8;
    else if (S.d <= 16) g = 16;
    int grid = grid_for(max_rows, kThreads / g, sms * 8);
    switch (g) {
        case 1: k_refine_moved<1><<<grid, kThreads, 0, st>>>(S, stat, qscale); break;
        case 2: k_refine_moved<2><<<grid, kThreads, 0, st>>>(S, stat, qscale); break;
        case 4: k_refine_moved<4><<<grid, kThreads, 0, st>>>(S, stat, qscale); break;
        case 8: k_refine_moved<8><<<grid, kThreads, 0, st>>>(S, stat, qscale); break;
        case 16: k_refine_moved<16><<<grid, kThreads, 0, st>>>(S, stat, qscale); break;
        default:
            if (S.d <= 32) k_refine_moved_b32<<<grid_for(max_rows, kThreads / 4, sms * 8), kThreads, 0, st>>>(S, stat, qscale);
            else k_refine_moved<32><<<grid, kThreads, 0, st>>>(S, stat, qscale);
            break;
    }
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_update(const DevState& S, const double* qscale, const double* qinv,
                        double* sse_part, bool need_half, cudaStream_t st) {
    int grid = (S.k + (kThreads / 32) - 1) / (kThreads / 32);
    LK_CUDA_CHECK(lk::launch_pdl(k_update_centroids, dim3(grid), dim3(kThreads), 0, st, S, qscale, qinv, sse_part));
    LK_LAUNCH_CHECK();
    if (need_half) {
        // the largest tile whose grid still has >= 128 blocks (else 16 x 16 tiles)
        auto blocks = [&](int T) { const int g = (S.k + T - 1) / T; return g * g; };
        if (blocks(64) >= 128) {
            dim3 g((S.k + 63) / 64, (S.k + 63) / 64);
            LK_CUDA_CHECK(lk::launch_pdl(k_half_sep<4>, g, dim3(kThreads), 0, st, S));
        } else if (blocks(32) >= 128) {
            dim3 g((S.k + 31) / 32, (S.k + 31) / 32);
            LK_CUDA_CHECK(lk::launch_pdl(k_half_sep<2>, g, dim3(kThreads), 0, st, S));
        } else {
            dim3 g((S.k + 15) / 16, (S.k + 15) / 16);
            LK_CUDA_CHECK(lk::launch_pdl(k_half_sep<1>, g, dim3(kThreads), 0, st, S));
        }
        LK_LAUNCH_CHECK();
    }
    return LK_OK;
}

// ---------------------------------------------------------------------------
// k-means++ seeding (init_kmeanspp, core.py:192-217): one D^2 update
//   d2[i] = (first ? s_i : min(d2[i], s_i)),  s_i = np.sum((x_i - c) ** 2)
// in fp64 with numpy's pairwise order over d (the same values the reference's
// numpy expression produces, so the host's draws are identical).

__global__ void k_d2_update(const float* __restrict__ x32, const double* __restrict__ x64, int64_t n,
                            int d, int64_t ldx, const double* __restrict__ c, double* __restrict__ d2,
                            int first, PwProg prog) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double sum;
        if (prog.len == 3) {
            sum = x64 ? pw_leaf(x64 + i * ldx, c, 0, d) : pw_leaf(x32 + i * ldx, c, 0, d);
        } else {
            double st[24];
            int sp = 0;
            for (int p = 0; p < prog.len; p += 3) {
                if (prog.ops[p] == 0) {
                    st[sp++] = x64 ? pw_leaf(x64 + i * ldx, c, prog.ops[p + 1], prog.ops[p + 2])
                                   : pw_leaf(x32 + i * ldx, c, prog.ops[p + 1], prog.ops[p + 2]);
                } else {
                    const double b = st[--sp], a = st[--sp];
                    st[sp++] = __dadd_rn(a, b);
                }
            }
            sum = st[0];
        }
        d2[i] = first ? sum : fmin(d2[i], sum);
    }
}

lk_status launch_d2_update(const float* x32, const double* x64, int64_t n, int d, int64_t ldx,
                           const double* c, double* d2, int first, const PwProg& prog,
                           cudaStream_t st) {
    if (n <= 0) return LK_OK;
    const int64_t blocks = (n + kThreads - 1) / kThreads;
    k_d2_update<<<(unsigned)(blocks < 4096 ? blocks : 4096), kThreads, 0, st>>>(x32, x64, n, d, ldx, c,
                                                                                d2, first, prog);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_log_history(const DevState& S, int sms, cudaStream_t st) {
    if (!S.hlog) return LK_OK;
    LK_CUDA_CHECK(lk::launch_pdl(k_log_history, dim3(sms * 2), dim3(kThreads), 0, st, S));
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status init_simt_attributes() {

    const int cap = 96 * 1024;
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_reg<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_reg<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_reg<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_reg<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_reg<32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
    return LK_OK;
}

lk_status launch_scan_exp(const DevState& S, int sms, cudaStream_t st) {
    const int d = S.d;
    const int bs = d <= 1024 ? d * (1024 / d) : 1024;
    const size_t smem = (size_t)2 * d * sizeof(int);
    if (smem > 48 * 1024)
        LK_CUDA_CHECK(cudaFuncSetAttribute(k_scan_range, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    const int64_t rows_per_block = d <= 1024 ? bs / d : 1;
    k_scan_range<<<grid_for(S.n, (int)rows_per_block * 8, sms * 2), bs, smem, st>>>(S);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

}  // namespace lkh
