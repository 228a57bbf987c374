// lk_yinyang.cu -- group-bound (Yinyang) pruning on the GPU.
//
// Reference: Yinyang.update_bounds / assign_pass (pruners.py:418-497),
// group_centroids (bounds.py:175-196).  Per point: label a, upper bound ub,
// and one lower bound per centroid group (lb[n, t]).  Labels never depend on
// the grouping, so t and the groups are chosen for bandwidth.
//
// Work-efficient mapping: instead of one thread walking a point's failing
// groups (warp-divergent: the warp would execute the union of its lanes'
// groups), the filter emits a flattened list of (point, group) pairs; one
// thread scans one group for one point; a per-point merge certifies the new
// label and rewrites the group bounds.
//
//   k_filter_yinyang  decay ub / every group bound, global gate, tighten,
//                     per-group gate, append worklist rows + (row, group) pairs
//   k_yy_pairs        fp32 difference-form distances to one group's members
//   k_yy_merge        certified label, new group bounds, old-group fix-up;
//                     ambiguous rows -> exact fp64 recheck, pair-capacity
//                     overflow -> full SIMT rescan
#include <math.h>

#include "lk_common.cuh"
#include "lk_internal.h"

namespace lk {
namespace yy {

constexpr int kThreads = 256;
constexpr int kYyG = 8;  // lanes per (row, group) scan

// Block-wide exclusive scan of cnt with one global atomic per block.
// Block-uniform call; scratch >= blockDim/32 + 1 entries.
__device__ __forceinline__ int64_t block_reserve(int cnt, unsigned long long* counter,
                                                 unsigned long long* scratch) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(LK_FULL_MASK, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) scratch[warp] = (unsigned long long)incl;
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
    int64_t off = (int64_t)(scratch[nw] + scratch[warp]) + (incl - cnt);
    __syncthreads();
    return off;
}

__device__ __forceinline__ float dist2_row(const DevState& S, const float* xp, int j) {
    const float* cp = S.C32 + (int64_t)j * S.ldc;
    float acc = 0.f;
    int z = 0;
    if ((S.ldx & 3) == 0) {
        for (; z + 4 <= S.d; z += 4) {
            float4 xv = *reinterpret_cast<const float4*>(xp + z);
            float4 cv = __ldg(reinterpret_cast<const float4*>(cp + z));
            float t0 = xv.x - cv.x, t1 = xv.y - cv.y, t2 = xv.z - cv.z, t3 = xv.w - cv.w;
            acc = fmaf(t0, t0, acc);
            acc = fmaf(t1, t1, acc);
            acc = fmaf(t2, t2, acc);
            acc = fmaf(t3, t3, acc);
        }
    }
    for (; z < S.d; z++) {
        float t = __ldg(xp + z) - __ldg(cp + z);
        acc = fmaf(t, t, acc);
    }
    return acc;
}

__device__ __forceinline__ float xnorm(const DevState& S, const float* xp) {
    float s = 0.f;
    for (int z = 0; z < S.d; z++) {
        float v = __ldg(xp + z);
        s = fmaf(v, v, s);
    }
    return sqrtf(s);
}

constexpr int kCh = 8;

__global__ void __launch_bounds__(kThreads, 4) k_filter_yinyang(DevState S, int64_t* stat,
                                                                int full_only) {
    if (*S.done) return;
    extern __shared__ float gd[];  // [t] group drifts
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    const int t = S.t_groups;
    for (int g = threadIdx.x; g < t; g += kThreads) gd[g] = S.gdrift[g];
    __syncthreads();
    const float rho = simt_rel_err(S.d);
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < S.n;
         base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < S.n;
        bool active = false, need = false;
        int cnt = 0;
        float acc_a = 0.f, u = 0.f, lun = INFINITY, xn = 0.f;
        int apos = 0;
        float* lbr = S.lb + i;  // group g at lbr[g * n]
        const int64_t ln = S.n;
        if (valid) {
            const int a = S.labels[i];
            u = __fadd_ru(S.ub[i], S.drift[a]);
            float gmin = INFINITY;
            // chunks of kCh groups: the chunk's loads are issued before its stores
            for (int g0 = 0; g0 < t; g0 += kCh) {
                float v[kCh];
#pragma unroll
                for (int q = 0; q < kCh; q++)
                    if (g0 + q < t) v[q] = __ldcs(lbr + (int64_t)(g0 + q) * ln);
#pragma unroll
                for (int q = 0; q < kCh; q++) {
                    if (g0 + q < t) {
                        v[q] = fmaxf(__fsub_rd(v[q], gd[g0 + q]), 0.f);
                        gmin = fminf(gmin, v[q]);
                        __stcs(lbr + (int64_t)(g0 + q) * ln, v[q]);
                    }
                }
            }
            // Hamerly's centroid-separation test holds for every bound family:
            // d(x, c_j) >= 2 s_a - ub >= ub for all j != a when s_a > ub.
            const float sa = S.s_half[a];
            gmin = fmaxf(gmin, sa);
            if (!(gmin > u) && full_only && S.d >= 32) {
                // long rows on the tensor cores: a tighten costs 2d loads per
                // row, the full rescan decides the row anyway
                active = true;
                need = true;
            } else if (!(gmin > u)) {
                active = true;
                const float* xp = S.X32 + i * S.ldx;
                acc_a = dist2_row(S, xp, a);
                xn = xnorm(S, xp);
                apos = S.ginv[a];
                const float U = (sqrtf(acc_a) + kU32 * (xn + S.cnorm[a])) * (1.0f + rho);
                u = fminf(u, U);
                need = !(gmin > u);
            }
            S.ub[i] = u;
            if (need && !full_only) {
                for (int g0 = 0; g0 < t; g0 += kCh) {
                    float v[kCh];
#pragma unroll
                    for (int q = 0; q < kCh; q++)
                        if (g0 + q < t) v[q] = lbr[(int64_t)(g0 + q) * ln];
#pragma unroll
                    for (int q = 0; q < kCh; q++) {
                        if (g0 + q < t) {
                            if (v[q] > u) lun = fminf(lun, v[q]);  // group stays unscanned
                            else cnt++;
                        }
                    }
                }
            }
        }
        block_count(active, stat + LK_STAT_ACTIVE, scr);
        if (full_only) {
            // high-d tensor-core runs: failing rows are rescanned in full
            const int64_t fpos = block_append(need, (unsigned long long*)(stat + LK_STAT_WORK), scr);
            if (need) S.work[fpos] = (int)i;
            continue;
        }
        const int64_t wpos = block_append(need, (unsigned long long*)(stat + LK_STAT_YWL), scr);
        const int64_t poff = block_reserve(need ? cnt : 0, (unsigned long long*)(stat + LK_STAT_PAIRS), scr);
        if (need) {
            S.ylun[wpos] = make_float2(lun, xn);
            if (poff + cnt <= S.pair_cap) {
                S.ywl[wpos] = make_int4((int)i, (int)poff, cnt, __float_as_int(acc_a));
                int p = 0;
                for (int g = 0; g < t; g++)
                    if (!(lbr[g * ln] > u)) S.ypairs[poff + p++] = make_int2((int)i, g | (apos << 16));
            } else {
                // over capacity: full rescan instead; neutralise any reserved slots
                S.ywl[wpos] = make_int4((int)i, -1, 0, __float_as_int(acc_a));
                for (int64_t q = poff; q < S.pair_cap && q < poff + cnt; q++)
                    S.ypairs[q] = make_int2((int)i, -1);
            }
        }
    }
}

template <int DP>
__device__ __forceinline__ float dist2_dp(const float (&xr)[DP], const float* cp, int d) {
    float acc = 0.f;
#pragma unroll
    for (int z = 0; z < DP; z++) {
        // rows of Cg are zero-padded to ldc >= DP for DP <= 8
        if (DP <= 8 || z < d) {
            const float t = xr[z] - cp[z];
            acc = fmaf(t, t, acc);
        }
    }
    return acc;
}

// Iteration 1 of the group strategies (SequentialStrategy.seed +
// Yinyang._seed_state, pruners.py:83-87 / :398-416): a full scan in group
// order that also leaves the exact per-group minima (excluding the winner) as
// the group bounds, so iteration 2 starts from tight bounds.
template <int DP, bool STAGED>
__global__ void __launch_bounds__(kThreads) k_seed_yinyang(DevState S, int64_t* stat) {
    if (*S.done) return;
    extern __shared__ __align__(16) float csm[];
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    if (STAGED) {
        const int tot = S.k * S.ldc;
        for (int e = threadIdx.x; e < tot; e += kThreads) csm[e] = S.Cg[e];
        __syncthreads();
    }
    const float* __restrict__ cg = STAGED ? csm : S.Cg;
    const int ldc = S.ldc, T = S.t_groups;
    const float rho = simt_rel_err(S.d);
    const int64_t ln = S.n;
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < S.n;
         base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < S.n;
        float xr[DP];
        const float* xp = S.X32 + i * S.ldx;
        float xn2 = 0.f;
#pragma unroll
        for (int z = 0; z < DP; z++) {
            xr[z] = (valid && z < S.d) ? __ldg(xp + z) : 0.f;
            xn2 = fmaf(xr[z], xr[z], xn2);
        }
        const float xn = sqrtf(xn2);
        const float cmax = S.scal[0];
        float bestD = INFINITY, secD = INFINITY, bestg2 = INFINITY;
        int bestP = 0, bestG = 0;
        for (int g = 0; g < T; g++) {
            const int j0 = S.goff[g], j9 = S.goff[g + 1];
            float b1 = INFINITY, b2 = INFINITY;
            int p1 = j0;
            for (int jj = j0; jj < j9; jj++) {
                const float acc = dist2_dp<DP>(xr, cg + jj * ldc, S.d);
                if (acc < b1) { b2 = b1; b1 = acc; p1 = jj; }
                else b2 = fminf(b2, acc);
            }
            if (valid && j9 > j0)
                S.lb[lb_index(S, i, g)] =
                    fmaxf((sqrtf(b1) - kU32 * (xn + cmax)) * (1.0f - rho), 0.f);
            else if (valid)
                S.lb[lb_index(S, i, g)] = INFINITY;
            if (b1 < bestD) {
                secD = fminf(secD, bestD);
                bestD = b1; bestP = p1; bestG = g; bestg2 = b2;
            } else {
                secD = fminf(secD, b1);
            }
            secD = fminf(secD, b2);
        }
        const int j1 = S.gperm[bestP];
        const float U1 = (sqrtf(bestD) + kU32 * (xn + S.cnorm[j1])) * (1.0f + rho);
        const float L2 = isinf(secD) ? INFINITY : (sqrtf(secD) - kU32 * (xn + cmax)) * (1.0f - rho);
        const bool certain = valid && L2 > U1;
        const bool flag = valid && !certain;
        bool moved = false;
        int old = 0;
        if (certain) {
            old = S.labels[i];
            moved = old != j1;
            S.labels[i] = j1;
            // iteration 1: the cumulative drifts of the lazy encoding are 0
            S.ub[i] = U1;
            S.lb[lb_index(S, i, bestG)] =
                isinf(bestg2) ? INFINITY
                              : fmaxf((sqrtf(bestg2) - kU32 * (xn + cmax)) * (1.0f - rho), 0.f);
            if (S.glb) S.glb[i] = fmaxf(L2, 0.f);  // bounds every non-winner: min of the groups
        }
        int64_t pos = block_append(moved, (unsigned long long*)(stat + LK_STAT_CHANGED), scr);
        if (moved) S.moved[pos] = make_int2((int)i, old);
        int64_t fpos = block_append(flag, (unsigned long long*)(stat + LK_STAT_FLAGGED), scr);
        if (flag) S.flagged[fpos] = (int)i;
    }
}

// d <= 2 seed (cfg2's first iteration, 1e9 pairs): centroids staged as
// negated pairs (-a0, -b0, -a1, -b1) so one LDS.128 feeds two distances in
// paired fp32 (FADD2 / FMUL2 / FFMA2: each lane rounded exactly as dist2_dp's
// fmaf chain), per-group minima by FMNMX3; the exact top-2 with its index runs
// only over the winning group.  Same values, bounds and labels as
// k_seed_yinyang<2>.
__device__ __forceinline__ unsigned long long f2pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2upk(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ float fmin3s(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__global__ void __launch_bounds__(kThreads) k_seed_yinyang_d2(DevState S, int64_t* stat) {
    if (*S.done) return;
    extern __shared__ __align__(16) float4 cpair[];  // [pairs]; then int pair offsets [T + 1]
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    const int T = S.t_groups, ldc = S.ldc;
    int* poff = reinterpret_cast<int*>(cpair + (S.k + T));
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int g = 0; g < T; g++) {
            poff[g] = acc;
            acc += (S.goff[g + 1] - S.goff[g] + 1) >> 1;
        }
        poff[T] = acc;
    }
    __syncthreads();
    for (int g = 0; g < T; g++) {
        const int j0 = S.goff[g], j9 = S.goff[g + 1];
        const int np = (j9 - j0 + 1) >> 1;
        for (int q = threadIdx.x; q < np; q += kThreads) {
            const int ja = j0 + 2 * q, jb = min(ja + 1, j9 - 1);  // odd group: the last member twice
            const float* ca = S.Cg + (int64_t)ja * ldc;
            const float* cb = S.Cg + (int64_t)jb * ldc;
            const float a1 = S.d > 1 ? ca[1] : 0.f, b1 = S.d > 1 ? cb[1] : 0.f;
            cpair[poff[g] + q] = make_float4(-ca[0], -cb[0], -a1, -b1);
        }
    }
    __syncthreads();
    const float rho = simt_rel_err(S.d);
    const float cmax = S.scal[0];
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < S.n; base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < S.n;
        float xr[2];
        const float* xp = S.X32 + i * S.ldx;
        float xn2 = 0.f;
#pragma unroll
        for (int z = 0; z < 2; z++) {
            xr[z] = (valid && z < S.d) ? __ldg(xp + z) : 0.f;
            xn2 = fmaf(xr[z], xr[z], xn2);
        }
        const float xn = sqrtf(xn2);
        const unsigned long long xx = f2pk(xr[0], xr[0]), xy = f2pk(xr[1], xr[1]);
        float bestD = INFINITY, secD = INFINITY;
        int bestG = 0;
        for (int g = 0; g < T; g++) {
            const int p0 = poff[g], p9 = poff[g + 1];
            auto pair_d = [&](const float4 c, float& d0, float& d1) {
                unsigned long long t, u, dd;
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(xx), "l"(f2pk(c.x, c.y)));
                asm("add.rn.f32x2 %0, %1, %2;" : "=l"(u) : "l"(xy), "l"(f2pk(c.z, c.w)));
                asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(dd) : "l"(t));
                asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(dd) : "l"(u), "l"(dd));
                f2upk(dd, d0, d1);
            };
            // two independent minimum chains (ILP), merged at the end
            float m = INFINITY, m2 = INFINITY;
            int q = p0;
            for (; q + 1 < p9; q += 2) {
                float d0, d1, d2, d3;
                pair_d(cpair[q], d0, d1);
                pair_d(cpair[q + 1], d2, d3);
                m = fmin3s(m, d0, d1);
                m2 = fmin3s(m2, d2, d3);
            }
            if (q < p9) {
                float d0, d1;
                pair_d(cpair[q], d0, d1);
                m = fmin3s(m, d0, d1);
            }
            m = fminf(m, m2);
            if (valid)
                S.lb[lb_index(S, i, g)] = p9 > p0 ? fmaxf((sqrtf(m) - kU32 * (xn + cmax)) * (1.0f - rho), 0.f)
                                                  : INFINITY;
            if (m < bestD) {
                secD = fminf(secD, bestD);
                bestD = m;
                bestG = g;
            } else {
                secD = fminf(secD, m);
            }
        }
        // the winning group exactly (first minimum in group order, second best),
        // from the staged pairs: x + (-c) is x - c, the same fmaf chain as dist2_dp
        float b1 = INFINITY, b2 = INFINITY;
        const int g0 = S.goff[bestG], g9 = S.goff[bestG + 1];
        int bestP = g0;
        for (int jj = g0; jj < g9; jj++) {
            const float4 c = cpair[poff[bestG] + ((jj - g0) >> 1)];
            const bool hi = (jj - g0) & 1;
            const float t0 = xr[0] + (hi ? c.y : c.x);
            const float t1 = xr[1] + (hi ? c.w : c.z);
            float acc = fmaf(t0, t0, 0.f);
            if (S.d > 1) acc = fmaf(t1, t1, acc);
            if (acc < b1) { b2 = b1; b1 = acc; bestP = jj; }
            else b2 = fminf(b2, acc);
        }
        secD = fminf(secD, b2);
        const int j1 = S.gperm[bestP];
        const float U1 = (sqrtf(bestD) + kU32 * (xn + S.cnorm[j1])) * (1.0f + rho);
        const float L2 = isinf(secD) ? INFINITY : (sqrtf(secD) - kU32 * (xn + cmax)) * (1.0f - rho);
        const bool certain = valid && L2 > U1;
        const bool flag = valid && !certain;
        bool moved = false;
        int old = 0;
        if (certain) {
            old = S.labels[i];
            moved = old != j1;
            S.labels[i] = j1;
            S.ub[i] = U1;  // iteration 1: the cumulative drifts of the lazy encoding are 0
            S.lb[lb_index(S, i, bestG)] =
                isinf(b2) ? INFINITY : fmaxf((sqrtf(b2) - kU32 * (xn + cmax)) * (1.0f - rho), 0.f);
            if (S.glb) S.glb[i] = fmaxf(L2, 0.f);
        }
        int64_t pos = block_append(moved, (unsigned long long*)(stat + LK_STAT_CHANGED), scr);
        if (moved) S.moved[pos] = make_int2((int)i, old);
        int64_t fpos = block_append(flag, (unsigned long long*)(stat + LK_STAT_FLAGGED), scr);
        if (flag) S.flagged[fpos] = (int)i;
    }
}

__device__ __forceinline__ float dist2_ptr(const float* xp, const float* cp, int d, bool vec4) {
    float acc = 0.f;
    int z = 0;
    if (vec4) {
        for (; z + 4 <= d; z += 4) {
            float4 xv = *reinterpret_cast<const float4*>(xp + z);
            float4 cv = *reinterpret_cast<const float4*>(cp + z);
            float t0 = xv.x - cv.x, t1 = xv.y - cv.y, t2 = xv.z - cv.z, t3 = xv.w - cv.w;
            acc = fmaf(t0, t0, acc);
            acc = fmaf(t1, t1, acc);
            acc = fmaf(t2, t2, acc);
            acc = fmaf(t3, t3, acc);
        }
    }
    for (; z < d; z++) {
        float t = xp[z] - cp[z];
        acc = fmaf(t, t, acc);
    }
    return acc;
}

// G lanes per (row, group) pair: the group's members are contiguous in Cg
// (staged in shared memory when all centroids fit) and strided over the G
// lanes; a G-lane shuffle merges the partial top-2.  Positions ascend with
// centroid id inside a group, so (value, position) order is (value, id) order.
template <int G>
__global__ void __launch_bounds__(kThreads) k_yy_pairs(DevState S, int64_t* stat, int staged) {
    if (*S.done) return;
    extern __shared__ __align__(16) float csm[];
    const int64_t np_ = min((int64_t)stat[LK_STAT_PAIRS], S.pair_cap);
    constexpr int kPPW = 32 / G;  // pairs per warp
    constexpr int kWarps = kThreads / 32;
    if ((int64_t)blockIdx.x * kWarps * kPPW >= np_) return;
    const float* cbase = S.Cg;
    if (staged) {
        const int tot = S.k * S.ldc;
        for (int e = threadIdx.x; e < tot; e += kThreads) csm[e] = S.Cg[e];
        __syncthreads();
        cbase = csm;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane % G, slot = lane / G;
    const bool vec4 = (S.ldc & 3) == 0 && (S.ldx & 3) == 0;
    int64_t ndist = 0;
    for (int64_t pb = ((int64_t)blockIdx.x * kWarps + warp) * kPPW; pb < np_;
         pb += (int64_t)gridDim.x * kWarps * kPPW) {
        const int64_t p = pb + slot;
        int2 pr = make_int2(0, -1);
        if (p < np_) pr = S.ypairs[p];
        const bool valid = pr.y >= 0;
        const int64_t row = pr.x;
        const int g = valid ? (pr.y & 0xFFFF) : 0, apos = pr.y >> 16;
        const int j0 = valid ? S.goff[g] : 0, j9 = valid ? S.goff[g + 1] : 0;
        const float* xp = S.X32 + row * S.ldx;
        float b1 = INFINITY, b2 = INFINITY;
        int p1 = 0x7fffffff;
        if (S.d <= 4) {
            float xr[4];
#pragma unroll
            for (int z = 0; z < 4; z++) xr[z] = (valid && z < S.d) ? __ldg(xp + z) : 0.f;
            for (int jj = j0 + sub; jj < j9; jj += G) {
                if (jj == apos) continue;  // the label competes via the tightened bound
                const float* cp = cbase + (int64_t)jj * S.ldc;
                float acc = 0.f;
#pragma unroll
                for (int z = 0; z < 4; z++) {
                    if (z < S.d) {
                        float t = xr[z] - cp[z];
                        acc = fmaf(t, t, acc);
                    }
                }
                if (acc < b1) { b2 = b1; b1 = acc; p1 = jj; }
                else b2 = fminf(b2, acc);
            }
        } else {
            for (int jj = j0 + sub; jj < j9; jj += G) {
                if (jj == apos) continue;
                const float acc = dist2_ptr(xp, cbase + (int64_t)jj * S.ldc, S.d, vec4);
                if (acc < b1) { b2 = b1; b1 = acc; p1 = jj; }
                else b2 = fminf(b2, acc);
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            const float ob1 = __shfl_xor_sync(LK_FULL_MASK, b1, o, G);
            const float ob2 = __shfl_xor_sync(LK_FULL_MASK, b2, o, G);
            const int op1 = __shfl_xor_sync(LK_FULL_MASK, p1, o, G);
            if (ob1 < b1 || (ob1 == b1 && op1 < p1)) {
                b2 = fminf(b1, ob2);
                b1 = ob1;
                p1 = op1;
            } else {
                b2 = fminf(b2, ob1);
            }
        }
        if (valid && sub == 0) {
            ndist += (j9 - j0) - (apos >= j0 && apos < j9 ? 1 : 0);
            S.yres[p] = make_float4(__int_as_float(p1 < 0x7fffffff ? S.gperm[p1] : -1), b1, b2, 0.f);
        }
    }
    warp_add(ndist, stat + LK_STAT_DIST);
}

__global__ void __launch_bounds__(kThreads) k_yy_merge(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    const int64_t m = stat[LK_STAT_YWL];
    const int t = S.t_groups;
    const float rho = simt_rel_err(S.d);
    const float cmax = S.scal[0];
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < m;
         base += (int64_t)gridDim.x * kThreads) {
        const int64_t e = base + threadIdx.x;
        bool mv = false, flag = false, full = false;
        int64_t row = 0;
        int old = 0;
        if (e < m) {
            const int4 w = S.ywl[e];
            row = w.x;
            old = S.labels[row];
            if (w.y < 0) {
                full = true;
            } else {
                const float2 lx = S.ylun[e];
                const float lun = lx.x;  // min bound over the unscanned groups
                const float xn = lx.y;
                const float acc_a = __int_as_float(w.w);
                float bestD = acc_a, secD = INFINITY;
                int bestJ = old;
                for (int p = w.y; p < w.y + w.z; p++) {
                    const float4 r = S.yres[p];
                    const int pj = __float_as_int(r.x);
                    if (pj < 0) continue;  // group had no member other than the label
                    if (r.y < bestD || (r.y == bestD && pj < bestJ)) {
                        secD = fminf(secD, bestD);
                        bestD = r.y;
                        bestJ = pj;
                    } else {
                        secD = fminf(secD, r.y);
                    }
                    secD = fminf(secD, r.z);
                }
                float* lbr = S.lb + row;  // group g at lbr[g * n]
                const int64_t ln = S.n;
                const float U1 = (sqrtf(bestD) + kU32 * (xn + S.cnorm[bestJ])) * (1.0f + rho);
                const float Ls = isinf(secD) ? INFINITY
                                             : (sqrtf(secD) - kU32 * (xn + cmax)) * (1.0f - rho);
                const float L2 = fminf(Ls, lun);
                if (L2 > U1) {
                    mv = bestJ != old;
                    S.labels[row] = bestJ;
                    S.ub[row] = U1;
                    // scanned groups: certified min over members other than the new label
                    for (int q = w.y; q < w.y + w.z; q++) {
                        const float4 r = S.yres[q];
                        const int pj = __float_as_int(r.x);
                        const float gm = (pj == bestJ) ? r.z : r.y;
                        lbr[(int64_t)(S.ypairs[q].y & 0xFFFF) * ln] =
                            isinf(gm) ? INFINITY
                                      : fmaxf((sqrtf(gm) - kU32 * (xn + cmax)) * (1.0f - rho), 0.f);
                    }
                    if (mv) {
                        // the old label becomes an "other" member of its group
                        const int go = S.group_of[old];
                        const float la = fmaxf((sqrtf(acc_a) - kU32 * (xn + S.cnorm[old])) * (1.0f - rho), 0.f);
                        lbr[go * ln] = fminf(lbr[go * ln], la);
                    }
                } else {
                    flag = true;
                }
            }
        }
        int64_t pos = block_append(mv, (unsigned long long*)(stat + LK_STAT_CHANGED), scr);
        if (mv) S.moved[pos] = make_int2((int)row, old);
        int64_t fpos = block_append(flag, (unsigned long long*)(stat + LK_STAT_FLAGGED), scr);
        if (flag) S.flagged[fpos] = (int)row;
        int64_t wpos = block_append(full, (unsigned long long*)(stat + LK_STAT_WORK), scr);
        if (full) S.work[wpos] = (int)row;
    }
}

}  // namespace yy
}  // namespace lk

namespace lkh {

using namespace lk::yy;

static int grid_for_rows(int64_t rows, int sms, int per_sm) {
    int64_t b = (rows + kThreads - 1) / kThreads;
    if (b < 1) b = 1;
    if (b > (int64_t)sms * per_sm) b = sms * per_sm;
    return (int)b;
}

lk_status init_yy_attributes() {
#define LK_SMEM96(kern) \
    LK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024))
    LK_SMEM96((k_seed_yinyang<2, true>));
    LK_SMEM96((k_seed_yinyang<4, true>));
    LK_SMEM96((k_seed_yinyang<8, true>));
    LK_SMEM96((k_seed_yinyang<16, true>));
    LK_SMEM96((k_seed_yinyang<32, true>));
#undef LK_SMEM96
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_yy_pairs<kYyG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       96 * 1024));
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_filter_yinyang, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       64 * 1024));
    return LK_OK;
}

bool yy_masked(const lk::DevState& S) { return S.t_groups <= 32 && S.d <= 32; }

template <int DP>
static void launch_seed(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st) {
    const size_t csm = (size_t)S.k * S.ldc * sizeof(float);
    const int grid = grid_for_rows(S.n, sms, 6);
    if (csm <= 96 * 1024)
        k_seed_yinyang<DP, true><<<grid, kThreads, csm, st>>>(S, stat);
    else
        k_seed_yinyang<DP, false><<<grid, kThreads, 0, st>>>(S, stat);
}

lk_status launch_yy_seed(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st) {
    const int d = S.d;
    // (pairs <= (k + t) / 1 float4 + t + 1 offsets)
    const size_t d2smem = (size_t)(S.k + S.t_groups) * 16 + (size_t)(S.t_groups + 1) * 4;
    if (d <= 2 && d2smem <= 48 * 1024) {
        k_seed_yinyang_d2<<<grid_for_rows(S.n, sms, 6), kThreads, d2smem, st>>>(S, stat);
        LK_LAUNCH_CHECK();
        return LK_OK;
    }
    if (d <= 2) launch_seed<2>(S, stat, sms, st);
    else if (d <= 4) launch_seed<4>(S, stat, sms, st);
    else if (d <= 8) launch_seed<8>(S, stat, sms, st);
    else if (d <= 16) launch_seed<16>(S, stat, sms, st);
    else launch_seed<32>(S, stat, sms, st);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_yy_filter(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st,
                           bool full_only) {
    const size_t smem = (size_t)S.t_groups * sizeof(float);  // <= 64 KB (k <= 16384)
    k_filter_yinyang<<<grid_for_rows(S.n, sms, 8), kThreads, smem, st>>>(S, stat, full_only ? 1 : 0);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_yy_pairs(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st,
                          bool full_only) {
    if (full_only) return LK_OK;
    const size_t csm = (size_t)S.k * S.ldc * sizeof(float);
    const int staged = csm <= 96 * 1024;
    k_yy_pairs<kYyG><<<sms * (staged ? 4 : 8), kThreads, staged ? csm : 0, st>>>(S, stat, staged);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

lk_status launch_yy_merge(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st,
                          bool full_only) {
    if (full_only) return LK_OK;
    k_yy_merge<<<grid_for_rows(S.n, sms, 4), kThreads, 0, st>>>(S, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

}  // namespace lkh
