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

#include "lk_common.cuh"
#include "lk_internal.h"

namespace lk {
namespace tgy {

constexpr int kThreads = 256;

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
        if (i < S.n) {
            const int a = __ldcs(S.labels + i);
            const float ub_s = __ldcs(S.ub + i), glb_s = __ldcs(S.glb + i);
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
        }
        const int64_t pos = block_append(need, (unsigned long long*)(stat + LK_STAT_WORK), scr);
        if (need) {
            S.work[pos] = (int)i;
            S.ymask[pos] = mask;
            S.ylun[pos] = make_float2(lun, 0.f);
        }
    }
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
    if (S.d <= 8)
        lk::tgy::k_filter_tgy<8><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
    else if (S.d <= 16)
        lk::tgy::k_filter_tgy<16><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
    else
        lk::tgy::k_filter_tgy<32><<<(unsigned)blocks, lk::tgy::kThreads, 0, st>>>(S, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

}  // namespace lkh
