// lk_regroup.cu -- Regroup: the centroid-to-group map rebuilt after every
// centroid update, with the per-point group bounds remapped.
//
// Reference: Yinyang.update_bounds with regroup = True (pruners.py:429-436,
// Regroup :500-504), regroup_pass (bounds.py:199-212: one nearest-group-mean
// pass, empty groups excluded, ties to the lowest group) and
// remap_group_bounds (bounds.py:215-228: a new group's bound is the minimum of
// the old bounds of the old groups that contribute a member).
//
//   k_regroup       one block: group means (members in gperm order), every
//                   centroid's nearest mean, the changed flag, the source
//                   masks M[g'] = {old groups of g' members}; when the map
//                   changed, the group-ordered layout (goff, gperm, ginv,
//                   group_of, Cg) is rebuilt by a counting sort
//   k_regroup_remap per row: new bound of g' = min over M[g'] of the old
//                   (decayed) bounds; the lazy encoding is re-based on zero
//                   cumulative group drifts, the plain layout's pending group
//                   decay is applied (k_regroup_finish clears either)
// All of it is device-side and runs every iteration inside the captured graph
// (the remap is a no-op when the map did not change).  t <= 32 groups.
#include <math.h>

#include "lk_common.cuh"
#include "lk_internal.h"

namespace lk {
namespace rg {

// scratch: [0] changed flag, [1 .. 32] source masks, then new_of [k],
// then the means [t, d] (doubles, 8-aligned)
__global__ void __launch_bounds__(1024) k_regroup(DevState S, int32_t* scr, double* means) {
    if (*S.done) return;
    const int t = S.t_groups, k = S.k, d = S.d;
    int32_t* flag = scr;
    uint32_t* src = reinterpret_cast<uint32_t*>(scr + 1);
    int32_t* new_of = scr + 33;
    __shared__ int cnt[32];
    __shared__ int fill[33];
    if (threadIdx.x == 0) *flag = 0;
    if (threadIdx.x < 32) src[threadIdx.x] = 0;
    // group means over the current members (gperm order within a group)
    for (int e = threadIdx.x; e < t * d; e += blockDim.x) {
        const int g = e / d, z = e % d;
        double s = 0.0;
        const int p0 = S.goff[g], p1 = S.goff[g + 1];
        for (int p = p0; p < p1; p++) s += S.C64[(int64_t)S.gperm[p] * d + z];
        means[e] = p1 > p0 ? s / (double)(p1 - p0) : 0.0;
    }
    __syncthreads();
    // nearest non-empty group mean of every centroid
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        double best = INFINITY;
        int bg = 0;
        for (int g = 0; g < t; g++) {
            if (S.goff[g + 1] == S.goff[g]) continue;
            double acc = 0.0;
            for (int z = 0; z < d; z++) {
                const double v = S.C64[(int64_t)j * d + z] - means[g * d + z];
                acc = fma(v, v, acc);
            }
            if (acc < best) {
                best = acc;
                bg = g;
            }
        }
        new_of[j] = bg;
        const int og = S.group_of[j];
        atomicOr(src + bg, 1u << og);
        if (bg != og) atomicExch(flag, 1);
    }
    __syncthreads();
    if (!*flag) return;
    if (threadIdx.x == 0) S.cur[LK_STAT_REGROUPED] = 1;  // (counted in the next iteration's stats)
    // the group-ordered layout of the new map (counting sort; ascending j
    // inside a group, as lk_set_groups builds it)
    if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) atomicAdd(cnt + new_of[j], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int g = 0; g < t; g++) {
            fill[g] = run;
            S.goff[g] = run;
            run += cnt[g];
        }
        S.goff[t] = run;
        // (ascending j within a group: one thread walks the centroids in order)
        for (int j = 0; j < k; j++) {
            const int g = new_of[j];
            const int pos = fill[g]++;
            S.gperm[pos] = j;
            S.ginv[j] = pos;
            S.group_of[j] = g;
        }
    }
    __syncthreads();
    if (S.Cg)
        for (int e = threadIdx.x; e < k * S.ldc; e += blockDim.x) {
            const int j = e / S.ldc, z = e % S.ldc;
            S.Cg[(int64_t)S.ginv[j] * S.ldc + z] = S.C32[(int64_t)j * S.ldc + z];
        }
}

__global__ void k_regroup_remap(DevState S, const int32_t* scr) {
    if (*S.done || !scr[0]) return;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(scr + 1);
    const int t = S.t_groups;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float old[32], nw[32];
#pragma unroll
        for (int g = 0; g < 32; g++) {
            old[g] = INFINITY;
            if (g < t) {
                // the decayed bound of old group g (plain layout: the decay the
                // next filter would apply, done here; k_regroup_finish zeroes it)
                old[g] = S.lazy ? __fsub_rd(S.lb[i * S.nlb + g], S.dgcum[g])
                                : fmaxf(__fsub_rd(S.lb[(int64_t)g * S.n + i], S.gdrift[g]), 0.f);
            }
        }
#pragma unroll
        for (int g = 0; g < 32; g++) {
            float v = INFINITY;
            const uint32_t m = g < t ? src[g] : 0u;
#pragma unroll
            for (int h = 0; h < 32; h++)
                if ((m >> h) & 1u) v = fminf(v, old[h]);
            nw[g] = v;
        }
#pragma unroll
        for (int g = 0; g < 32; g++) {
            if (g < t) {
                if (S.lazy) S.lb[i * S.nlb + g] = nw[g];  // re-based: cumulative group drifts restart at 0
                else S.lb[(int64_t)g * S.n + i] = nw[g];
            }
        }
    }
}

__global__ void k_regroup_finish(DevState S, const int32_t* scr) {
    if (*S.done || !scr[0]) return;
    if (threadIdx.x < S.t_groups) {
        if (S.lazy) S.dgcum[threadIdx.x] = 0.f;
        else S.gdrift[threadIdx.x] = 0.f;  // (the remap applied this iteration's decay)
    }
}

}  // namespace rg
}  // namespace lk

namespace lkh {

lk_status launch_regroup(const lk::DevState& S, int32_t* scr, double* means, int sms, cudaStream_t st) {
    if (S.t_groups > 32) {
        set_error("regroup: at most 32 groups (got %d)", S.t_groups);
        return LK_ERR_UNSUPPORTED;
    }
    lk::rg::k_regroup<<<1, 1024, 0, st>>>(S, scr, means);
    LK_LAUNCH_CHECK();
    lk::rg::k_regroup_remap<<<sms * 4, 256, 0, st>>>(S, scr);
    LK_LAUNCH_CHECK();
    lk::rg::k_regroup_finish<<<1, 32, 0, st>>>(S, scr);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

}  // namespace lkh
