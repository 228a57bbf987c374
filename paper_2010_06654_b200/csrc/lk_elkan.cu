// lk_elkan.cu -- Elkan's per-centroid bounds on the GPU (n * k <= 2^26).
//
// Reference: Elkan (pruners.py:117-177).  Per point an upper bound ub and one
// lower bound per centroid lb[i, j], decayed by that centroid's drift
// (update_bounds, :128-133); the assignment visits the centroids in index
// order and evaluates d(x, c_j) only when neither lb[i, j] nor half the
// distance between the current best centroid and c_j (the s-matrix filter,
// :156-172) already proves c_j farther than the best.
//
// GPU form (one thread per row, lb group-major [k, n] so a warp's loads of one
// centroid's bounds coalesce): every distance is an fp32 difference-form value
// with a certified interval [L, U]; the running best b carries
// its interval, a centroid replaces it only when strictly closer (U_j < L_b),
// and the row is decided only when the best's U is below the lower bound of
// every other centroid (computed, or pruned by a bound / the half distance,
// both strictly above the running U).  Rows left ambiguous go to the exact fp64
// recheck.  Iteration 1 (labels -1) runs the same loop from an empty best, so
// the per-centroid bounds are exact from the start.
#include <math.h>

#include "lk_common.cuh"
#include "lk_internal.h"

namespace lk {
namespace elk {

constexpr int kThreads = 256;

// cch[a][j] = certified lower bound of 1/2 ||c_a - c_j|| (fp32 difference form,
// the k_half_sep rounding), 0 on the diagonal.
__global__ void k_elkan_cc(DevState S) {
    if (*S.done) return;
    const float rho = simt_rel_err(S.d);
    const int64_t kk = (int64_t)S.k * S.k;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < kk;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / S.k), j = (int)(e % S.k);
        float v = 0.f;
        if (a != j) {
            const float* ca = S.C32 + (int64_t)a * S.ldc;
            const float* cj = S.C32 + (int64_t)j * S.ldc;
            float acc = 0.f;
            for (int z = 0; z < S.d; z++) {
                const float t = __ldg(ca + z) - __ldg(cj + z);
                acc = fmaf(t, t, acc);
            }
            const float lbd = (sqrtf(acc) - kU32 * (S.cnorm[a] + S.cnorm[j])) * (1.0f - rho);
            v = fmaxf(0.5f * lbd * (1.0f - 4.0f * kU32), 0.f);
        }
        S.cch[e] = v;
    }
}

template <int DP>
__device__ __forceinline__ float dist2_row(const DevState& S, const float (&xr)[DP == 0 ? 1 : DP],
                                           const float* xg, const float* cp) {
    float acc = 0.f;
    if (DP > 0) {
#pragma unroll
        for (int z = 0; z < (DP == 0 ? 1 : DP); z++) {
            if (z < S.d) {
                const float t = xr[z] - __ldg(cp + z);
                acc = fmaf(t, t, acc);
            }
        }
    } else {
        for (int z = 0; z < S.d; z++) {
            const float t = __ldg(xg + z) - __ldg(cp + z);
            acc = fmaf(t, t, acc);
        }
    }
    return acc;
}

template <int DP>
__global__ void __launch_bounds__(kThreads) k_elkan(DevState S, int64_t* stat) {
    if (*S.done) return;
    __shared__ unsigned long long scr[kThreads / 32 + 1];
    const float rho = simt_rel_err(S.d);
    const int k = S.k;
    const int64_t n = S.n;
    int64_t n_dist = 0, n_active = 0;
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < n; base += (int64_t)gridDim.x * kThreads) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < n;
        const int a = valid ? S.labels[i] : -1;
        float xr[DP == 0 ? 1 : DP];
        const float* xg = S.X32 + (valid ? i : 0) * S.ldx;
        float xn2 = 0.f;
        if (DP > 0) {
#pragma unroll
            for (int z = 0; z < (DP == 0 ? 1 : DP); z++) {
                xr[z] = (valid && z < S.d) ? __ldg(xg + z) : 0.f;
                xn2 = fmaf(xr[z], xr[z], xn2);
            }
        } else if (valid) {
            for (int z = 0; z < S.d; z++) xn2 = fmaf(__ldg(xg + z), __ldg(xg + z), xn2);
        }
        const float xn = sqrtf(xn2);
        // running best b with its certified interval; L2 = lower bound over
        // every other centroid evaluated so far
        int b = -1;
        float Ub = INFINITY, Lb = INFINITY, L2 = INFINITY;
        bool tight = a < 0;
        if (valid && a >= 0) {
            b = a;
            Ub = __fadd_ru(S.ub[i], S.drift[a]);
            Lb = 0.f;
        }
        bool act = false;
        for (int j = 0; j < k; j++) {
            float* lp = S.lb + (int64_t)j * n + i;
            float l = 0.f;
            if (valid) {
                l = *lp;
                if (a >= 0) l = fmaxf(__fsub_rd(l, __ldg(S.drift + j)), 0.f);  // update_bounds
            }
            bool eval = valid && j != b && !(l > Ub) && !(b >= 0 && __ldg(S.cch + (int64_t)b * k + j) > Ub);
            if (eval && !tight) {
                // the label's own distance first (Elkan's tighten of ub)
                const float* cp = S.C32 + (int64_t)a * S.ldc;
                const float D = dist2_row<DP>(S, xr, xg, cp);
                const float e = kU32 * (xn + __ldg(S.cnorm + a));
                Ub = (sqrtf(D) + e) * (1.0f + rho);
                Lb = fmaxf((sqrtf(D) - e) * (1.0f - rho), 0.f);
                tight = true;
                act = true;
                n_dist++;
                S.lb[(int64_t)a * n + i] = Lb;
                eval = j != b && !(l > Ub) && !(__ldg(S.cch + (int64_t)b * k + j) > Ub);
            }
            if (eval) {
                const float* cp = S.C32 + (int64_t)j * S.ldc;
                const float D = dist2_row<DP>(S, xr, xg, cp);
                const float e = kU32 * (xn + __ldg(S.cnorm + j));
                const float Uj = (sqrtf(D) + e) * (1.0f + rho);
                const float Lj = fmaxf((sqrtf(D) - e) * (1.0f - rho), 0.f);
                n_dist++;
                act = true;
                l = Lj;
                if (Uj < Lb) {
                    // strictly closer than the best: it becomes the best
                    L2 = fminf(L2, Lb);
                    b = j;
                    Ub = Uj;
                    Lb = Lj;
                } else {
                    L2 = fminf(L2, Lj);
                }
            }
            if (valid && (j != a || !tight)) *lp = l;
        }
        n_active += act;
        // decided iff the best's upper bound is below every other centroid's
        // lower bound (pruned ones are above the running Ub, which only falls)
        const bool certain = valid && b >= 0 && L2 > Ub;
        const bool flag = valid && !certain;
        bool moved = false;
        if (certain) {
            moved = b != a;
            if (moved) S.labels[i] = b;
            S.ub[i] = Ub;
        }
        int64_t pos = block_append(moved, (unsigned long long*)(stat + LK_STAT_CHANGED), scr);
        if (moved) S.moved[pos] = make_int2((int)i, a);
        int64_t fpos = block_append(flag, (unsigned long long*)(stat + LK_STAT_FLAGGED), scr);
        if (flag) S.flagged[fpos] = (int)i;
    }
    warp_add(n_dist, stat + LK_STAT_DIST);
    warp_add(n_active, stat + LK_STAT_ACTIVE);
}

}  // namespace elk
}  // namespace lk

namespace lkh {

lk_status launch_elkan(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st) {
    using namespace lk::elk;
    const int64_t kk = (int64_t)S.k * S.k;
    k_elkan_cc<<<(unsigned)((kk + 255) / 256 < 4096 ? (kk + 255) / 256 : 4096), 256, 0, st>>>(S);
    LK_LAUNCH_CHECK();
    int64_t blocks = (S.n + kThreads - 1) / kThreads;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    if (blocks < 1) blocks = 1;
    const dim3 g((unsigned)blocks);
    if (S.d <= 4) k_elkan<4><<<g, kThreads, 0, st>>>(S, stat);
    else if (S.d <= 8) k_elkan<8><<<g, kThreads, 0, st>>>(S, stat);
    else if (S.d <= 16) k_elkan<16><<<g, kThreads, 0, st>>>(S, stat);
    else if (S.d <= 32) k_elkan<32><<<g, kThreads, 0, st>>>(S, stat);
    else k_elkan<0><<<g, kThreads, 0, st>>>(S, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

}  // namespace lkh
