// lk_validate.cu -- debug shadow check of the stored bounds (RunContext.
// debug_validate): every row's bounds against the exact fp64 distances.
//
// Reference: validate_bounds (bounds.py:280-328), called by run_pruner at
// "iter{t}:decayed" (after update_bounds) and "iter{t}:post" (after the
// assignment) when ctx.debug_validate is set (pruners.py:896-902).  The kinds
// and the tolerance (1e-8 + 1e-9 |ref|, bounds.py:272-278) are the
// reference's:
//   ub           d(x, c_label) <= ub + tol
//   lb_global    lb <= min_{j != label} d(x, c_j) + tol   (Hamerly lb, Yinyang
//                global bound)
//   lb_group[g]  lb_g <= min_{j in g, j != label} d(x, c_j) + tol
// Stored bounds are decoded exactly as the filters read them (lazy encoding:
// against the cumulative drifts; plain layouts at the "decayed" point: with
// the pending decay applied the way the next filter applies it).
//
// out[0] = worst ub overshoot, out[1] = worst lb_global overshoot, out[2 + g]
// = worst lb_group[g] overshoot (0: none); nonnegative doubles reduced with
// an integer atomicMax on their bit patterns.
#include <math.h>

#include "lk_common.cuh"
#include "lk_exact.cuh"
#include "lk_internal.h"

namespace lk {
namespace val {

__device__ __forceinline__ void omax(double* out, double v) {
    if (v > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ double vtol(double ref) { return 1e-8 + 1e-9 * fabs(ref); }

__device__ __forceinline__ double true_dist(const DevState& S, int64_t row, int j) {
    const double* cp = S.C64 + (int64_t)j * S.d;
    return __dsqrt_rn(S.X64 ? pw_dist2(S.X64 + row * S.d, cp, S.pw_prog, S.pw_len)
                            : pw_dist2(S.X32 + row * S.ldx, cp, S.pw_prog, S.pw_len));
}

__global__ void k_validate(DevState S, int decayed, double* out) {
    const float dmax1 = S.scal[1], dmax2 = S.scal[2];
    const int amax = __float_as_int(S.scal[3]);
    const bool groups = S.strategy != LK_STRAT_HAMERLY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int a = S.labels[i];
        if (a < 0) continue;
        const double da = true_dist(S, i, a);
        // ---- ub
        float ub = S.ub[i];
        if (S.lazy) ub = __fadd_ru(ub, S.dcum[a]);
        else if (decayed) ub = __fadd_ru(ub, S.drift[a]);
        omax(out + 0, da - (double)ub - vtol(da));
        // ---- the global lower bound and the group bounds
        double second = INFINITY;
        if (S.elkan) {
            // lb_center: every centroid's own bound (bounds.py:304-305)
            for (int j = 0; j < S.k; j++) {
                if (j == a) continue;
                const double dj = true_dist(S, i, j);
                float lj = S.lb[(int64_t)j * S.n + i];
                if (decayed) lj = fmaxf(__fsub_rd(lj, S.drift[j]), 0.f);
                omax(out + 1, (double)lj - dj - vtol(dj));
            }
            continue;
        }
        if (!groups) {
            for (int j = 0; j < S.k; j++)
                if (j != a) second = fmin(second, true_dist(S, i, j));
            float lb = S.lb[i];
            if (decayed) lb = fmaxf(__fsub_rd(lb, a == amax ? dmax2 : dmax1), 0.f);
            omax(out + 1, (double)lb - second - vtol(second));
            continue;
        }
        for (int g = 0; g < S.t_groups; g++) {
            double gm = INFINITY;
            if (S.colperm) {
                for (int c = 128 * g; c < 128 * g + 128 && c < S.kpad; c++) {
                    const int j = S.colperm[c];
                    if (j >= 0 && j != a) gm = fmin(gm, true_dist(S, i, j));
                }
            } else {
                for (int p = S.goff[g]; p < S.goff[g + 1]; p++) {
                    const int j = S.gperm[p];
                    if (j != a) gm = fmin(gm, true_dist(S, i, j));
                }
            }
            second = fmin(second, gm);
            float lg;
            if (S.lazy) {
                lg = __fsub_rd(S.lb[i * S.nlb + g], S.dgcum[g]);
            } else {
                lg = S.lb[(int64_t)g * S.n + i];
                if (decayed) lg = fmaxf(__fsub_rd(lg, S.gdrift[g]), 0.f);
            }
            if (!isinf(gm)) omax(out + 2 + g, (double)lg - gm - vtol(gm));
        }
        if (S.lazy) {
            const float glb = __fsub_rd(S.glb[i], S.scal[4]);
            if (!isinf(second)) omax(out + 1, (double)glb - second - vtol(second));
        }
    }
}

}  // namespace val
}  // namespace lk

namespace lkh {

lk_status launch_validate(const lk::DevState& S, int decayed, double* host_out, int nout,
                          double* dev_scratch, cudaStream_t st) {
    LK_CUDA_CHECK(cudaMemsetAsync(dev_scratch, 0, (size_t)nout * 8, st));
    if (S.n > 0 && S.strategy != LK_STRAT_LLOYD)
        lk::val::k_validate<<<(unsigned)((S.n + 127) / 128 < 4096 ? (S.n + 127) / 128 : 4096), 128, 0, st>>>(
            S, decayed, dev_scratch);
    LK_LAUNCH_CHECK();
    LK_CUDA_CHECK(cudaMemcpyAsync(host_out, dev_scratch, (size_t)nout * 8, cudaMemcpyDeviceToHost, st));
    LK_CUDA_CHECK(cudaStreamSynchronize(st));
    return LK_OK;
}

}  // namespace lkh
