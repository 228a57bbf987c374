// lk_exact.cuh -- the oracle's own arithmetic on the device, shared by the
// kernels that re-decide ambiguous rows (fp64, numpy's pairwise association
// order: core.py:98-108) and by the kernels that refine centroids from moved
// rows (fixed-point member sums: lloyd.py:78-97).
#pragma once

#include "lk_common.cuh"

namespace lk {

// Sum of (x_z - c_z)^2 over [start, start+len) exactly as numpy's pairwise_sum
// leaf does it: sequential from 0 below 8 terms, else 8 strided accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail in order.
template <typename TX>
__device__ __forceinline__ double pw_leaf(const TX* x, const double* c, int start, int len) {
    if (len < 8) {
        double res = 0.0;
        for (int z = start; z < start + len; z++) {
            double t = __dsub_rn((double)x[z], c[z]);
            res = __dadd_rn(res, __dmul_rn(t, t));
        }
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
        double t = __dsub_rn((double)x[start + j], c[start + j]);
        r[j] = __dmul_rn(t, t);
    }
    int i = 8;
    const int main_end = len - (len % 8);
    for (; i < main_end; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            double t = __dsub_rn((double)x[start + i + j], c[start + i + j]);
            r[j] = __dadd_rn(r[j], __dmul_rn(t, t));
        }
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < len; i++) {
        double t = __dsub_rn((double)x[start + i], c[start + i]);
        res = __dadd_rn(res, __dmul_rn(t, t));
    }
    return res;
}

template <typename TX>
__device__ double pw_dist2(const TX* x, const double* c, const int32_t* prog, int plen) {
    if (plen == 3) return pw_leaf(x, c, __ldg(prog + 1), __ldg(prog + 2));
    double st[24];
    int sp = 0;
    for (int p = 0; p < plen; p += 3) {
        int op = __ldg(prog + p);
        if (op == 0) {
            st[sp++] = pw_leaf(x, c, __ldg(prog + p + 1), __ldg(prog + p + 2));
        } else {
            double b = st[--sp];
            double a = st[--sp];
            st[sp++] = __dadd_rn(a, b);
        }
    }
    return st[0];
}

__device__ __forceinline__ void merge_top2(double& b1, int& j1, double& b2, double ob1, int oj1,
                                           double ob2) {
    const bool mine = (b1 < ob1) || (b1 == ob1 && j1 < oj1);
    if (mine) {
        b2 = fmin(b2, ob1);
    } else {
        b2 = fmin(ob2, b1);
        b1 = ob1;
        j1 = oj1;
    }
}


__device__ __forceinline__ double load_x(const DevState& S, int64_t row, int z) {
    return S.X64 ? S.X64[row * S.d + z] : (double)__ldg(S.X32 + row * S.ldx + z);
}

// x_z - m_z: what the fixed-point member sums accumulate (the shift m is the
// middle of the data's range, so the sums and the SSE do not cancel for data
// far from the origin)
__device__ __forceinline__ double load_xs(const DevState& S, int64_t row, int z) {
    return load_x(S, row, z) - __ldg(S.xshift + z);
}

// Lanes per moved row in k_refine_moved (power of two >= min(d, 32)).
__host__ __device__ __forceinline__ int refine_lanes(int d) {
    return d <= 1 ? 1 : d <= 2 ? 2 : d <= 4 ? 4 : d <= 8 ? 8 : d <= 16 ? 16 : 32;
}

// ||x||^2 of a row in fp64 exactly as k_refine_moved's G-lane reduction
// computes it (lane s sums dimensions s, s+G, ...; then a xor butterfly), so
// a row's fixed-point ||x||^2 is the same integer whichever kernel moves it.
__device__ __forceinline__ double row_norm2_refine(const DevState& S, int64_t row) {
    const int G = refine_lanes(S.d);
    double p[32];
    for (int s = 0; s < G; s++) {
        double a = 0.0;
        for (int z = s; z < S.d; z += G) {
            const double v = load_xs(S, row, z);
            a = fma(v, v, a);
        }
        p[s] = a;
    }
    for (int o = G >> 1; o > 0; o >>= 1)
        for (int s = 0; s < o; s++) p[s] = p[s] + p[s + o];
    return p[0];
}

// The same value for d <= DP (DP a power of two <= 32) with every index a
// compile-time constant, so the partial sums stay in registers.
template <int DP>
__device__ __forceinline__ double row_norm2_refine_r(const DevState& S, int64_t row) {
    const int G = refine_lanes(S.d);
    double p[DP];
#pragma unroll
    for (int s = 0; s < DP; s++) {
        double a = 0.0;
#pragma unroll
        for (int z = s; z < DP; z += 1) {
            // dimension z belongs to lane z % G
            if (z < S.d && (z & (G - 1)) == s) {
                const double v = load_xs(S, row, z);
                a = fma(v, v, a);
            }
        }
        p[s] = a;
    }
#pragma unroll
    for (int o = DP >> 1; o > 0; o >>= 1) {
        if (o < G) {
#pragma unroll
            for (int s = 0; s < o; s++) p[s] = p[s] + p[s + o];
        }
    }
    return p[0];
}

// Fixed-point refinement deltas of one moved row (old = -1: first assignment),
// identical to one row of k_refine_moved.  DP = 0: any d (runtime loops).
template <int DP = 0>
__device__ __forceinline__ void refine_move(const DevState& S, const double* qscale, int64_t row,
                                            int old, int nw) {
    int64_t* dS = S.delta;
    int64_t* dN = S.delta + (int64_t)S.k * S.d;
    int64_t* dQ = dN + S.k;
    if (DP > 0) {
        // short rows: all loads first (independent), then the atomics
        constexpr int P = DP > 0 ? DP : 1;
        double v[P], sc[P];
#pragma unroll
        for (int z = 0; z < P; z++) {
            v[z] = z < S.d ? load_xs(S, row, z) : 0.0;
            sc[z] = z < S.d ? __ldg(qscale + z) : 0.0;
        }
#pragma unroll
        for (int z = 0; z < P; z++) {
            const long long q = z < S.d ? __double2ll_rn(v[z] * sc[z]) : 0;
            if (q) {
                atomicAdd((unsigned long long*)(dS + (int64_t)nw * S.d + z), (unsigned long long)q);
                if (old >= 0)
                    atomicAdd((unsigned long long*)(dS + (int64_t)old * S.d + z),
                              (unsigned long long)(-q));
            }
        }
    } else {
        for (int z = 0; z < S.d; z++) {
            const double v = load_xs(S, row, z);
            const long long q = __double2ll_rn(v * qscale[z]);
            if (q) {
                atomicAdd((unsigned long long*)(dS + (int64_t)nw * S.d + z), (unsigned long long)q);
                if (old >= 0)
                    atomicAdd((unsigned long long*)(dS + (int64_t)old * S.d + z), (unsigned long long)(-q));
            }
        }
    }
    const double x2 = DP > 0 ? row_norm2_refine_r<(DP > 0 ? DP : 1)>(S, row) : row_norm2_refine(S, row);
    const long long qq = __double2ll_rn(x2 * qscale[S.d]);
    atomicAdd((unsigned long long*)(dN + nw), 1ull);
    atomicAdd((unsigned long long*)(dQ + nw), (unsigned long long)qq);
    if (old >= 0) {
        atomicAdd((unsigned long long*)(dN + old), (unsigned long long)(-1ll));
        atomicAdd((unsigned long long*)(dQ + old), (unsigned long long)(-qq));
    }
}

// One flagged row, the whole block: x staged in shared memory (xr: >= d
// doubles), every thread takes k/256 centroids, lexicographic top-2 merge.
// Block-uniform call.
template <int NT>
__device__ __forceinline__ void recheck_row_block(const DevState& S, int64_t* stat,
                                                  const double* qscale_inline, int64_t row,
                                                  double* xr) {
    __shared__ double rb1[NT / 32], rb2[NT / 32];
    __shared__ int rj1[NT / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    for (int z = threadIdx.x; z < S.d; z += NT)
        xr[z] = S.X64 ? S.X64[row * S.d + z] : (double)S.X32[row * S.ldx + z];
    __syncthreads();
    double b1 = INFINITY, b2 = INFINITY;
    int j1 = 0x7fffffff;
    for (int j = threadIdx.x; j < S.k; j += NT) {
        double dd = __dsqrt_rn(pw_dist2(xr, S.C64 + (int64_t)j * S.d, S.pw_prog, S.pw_len));
        if (dd < b1) { b2 = b1; b1 = dd; j1 = j; }
        else b2 = fmin(b2, dd);
    }
    // lexicographic (value, index) top-2 merge: warp, then block
    for (int o = 16; o > 0; o >>= 1)
        merge_top2(b1, j1, b2, __shfl_xor_sync(LK_FULL_MASK, b1, o),
                   __shfl_xor_sync(LK_FULL_MASK, j1, o), __shfl_xor_sync(LK_FULL_MASK, b2, o));
    if (lane == 0) { rb1[warp] = b1; rj1[warp] = j1; rb2[warp] = b2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NT / 32; w++) merge_top2(b1, j1, b2, rb1[w], rj1[w], rb2[w]);
        const int old = S.labels[row];
        S.labels[row] = j1;
        if (S.strategy != LK_STRAT_LLOYD) {
            S.ub[row] = store_ub(S, __double2float_ru(b1 * (1.0 + 1e-12)), j1);
            write_lb_all(S, row, isinf(b2) ? INFINITY : __double2float_rd(b2 * (1.0 - 1e-12)));
        }
        if (old != j1) {
            unsigned long long p = atomicAdd((unsigned long long*)(stat + LK_STAT_CHANGED), 1ull);
            S.moved[p] = make_int2((int)row, old);
            if (qscale_inline) {
                refine_move(S, qscale_inline, row, old, j1);
                atomicAdd((unsigned long long*)(S.delta + (int64_t)S.k * S.d + 2 * S.k), 1ull);
                if (S.hlog_inline) {  // (the fused path logs its own moves)
                    const int t = *S.iter;
                    const int64_t hb = (t >= 1 && t <= S.t_max) ? S.hlog_off[t - 1] : -1;
                    if (hb >= 0 && hb + (int64_t)p < S.hlog_cap) S.hlog[hb + p] = make_int2((int)row, j1);
                }
            }
        }
    }
}


}  // namespace lk
