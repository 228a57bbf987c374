// lk_yy_fused.cu -- the whole Yinyang assignment of one iteration in one
// kernel, for d <= 32 and t <= 32 groups.
//
// Reference: Yinyang.update_bounds (pruners.py:418-436), the global / group
// gates and the per-group scan of assign_pass (pruners.py:445-478), the
// group-bound rewrite and old-group fix-up (:480-494), and the refinement
// deltas of refine_full (lloyd.py:78-97) for the rows that moved.  Labels are
// certified exactly as in the multi-kernel paths.
//
//   filter   (one thread per row, software-pipelined loads) decay ub and the
//            t group bounds, global gate (with Hamerly's centroid-separation
//            test), tighten, group gate -> bitmask of groups to scan; failing
//            rows go to a block-local queue, their (row, group) pairs to a
//            shared-memory pair list counted per group
//   drain    (only when the queue is full, and at the end)
//     sort   pairs are bucketed by group, so one warp's lanes scan the same
//            group and the centroid loads are shared-memory broadcasts
//     scan   2^lg lanes per pair, fp32 difference-form top-2 over the group
//     merge  one thread per queued row: certified label, ub, rewritten group
//            bounds; a moved row adds its fixed-point refinement deltas
//            ambiguous rows are re-decided in place by the exact fp64
//            recheck (recheck_row_block, which refines the rows it moves)
//
// Only the labels, the bound table, the refinement deltas and the moved-row
// log touch HBM; the pair list and the scan results never leave the SM.
#include <math.h>
#include <stdlib.h>

#include "lk_common.cuh"
#include "lk_exact.cuh"
#include "lk_internal.h"

namespace lk {
namespace yyf {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxPairs = 512;   // pair slots of the block queue (swept: 512-1536, 512 best on cfg2)
constexpr int kQRows = 512;      // row slots of the block queue
// per-centroid filter info (cumulative drift, half-separation, norm, group
// position) is read through L1 rather than staged: k * 16 B stays L1-resident
constexpr bool kStageInfo = false;

template <int DP>
__device__ __forceinline__ float dist2(const float (&xr)[DP], const float* cp, int d) {
    float acc = 0.f;
#pragma unroll
    for (int z = 0; z < DP; z++) {
        // staged rows are zero-padded to >= DP for DP <= 8
        if (DP <= 8 || z < d) {
            const float t = xr[z] - cp[z];
            acc = fmaf(t, t, acc);
        }
    }
    return acc;
}

template <int DP>
struct Queue {
    int row[kQRows];
    int a[kQRows];
    float acc[kQRows];   // fp32 D~ to the (old) label
    float xn[kQRows];    // |x|
    float lun[kQRows];   // min decayed bound over the unscanned groups
    unsigned mask[kQRows];
    int poff[kQRows];
    int flag[kQRows];    // rows of this drain left ambiguous by the merge
    float x[DP <= 4 ? kQRows : 1][DP];
};

struct Shared {
    const float* dg;   // cumulative group drifts (lazy encoding offsets)
    float dm;          // cumulative max drift
    const int* goff;
    int* bcnt;
    int* boff;
    const uint32_t* ptmp;
    uint16_t* psort;
    int64_t hbase;     // this iteration's label-history log offset (-1: not logged)
    float* rb1;
    float* rb2;
    int* rp1;
    int* nflag;
};

// A moved row's fixed-point refinement deltas; out of line so the register
// pressure of the (rare) moved-row path does not weigh on the filter loop.
template <int DP>
__device__ __forceinline__ void move_deltas(const DevState* __restrict__ G, const double* qscale,
                                         int64_t row, int old, int nw) {
    refine_move<DP>(*G, qscale, row, old, nw);
}

// A row's new label and bounds are final: a moved row adds its refinement
// deltas and enters the moved-row log (label history).  Warp-uniform call.
template <int DP>
__device__ __forceinline__ void commit_move(const DevState& S, const double* qscale,
                                            int64_t* stat, bool mv, int64_t row, int old,
                                            int nw, int64_t hbase) {
    if (mv) move_deltas<DP>(S.self, qscale, row, old, nw);
    const int64_t pm = warp_append(mv, (unsigned long long*)(stat + LK_STAT_CHANGED));
    if (mv) S.moved[pm] = make_int2((int)row, old);
    // label history (lloyd.py:140) as the moved-row log, written here instead of
    // by k_log_history: slot base + position in the moved list
    if (mv && hbase >= 0 && hbase + pm < S.hlog_cap) S.hlog[hbase + pm] = make_int2((int)row, nw);
    // the changed count rides in the all-reduce payload
    warp_count(mv, S.delta + (int64_t)S.k * S.d + 2 * S.k);
}

template <int DP, int T>
__device__ __forceinline__ void drain(const DevState& S, int64_t* stat, const double* qscale,
                                   Queue<DP>& Q, int nrow, int npair, const Shared& sh,
                                   const float* cg, int cstride, int lg_parts, float rho,
                                   float cmax, int64_t& n_dist) {
    // ---- bucket offsets of the groups
    if (threadIdx.x < 32) {
        const int c = threadIdx.x < T ? sh.bcnt[threadIdx.x] : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u2 = __shfl_up_sync(LK_FULL_MASK, incl, o);
            if ((int)threadIdx.x >= o) incl += u2;
        }
        if (threadIdx.x < T) {
            sh.boff[threadIdx.x] = incl - c;
            sh.bcnt[threadIdx.x] = 0;
        }
        if (threadIdx.x == 0) *sh.nflag = 0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < npair; e += kThreads) {
        const uint32_t w = sh.ptmp[e];
        sh.psort[sh.boff[(w >> 10) & 0x3f] + (w >> 16)] = (uint16_t)e;
    }
    __syncthreads();

    // ---- scans: 2^lg_parts adjacent lanes per (row, group); part p takes
    // members p, p + nparts, ... (consecutive lanes read consecutive centroids,
    // lanes of other rows in the same group read the same ones: broadcasts);
    // the label's own centroid is scanned too (the merge recognises it)
    const int nparts = 1 << lg_parts;
    const int nsub = npair << lg_parts;
    for (int s0 = 0; s0 < nsub; s0 += kThreads) {
        const int sidx = s0 + threadIdx.x;
        const bool ok = sidx < nsub;
        const int part = sidx & (nparts - 1);
        float b1 = INFINITY, b2 = INFINITY;
        int p1 = -1, e = 0;
        if (ok) {
            e = sh.psort[sidx >> lg_parts];
            const uint32_t w = sh.ptmp[e];
            const int q = w & 0x3ff, g = (w >> 10) & 0x3f;
            float xq[DP];
            if (DP <= 4) {
#pragma unroll
                for (int z = 0; z < DP; z++) xq[z] = Q.x[DP <= 4 ? q : 0][z];
            } else {
                const float* xp = S.X32 + (int64_t)Q.row[q] * S.ldx;
#pragma unroll
                for (int z = 0; z < DP; z++) xq[z] = z < S.d ? __ldg(xp + z) : 0.f;
            }
            const int j0 = sh.goff[g] + part, j9 = sh.goff[g + 1];
            const float* cp = cg + j0 * cstride;
            const int step = nparts * cstride;
            int jj = j0;
            for (; jj + 3 * nparts < j9; jj += 4 * nparts) {
                float a4[4];
#pragma unroll
                for (int u = 0; u < 4; u++) a4[u] = dist2<DP>(xq, cp + u * step, S.d);
                cp += 4 * step;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    b2 = fminf(b2, fmaxf(a4[u], b1));
                    p1 = a4[u] < b1 ? jj + u * nparts : p1;
                    b1 = fminf(b1, a4[u]);
                }
            }
            for (; jj < j9; jj += nparts) {
                const float acc = dist2<DP>(xq, cp, S.d);
                cp += step;
                b2 = fminf(b2, fmaxf(acc, b1));
                p1 = acc < b1 ? jj : p1;
                b1 = fminf(b1, acc);
            }
            if (j9 > j0) n_dist += (j9 - j0 + nparts - 1) >> lg_parts;
        }
        for (int o = nparts >> 1; o > 0; o >>= 1) {
            const float ob1 = __shfl_xor_sync(LK_FULL_MASK, b1, o);
            const float ob2 = __shfl_xor_sync(LK_FULL_MASK, b2, o);
            const int op1 = __shfl_xor_sync(LK_FULL_MASK, p1, o);
            // (value, position) order; positions ascend with centroid id in a group
            const bool take = ob1 < b1 || (ob1 == b1 && op1 >= 0 && (p1 < 0 || op1 < p1));
            b2 = take ? fminf(b1, ob2) : fminf(b2, ob1);
            b1 = take ? ob1 : b1;
            p1 = take ? op1 : p1;
        }
        if (ok && part == 0) {
            sh.rb1[e] = b1;
            sh.rb2[e] = b2;
            sh.rp1[e] = (p1 >= 0 && !isinf(b1)) ? __ldg(S.gperm + p1) : -1;
        }
    }
    __syncthreads();

    // ---- certified merge, one thread per queued row
    for (int q0 = 0; q0 < nrow; q0 += kThreads) {
        const int q = q0 + threadIdx.x;
        bool mv = false;
        int64_t i = 0;
        int a = 0, bestJ = 0;
        if (q < nrow) {
            i = Q.row[q];
            a = Q.a[q];
            const float acc_a = Q.acc[q], xn = Q.xn[q];
            const unsigned mask = Q.mask[q];
            const int poff = Q.poff[q];
            // the label competes through its tightened distance; if its own
            // group was scanned, the scan met it too: that group's competitor
            // is then its second best
            float bestD = acc_a, secD = INFINITY;
            bestJ = a;
            int e = poff;
            for (unsigned mm = mask; mm; mm &= mm - 1, e++) {
                const int pj = sh.rp1[e];
                const float r1 = sh.rb1[e], r2 = sh.rb2[e];
                if (pj == a) {
                    secD = fminf(secD, r2);
                    continue;
                }
                if (pj >= 0) {
                    if (r1 < bestD || (r1 == bestD && pj < bestJ)) {
                        secD = fminf(secD, bestD);
                        bestD = r1;
                        bestJ = pj;
                    } else {
                        secD = fminf(secD, r1);
                    }
                }
                secD = fminf(secD, r2);
            }
            const float U1 = (sqrtf(bestD) + kU32 * (xn + S.cnorm[bestJ])) * (1.0f + rho);
            const float a2 = kU32 * (xn + cmax);
            const float Ls = isinf(secD) ? INFINITY : (sqrtf(secD) - a2) * (1.0f - rho);
            if (fminf(Ls, Q.lun[q]) > U1) {
                // stored in the lazy encoding: ub - Dc[label], lb + Dg[g], glb + Dm
                mv = bestJ != a;
                if (mv) S.labels[i] = bestJ;
                S.ub[i] = __fsub_ru(U1, S.dcum[bestJ]);
                float* lbr = S.lb + i * T;  // row-major group table (lazy encoding)
                float gnew = Q.lun[q];  // min over the unscanned groups
                e = poff;
                for (unsigned mm = mask; mm; mm &= mm - 1, e++) {
                    const int g = __ffs(mm) - 1;
                    // every member but the winner (the old label included)
                    const float gm = (sh.rp1[e] == bestJ) ? sh.rb2[e] : sh.rb1[e];
                    const float lg = isinf(gm) ? INFINITY : (sqrtf(gm) - a2) * (1.0f - rho);
                    gnew = fminf(gnew, lg);
                    lbr[g] = __fadd_rd(lg, sh.dg[g]);
                }
                if (mv) {
                    // the old label joins its group's competitors (needed when
                    // that group was not scanned; harmless otherwise)
                    const int go = S.group_of[a];
                    const float la = (sqrtf(acc_a) - kU32 * (xn + S.cnorm[a])) * (1.0f - rho);
                    gnew = fminf(gnew, la);
                    lbr[go] = fminf(lbr[go], __fadd_rd(la, sh.dg[go]));
                }
                S.glb[i] = __fadd_rd(gnew, sh.dm);
            } else {
                Q.flag[atomicAdd(sh.nflag, 1)] = q;
            }
        }
        commit_move<DP>(S, qscale, stat, mv, i, a, bestJ, sh.hbase);
    }
    __syncthreads();

    // ---- ambiguous rows (a few per iteration) are re-decided here by the exact
    // fp64 recheck (numpy order over all k, the whole block per row), which
    // also adds the refinement deltas of the rows it moves: no recheck launch
    const int nfl = *sh.nflag;
    if (nfl > 0) {
        __shared__ double xr[32];
        if (threadIdx.x == 0) atomicAdd((unsigned long long*)(stat + LK_STAT_FLAGGED), (unsigned long long)nfl);
        for (int f = 0; f < nfl; f++) recheck_row_block<kThreads>(S, stat, qscale, Q.row[Q.flag[f]], xr);
    }
}

template <int DP, int T, bool STAGED>
__global__ void __launch_bounds__(kThreads, (DP <= 4 ? 3 : 2)) k_yy_fused(DevState S, int64_t* stat,
                                                      const double* qscale, int pcap,
                                                      int lg_parts) {
    pdl_wait();
    pdl_trigger();  // the update may be scheduled while this kernel drains
    if (*S.done) return;
    // dynamic: staged centroids (group order) + per-centroid info | pair list
    // | sorted order | scan results
    extern __shared__ __align__(16) float dsm[];
    __shared__ float dg[T];
    __shared__ int goff[T + 1];
    __shared__ int bcnt[T];
    __shared__ int boff[T];
    __shared__ int wrows[kWarps], wpairs[kWarps];
    __shared__ int s_first;  // (chunk rank << 16 | chunk pair offset) of the first unqueued row
    __shared__ int s_nflag;
    __shared__ Queue<DP> Q;

    const int k = S.k, ldc = S.ldc;
    const int sd = DP <= 4 ? DP : ldc;  // stride of the staged centroid rows
    // staged (STAGED): centroids in group order, then per-centroid cumulative
    // drift, half-separation, norm bound and group position, so the filter's
    // label-dependent loads are shared-memory reads
    float* cgs = dsm;
    constexpr bool SI = STAGED && kStageInfo;
    float* s_drift = dsm + (STAGED ? k * sd : 0);
    float* s_shalf = s_drift + (SI ? k : 0);
    float* s_cnorm = s_shalf + (SI ? k : 0);
    int* s_ginv = reinterpret_cast<int*>(s_cnorm + (SI ? k : 0));
    uint32_t* ptmp = reinterpret_cast<uint32_t*>(s_ginv + (SI ? k : 0));
    uint16_t* psort = reinterpret_cast<uint16_t*>(ptmp + pcap);
    float* rb1 = reinterpret_cast<float*>(psort + ((pcap + 1) & ~1));
    float* rb2 = rb1 + pcap;
    int* rp1 = reinterpret_cast<int*>(rb2 + pcap);
    const float dm = S.scal[4];
    int64_t hbase = -1;
    if (S.hlog_inline) {
        const int t = *S.iter;
        if (t >= 1 && t <= S.t_max) hbase = S.hlog_off[t - 1];
    }
    const Shared sh{dg, dm, goff, bcnt, boff, ptmp, psort, hbase, rb1, rb2, rp1, &s_nflag};

    if (threadIdx.x < T) {
        dg[threadIdx.x] = S.dgcum[threadIdx.x];
        bcnt[threadIdx.x] = 0;
    }
    if (threadIdx.x <= T) goff[threadIdx.x] = S.goff[threadIdx.x];
    if (threadIdx.x == 0) s_first = 0x7fffffff;
    if (STAGED) {
        for (int j = threadIdx.x; j < k; j += kThreads) {
            const float* src = S.Cg + (int64_t)j * ldc;
            if (DP == 2) {
                *reinterpret_cast<float2*>(cgs + j * 2) = *reinterpret_cast<const float2*>(src);
            } else {
                for (int z = 0; z < sd; z++) cgs[j * sd + z] = src[z];
            }
            if (SI) {
                s_drift[j] = S.dcum[j];
                s_shalf[j] = S.s_half[j];
                s_cnorm[j] = S.cnorm[j];
                s_ginv[j] = S.ginv[j];
            }
        }
    }
    __syncthreads();
    const float* __restrict__ cg = STAGED ? cgs : S.Cg;
    const int cstride = STAGED ? sd : ldc;
    const float* __restrict__ c_dcum = SI ? s_drift : S.dcum;
    const float* __restrict__ c_shalf = SI ? s_shalf : S.s_half;
    const float* __restrict__ c_cnorm = SI ? s_cnorm : S.cnorm;
    const int* __restrict__ c_ginv = SI ? s_ginv : S.ginv;

    const float rho = simt_rel_err(S.d);
    const float cmax = S.scal[0];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t n_dist = 0, n_active = 0, n_need = 0, n_pairs = 0;
    int q0 = 0, p0 = 0;  // queued rows / pairs (block-uniform)

    // software pipeline: the label, ub and global bound of the next chunk are
    // loaded while this chunk is filtered, queued and (maybe) drained
    const int64_t cstep = (int64_t)gridDim.x * kThreads;
    int a_n = 0;
    float ub_n = 0.f, glb_n = 0.f;
    {
        const int64_t i0 = (int64_t)blockIdx.x * kThreads + threadIdx.x;
        if (i0 < S.n) {
            a_n = S.labels[i0];
            ub_n = S.ub[i0];
            glb_n = S.glb[i0];
        }
    }
    for (int64_t base = (int64_t)blockIdx.x * kThreads; base < S.n; base += cstep) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < S.n;
        bool need = false;
        unsigned mask = 0;
        const int a = a_n;
        const float ub_s = ub_n, glb_s = glb_n;
        {
            const int64_t in = i + cstep;
            if (in < S.n) {
                a_n = S.labels[in];
                ub_n = S.ub[in];
                glb_n = S.glb[in];
            }
        }
        float acc_a = 0.f, lun = INFINITY, xn = 0.f;
        float xr[DP];
#pragma unroll
        for (int z = 0; z < DP; z++) xr[z] = 0.f;

        // ---- filter.  Bounds are stored against cumulative drifts (lazy
        // encoding): u = ub_s + Dc[a] bounds d(x, c_a) from above, glb_s - Dm
        // and lb_s[g] - Dg[g] bound every other centroid (of group g) from
        // below, all with directed rounding.  A row that passes writes nothing.
        if (valid) {
            float u = __fadd_ru(ub_s, c_dcum[a]);
            const float sa = c_shalf[a];
            // Hamerly's separation test holds for every bound family
            const float gate = fmaxf(__fsub_rd(glb_s, dm), sa);
            if (!(gate > u)) {
                n_active++;
                // the group table, loaded alongside the point for the tighten
                float v[T];
                const float4* lp = reinterpret_cast<const float4*>(S.lb + i * T);
#pragma unroll
                for (int g4 = 0; g4 < T / 4; g4++) {
                    const float4 q4 = __ldcs(lp + g4);
                    v[4 * g4] = q4.x;
                    v[4 * g4 + 1] = q4.y;
                    v[4 * g4 + 2] = q4.z;
                    v[4 * g4 + 3] = q4.w;
                }
                const float* xp = S.X32 + i * S.ldx;
                const float* cp = STAGED ? cgs + c_ginv[a] * sd : S.C32 + (int64_t)a * ldc;
                float xn2 = 0.f;
#pragma unroll
                for (int z = 0; z < DP; z++) {
                    if (z < S.d) {
                        xr[z] = __ldg(xp + z);
                        const float t = xr[z] - cp[z];
                        acc_a = fmaf(t, t, acc_a);
                        xn2 = fmaf(xr[z], xr[z], xn2);
                    }
                }
                xn = sqrtf(xn2);
                const float U = (sqrtf(acc_a) + kU32 * (xn + c_cnorm[a])) * (1.0f + rho);
                const bool tight = U < u;
                u = fminf(u, U);
                if (!(gate > u)) {
                    float gmin = INFINITY;
#pragma unroll
                    for (int g = 0; g < T; g++) {
                        v[g] = __fsub_rd(v[g], dg[g]);  // a negative lower bound is still valid
                        gmin = fminf(gmin, v[g]);
                    }
                    need = !(fmaxf(gmin, sa) > u);
                    if (need) {
#pragma unroll
                        for (int g = 0; g < T; g++) {
                            if (v[g] > u) lun = fminf(lun, v[g]);
                            else mask |= 1u << g;
                        }
                    } else {
                        // the groups prune: keep their (tighter) minimum as the global bound
                        S.glb[i] = __fadd_rd(gmin, dm);
                    }
                }
                if (tight && !need) S.ub[i] = __fsub_ru(u, c_dcum[a]);
            }
        }

        // ---- enqueue this chunk's failing rows in chunk order, draining the
        // queue whenever the next row does not fit (a row has <= 32 pairs, so
        // an empty queue always takes it)
        const int cnt = __popc(mask);
        const unsigned nb = __ballot_sync(LK_FULL_MASK, need);
        int pincl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u2 = __shfl_up_sync(LK_FULL_MASK, pincl, o);
            if (lane >= o) pincl += u2;
        }
        if (lane == 31) {
            wrows[warp] = __popc(nb);
            wpairs[warp] = pincl;
        }
        __syncthreads();
        int rb = 0, pb = 0, rt = 0, pt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const int r = wrows[w], p = wpairs[w];
            rb += w < warp ? r : 0;
            pb += w < warp ? p : 0;
            rt += r;
            pt += p;
        }
        const int myr = rb + __popc(nb & lanemask_lt());  // rank among the chunk's failing rows
        const int myp = pb + pincl - cnt;                   // pairs before mine in the chunk
        if (need) {
            n_need++;
            n_pairs += cnt;
        }
        int rstart = 0, pstart = 0;
        bool queued = !need;
        while (rt > rstart) {
            const bool fits = !queued && (myr - rstart) < (kQRows - q0) &&
                              (myp - pstart) + cnt <= (pcap - p0);
            if (fits) {
                const int slot = q0 + myr - rstart;
                const int poff = p0 + myp - pstart;
                Q.row[slot] = (int)i;
                Q.a[slot] = a;
                Q.acc[slot] = acc_a;
                Q.xn[slot] = xn;
                Q.lun[slot] = lun;
                Q.mask[slot] = mask;
                Q.poff[slot] = poff;
                if (DP <= 4) {
#pragma unroll
                    for (int z = 0; z < DP; z++) Q.x[DP <= 4 ? slot : 0][z] = xr[z];
                }
                int p = poff;
                for (unsigned mm = mask; mm; mm &= mm - 1) {
                    const int g = __ffs(mm) - 1;
                    const int rank = atomicAdd(&bcnt[g], 1);
                    ptmp[p++] = (uint32_t)slot | ((uint32_t)g << 10) | ((uint32_t)rank << 16);
                }
                queued = true;
            }
            if (!queued) atomicMin(&s_first, (myr << 16) | myp);
            const int left = __syncthreads_or(!queued);
            if (!left) {
                q0 += rt - rstart;
                p0 += pt - pstart;
                break;
            }
            const int first = s_first;
            const int fr = first >> 16, fp = first & 0xffff;
            q0 += fr - rstart;
            p0 += fp - pstart;
            rstart = fr;
            pstart = fp;
            __syncthreads();  // everyone has read s_first
            if (threadIdx.x == 0) s_first = 0x7fffffff;
            drain<DP, T>(S, stat, qscale, Q, q0, p0, sh, cg, cstride, lg_parts, rho, cmax, n_dist);
            __syncthreads();  // the queue is free again
            q0 = 0;
            p0 = 0;
        }
    }
    if (q0 > 0) {
        __syncthreads();  // the last chunk's queue writes are visible
        drain<DP, T>(S, stat, qscale, Q, q0, p0, sh, cg, cstride, lg_parts, rho, cmax, n_dist);
    }
    warp_add(n_active, stat + LK_STAT_ACTIVE);
    warp_add(n_need, stat + LK_STAT_YWL);
    warp_add(n_pairs, stat + LK_STAT_PAIRS);
    warp_add(n_dist, stat + LK_STAT_DIST);
}

}  // namespace yyf
}  // namespace lk

namespace lkh {

using namespace lk::yyf;

template <int DP, int T, bool STAGED>
static lk_status launch_fused_t(const lk::DevState& S, int64_t* stat, const double* qscale,
                                int sms, size_t smem, int pcap, cudaStream_t st) {
    // lanes per (row, group) scan: split the average group into parts of >= 16
    // members, or of >= 96 member-dimensions when the rows are long
    const int gs = S.k / (S.t_groups > 0 ? S.t_groups : 1);
    int lg = 0;
    while (lg < 5 && (gs / (2 << lg) >= 16 || gs * DP / (2 << lg) >= 96)) lg++;
    auto kern = k_yy_fused<DP, T, STAGED>;
    int occ = 0;
    LK_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
    if (occ < 1) occ = 1;
    int64_t blocks = (S.n + kThreads - 1) / kThreads;
    if (blocks > (int64_t)sms * occ) blocks = (int64_t)sms * occ;
    if (blocks < 1) blocks = 1;
    LK_CUDA_CHECK(lk::launch_pdl(kern, dim3((unsigned)blocks), dim3(kThreads), smem, st, S, stat, qscale, pcap, lg));
    LK_LAUNCH_CHECK();
    return LK_OK;
}

template <int DP, int T>
static lk_status launch_fused_dp(const lk::DevState& S, int64_t* stat, const double* qscale,
                                 int sms, cudaStream_t st) {
    static const int pcap_env = [] {
        const char* e = getenv("LK_YY_PCAP");  // tuning knob: pair slots per block
        const int v = e ? atoi(e) : 0;
        return (v >= 256 && v <= 8192) ? v : kMaxPairs;
    }();
    const int pcap = pcap_env;
    const size_t pairs = (size_t)pcap * 4 + (size_t)((pcap + 1) & ~1) * 2 + (size_t)pcap * 12;
    const int sd = DP <= 4 ? DP : S.ldc;
    const size_t cg = (size_t)S.k * sd * 4 + (kStageInfo ? (size_t)S.k * 16 : 0);  // centroids (+ info)
    if (cg + pairs <= 64 * 1024)
        return launch_fused_t<DP, T, true>(S, stat, qscale, sms, cg + pairs, pcap, st);
    return launch_fused_t<DP, T, false>(S, stat, qscale, sms, pairs, pcap, st);
}

template <int T>
static lk_status launch_fused_tt(const lk::DevState& S, int64_t* stat, const double* qscale,
                                 int sms, cudaStream_t st) {
    const int d = S.d;
    if (d <= 2) return launch_fused_dp<2, T>(S, stat, qscale, sms, st);
    if (d <= 4) return launch_fused_dp<4, T>(S, stat, qscale, sms, st);
    if (d <= 8) return launch_fused_dp<8, T>(S, stat, qscale, sms, st);
    if (d <= 16) return launch_fused_dp<16, T>(S, stat, qscale, sms, st);
    return launch_fused_dp<32, T>(S, stat, qscale, sms, st);
}

// the fused path owns the lazy bound encoding (allocated for d <= 32, t <= 32
// and no tensor cores)
bool yy_fused_ok(const lk::DevState& S) { return S.lazy != 0 && !S.tgy; }

template <int DP, int T>
static lk_status fused_attr_dp() {
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_yy_fused<DP, T, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_yy_fused<DP, T, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    return LK_OK;
}

template <int T>
static lk_status fused_attr_t() {
    lk_status s = fused_attr_dp<2, T>();
    if (s == LK_OK) s = fused_attr_dp<4, T>();
    if (s == LK_OK) s = fused_attr_dp<8, T>();
    if (s == LK_OK) s = fused_attr_dp<16, T>();
    if (s == LK_OK) s = fused_attr_dp<32, T>();
    return s;
}

// called once per context, outside any stream capture
lk_status init_fused_attributes() {
    lk_status s = fused_attr_t<4>();
    if (s == LK_OK) s = fused_attr_t<8>();
    if (s == LK_OK) s = fused_attr_t<16>();
    if (s == LK_OK) s = fused_attr_t<32>();
    return s;
}

lk_status launch_yy_fused(const lk::DevState& S, int64_t* stat, const double* qscale, int sms,
                          cudaStream_t st) {
    const int t = S.t_groups;
    if (t <= 4) return launch_fused_tt<4>(S, stat, qscale, sms, st);
    if (t <= 8) return launch_fused_tt<8>(S, stat, qscale, sms, st);
    if (t <= 16) return launch_fused_tt<16>(S, stat, qscale, sms, st);
    return launch_fused_tt<32>(S, stat, qscale, sms, st);
}

}  // namespace lkh
