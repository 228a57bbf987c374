// lk_tc.cu -- tcgen05 (5th-gen tensor core) assignment kernel for d >= 32.
//
// Replaces the fp32 SIMT scan of assign_full (lloyd.py:69-75 / dist_matrix
// core.py:98-108) with a dot-product contraction on the tensor cores:
//
//   D'(i, j) = ||c_j||^2 - 2 x_i . c_j      (order-equivalent to ||x_i - c_j||^2)
//
// x . c is computed in 3xTF32 (x = x_hi + x_lo, c = c_hi + c_lo;
// x_hi c_hi + x_hi c_lo + x_lo c_hi) with fp32 accumulation in TMEM.  The
// epilogue keeps a per-row top-2 and certifies the winner with a rigorous
// error bound; rows it cannot certify go to
// the exact fp64 recheck, so labels equal the fp64 oracle's.
//
// Structure (one persistent CTA per SM, 192 threads):
//   warp 0      TMA producer (one elected lane): A = point rows (x_hi, x_lo),
//               B = centroid rows (c_hi, c_lo), 32-float K chunks, 128B swizzle
//   warp 1      MMA issuer (one elected lane) + TMEM allocator
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time, top-2 per row
// TMEM holds two BN-column fp32 accumulators (double buffer), so the epilogue
// of centroid tile t overlaps the MMAs of tile t+1.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include "lk_async.cuh"
#include "lk_common.cuh"
#include "lk_internal.h"

namespace lk {
namespace tc {

constexpr int BM = 128;        // rows per tile (UMMA M)
constexpr int KC = 32;         // fp32 elements per K chunk (128 bytes)
constexpr int UK = 8;          // UMMA K for kind::tf32
constexpr int kEpiWarps = 4;
constexpr int kMaxCand = LK_MAX_CAND;
constexpr int kThreadsTC = 64 + 32 * kEpiWarps;

// Dynamic shared memory: [stages][resident A (ARES)][barriers 256 B][beta x 2]
// ARES (d <= 32, one K chunk): a row tile's A (x_hi, x_lo) is loaded once and
// stays resident while the centroid tiles stream through the stages.
template <int BN, bool ARES = false>
struct Smem {
    static constexpr int A_BYTES = BM * KC * 4;   // 16 KB
    static constexpr int B_BYTES = BN * KC * 4;   // 16/32 KB
    static constexpr int STAGE_BYTES = ARES ? 2 * B_BYTES : 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int STAGES = ARES ? 4 : (BN == 256 ? 2 : 3);
    static constexpr int ARES_OFF = STAGES * STAGE_BYTES;
    static constexpr int BAR_OFF = ARES_OFF + (ARES ? 2 * A_BYTES : 0);
    static constexpr int BETA_OFF = BAR_OFF + 256;
    static constexpr int TOTAL = BETA_OFF + 1024 /*align*/;  // + 2 * kpad * 4 when staging beta
};

// ---- PTX helpers -----------------------------------------------------------

// (smem_u32, the mbarrier helpers and bulk_load: lk_async.cuh)

// wait without suspending the thread (A/B knob for the TMEM handoff latency)
__device__ __forceinline__ void mbar_wait_k(uint64_t* bar, uint32_t parity, int spin) {
    if (!spin) {
        mbar_wait(bar, parity);
        return;
    }
    const uint32_t addr = smem_u32(bar);
    while (!mbar_test(addr, parity)) {
    }
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// K-major, 128B-swizzled UMMA shared-memory descriptor (SBO = 8 rows x 128 B).
__device__ __forceinline__ uint64_t umma_desc(const void* p) {
    uint64_t a = (uint64_t)(smem_u32(p) >> 4) & 0x3FFF;
    return a | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: kind::tf32, fp32 accumulate, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

// tcgen05.commit arriving on the same barrier in every CTA of the mask
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        ::"r"(smem_u32(bar)), "h"(mask)
        : "memory");
}

// TMA tile load delivered to the same shared-memory offset (and barrier) in
// every CTA of the mask
__device__ __forceinline__ void tma_load_2d_mc(const CUtensorMap* map, uint64_t* bar, void* dst,
                                               int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld without the wait (several loads in flight, one tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Paired fp32 arithmetic (FADD2 / FFMA2 on sm_100a): two epilogue columns per
// instruction, each lane still rounded as its scalar counterpart.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
// (cc - 2 (vh + vx)) for two columns: exactly fmaf(-2, vh + vx, cc) per lane
__device__ __forceinline__ void dp2(float vh0, float vh1, float vx0, float vx1, float c0, float c1,
                                    float& d0, float& d1) {
    unsigned long long s, r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(pk2(vh0, vh1)), "l"(pk2(vx0, vx1)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(s), "l"(pk2(-2.0f, -2.0f)), "l"(pk2(c0, c1)));
    upk2(r, d0, d1);
}

// three-input fp32 minimum (FMNMX3 on sm_100a)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// (cc - 2 v) for two columns of a single accumulator: fmaf(-2, v, cc) per lane
__device__ __forceinline__ void dp2s(float v0, float v1, float c0, float c1, float& d0, float& d1) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(v0, v1)), "l"(pk2(-2.0f, -2.0f)), "l"(pk2(c0, c1)));
    upk2(r, d0, d1);
}

// Centroid id of B-operand column c (-1: padding).  Columns are centroid ids
// except on the group-tile path, where they are in group order (S.colperm).
__device__ __forceinline__ int col_id(const DevState& S, int c) {
    if (S.colperm) return c < S.kpad ? __ldg(S.colperm + c) : -1;
    return c < S.k ? c : -1;
}

// ---- certification (D-space error bound) ------------------------------------

// |D_true - D~| <= kappa * |x| |c| + 8u (|x|^2 + |c|^2) for the 3xTF32 form;
// kappa = 2 (3.1 * 2^-20 + (3d + 1) * 2^-22 * 1.01)  (split truncation terms +
// fp32 accumulation with a truncation-safe unit).
__device__ __forceinline__ float tc_kappa(int d) {
    return 2.0f * (3.1f * 9.5367431640625e-07f + (float)(3 * d + 1) * 2.384185791015625e-07f * 1.01f);
}

// Split accumulators: x_hi c_hi (exact tf32 x tf32 products) accumulates
// alone, the two cross terms in a second TMEM accumulator, summed in the
// epilogue.  The fp32 accumulation error of the dominant term then counts d
// additions instead of 3d + 1; the cross accumulator's is 2^-10 smaller, plus
// one rounding of the final sum:
//   kappa = 2 (3.1 * 2^-20 + (d + 2) * 2^-22 * 1.01 + d * 2^-31).
__device__ __forceinline__ float tc_kappa_split(int d) {
    return 2.0f * (3.1f * 9.5367431640625e-07f + (float)(d + 2) * 2.384185791015625e-07f * 1.01f +
                   (float)d * 4.656612873077393e-10f);
}

// One accumulator with every cross-term product added before the hi*hi
// products (d <= 32: one K chunk).  The 2d cross additions happen while the
// accumulator is at most ~2^-9 |x| |c| (units 2^-31), the d hi*hi additions at
// full magnitude:  kappa = 2 (3.1 * 2^-20 + (d + 2) * 2^-22 * 1.01 + (2d + 2) * 2^-31).
__device__ __forceinline__ float tc_kappa_ordered(int d) {
    return 2.0f * (3.1f * 9.5367431640625e-07f + (float)(d + 2) * 2.384185791015625e-07f * 1.01f +
                   (float)(2 * d + 2) * 4.656612873077393e-10f);
}

// Aggregated append over the kEpiWarps epilogue warps (named barrier 1).
// (the certifying warps are always the first kEpiWarps epilogue warps)
__device__ __forceinline__ int64_t epi_append(bool pred, unsigned long long* counter,
                                              unsigned long long* scr, int ew) {
    unsigned msk = __ballot_sync(LK_FULL_MASK, pred);
    if (lane_id() == 0) scr[ew] = __popc(msk);
    asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
    if (ew == 0 && lane_id() == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < kEpiWarps; w++) {
            unsigned long long c = scr[w];
            scr[w] = tot;
            tot += c;
        }
        scr[kEpiWarps] = tot ? atomicAdd(counter, tot) : 0ull;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
    int64_t pos = pred ? (int64_t)(scr[kEpiWarps] + scr[ew] + __popc(msk & lanemask_lt())) : -1;
    asm volatile("bar.sync 1, %0;" ::"r"(kEpiWarps * 32) : "memory");
    return pos;
}

// ---- the kernel --------------------------------------------------------------

struct TcArgs {
    int64_t m;            // rows of A (n for a full scan, worklist size for a rescan)
    const int32_t* rowlist;   // A row r -> global row (nullptr: identity)
    int center;           // A rows are label-sorted tiles shifted by a centroid (k_gather_center)
    int sbeta;            // centered: the tiles' beta rows are double-buffered in shared memory
    int fast;             // centered top-2: index-free chains + searched columns
    int spin;             // pipeline waits poll (test_wait) instead of suspending
    int dbg;              // timing probe only (wrong labels): 1 = no epilogue work, 2 = no MMAs
    int kouter;           // K-outer MMA order when the centroid tiles fit the TMEM buffers
    const int64_t* rowcount;  // device row count (overrides m when non-null)
    // device-side choice between a worklist pass and a dense pass over every
    // row (launch_assign_tc_adaptive): gate 1 runs only if *gate_cnt > gate_thr,
    // gate 2 only if *gate_cnt <= gate_thr, 0 always
    const int64_t* gate_cnt;
    int64_t gate_thr;
    int gate;
    unsigned long long* prof;  // k_assign_tgy phase clocks (LK_TGY_PROF debug knob), null: off
    int n_ct;             // centroid tiles
    int n_kc;             // K chunks
    // collect mode
    const float* thr;     // [m] D' threshold per A row
    int* slots;           // [m, kMaxCand]
    int* cnt;             // [m]
};

constexpr int kTop2 = 0;
constexpr int kCollect = 1;

template <bool SPLIT>
struct TcShape {
    static constexpr int EW = SPLIT ? 2 * kEpiWarps : kEpiWarps;  // epilogue warps
    static constexpr int THREADS = 64 + 32 * EW;
    static constexpr int NACC = SPLIT ? 2 : 1;                     // accumulators per tile
};

template <int BN, int MODE, bool SPLIT, bool ARES, int CL>
__global__ void __launch_bounds__(TcShape<SPLIT>::THREADS, 1)
    k_assign_tc(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                DevState S, TcArgs A, int64_t* stat) {
    if (*S.done) return;
    if (A.gate && ((*A.gate_cnt > A.gate_thr) != (A.gate == 1))) return;
    using SM = Smem<BN, ARES>;
    // ORD (d <= 32, one K chunk): one accumulator, every cross-term MMA before
    // the hi*hi MMAs -- the cross phase accumulates at 2^-10 of the final
    // magnitude, so the bound matches split accumulators while the epilogue
    // reads half the TMEM bytes (the TMEM read port, 64 B/clk/SM, paces the
    // d = 32 epilogue: 128 KB per 128 x 128 tile split, 64 KB ordered)
    constexpr bool ORD = SPLIT && ARES;
    constexpr int EW = TcShape<SPLIT>::EW, NACC = ORD ? 1 : TcShape<SPLIT>::NACC;
    // TMEM accumulator buffers: ORD holds four (the MMA runs up to three
    // centroid tiles ahead of the epilogue, hiding the MMA <-> epilogue handoff)
    constexpr int NBUF = ORD ? 4 : 2;
    static_assert(NBUF * NACC * BN <= 512, "TMEM holds 512 fp32 columns");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* abuf = smem + SM::ARES_OFF;    // resident A (ARES)
    uint64_t* full = (uint64_t*)(smem + SM::BAR_OFF);
    uint64_t* empty = full + SM::STAGES;
    uint64_t* tfull = empty + SM::STAGES;   // [NBUF]
    uint64_t* tempty = tfull + NBUF;        // [NBUF]
    uint64_t* afull = tempty + NBUF;        // resident A loaded
    uint64_t* aempty = afull + 1;           // resident A free (all MMAs of the row tile done)
    uint64_t* bfull = aempty + 1;           // [2] staged beta rows
    uint64_t* bempty = bfull + 2;           // [2]
    uint32_t* tmem_slot = (uint32_t*)(bempty + 2);
    float* sbeta = (float*)(smem + SM::BETA_OFF);  // [2][kpad] (A.sbeta)
    // per-centroid offsets of a tile: ||c_j||^2, or ||c_j - o||^2 when centered
    auto beta_src = [&](int64_t t_) -> const float* {
        if (!A.center) return S.cn2;
        const int at = S.tile_lab[t_];
        return at >= 0 ? S.ptab + (int64_t)at * S.kpad : S.cn2;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int PW = EW, MW = EW + 1;
    const int64_t m = A.rowcount ? *A.rowcount : A.m;
    const int64_t n_rt = (m + BM - 1) / BM;
    // row tiles of this CTA; a cluster (CL > 1) walks the centroid tiles in
    // lockstep, so every CTA of it runs the same count (tail tiles past n_rt
    // are dummies: zero / stale A rows, nothing written)
    const int n_it = CL == 1 ? (int)(n_rt > (int64_t)blockIdx.x ? (n_rt - blockIdx.x + gridDim.x - 1) / gridDim.x : 0)
                             : (int)((n_rt + gridDim.x - 1) / gridDim.x);
    uint32_t crank = 0;
    if (CL > 1) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    // K-outer order (d > 32, exactly NBUF centroid tiles: k <= 256): the row
    // tile's A chunk is consumed by both centroid tiles back to back (an L2 hit
    // the second time), instead of the whole row tile's A twice (cfg4: 800 KB
    // per CTA, re-read from DRAM)
    const bool kouter = !ARES && A.kouter && A.n_ct == NBUF && A.n_kc > 1;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < SM::STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CL);  // every CTA's MMA releases the stage (multicast loads)
        }
        for (int b = 0; b < NBUF; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EW);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&bfull[b], 1);
            mbar_init(&bempty[b], EW);
        }
        mbar_init(afull, 1);
        mbar_init(aempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_map(&map_ahi);
        prefetch_map(&map_alo);
        prefetch_map(&map_bhi);
        prefetch_map(&map_blo);
    }
    // roles: epilogue warps 0 .. EW-1, TMA producer EW, MMA issuer EW+1 (the
    // issuer has the highest warp id of its SM sub-partition: the scheduler
    // serves it first, so the MMA issue is never starved by epilogue warps)
    if (warp == MW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(NBUF * NACC * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    if (CL > 1) cluster_sync();  // the peers' barriers exist before any multicast
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == PW) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (; it < n_it; it++) {
                const int64_t rt = blockIdx.x + (int64_t)it * gridDim.x;
                if (A.sbeta) {
                    // the tile's beta row into the double buffer (freed by the epilogue)
                    const int bb = it & 1;
                    mbar_wait(&bempty[bb], ((it >> 1) & 1) ^ 1);
                    mbar_expect_tx(&bfull[bb], (uint32_t)S.kpad * 4);
                    bulk_load(sbeta + bb * S.kpad, rt < n_rt ? beta_src(rt) : S.cn2, (uint32_t)S.kpad * 4, &bfull[bb]);
                }
                if (ARES) {
                    mbar_wait(aempty, (it & 1) ^ 1);
                    mbar_expect_tx(afull, 2 * SM::A_BYTES);
                    tma_load_2d(&map_ahi, afull, abuf, 0, (int)(rt * BM));
                    tma_load_2d(&map_alo, afull, abuf + SM::A_BYTES, 0, (int)(rt * BM));
                }
                for (int uo = 0; uo < (kouter ? A.n_kc : A.n_ct); uo++) {
                    for (int ui = 0; ui < (kouter ? A.n_ct : A.n_kc); ui++) {
                        const int ct = kouter ? ui : uo;
                        const int kc = kouter ? uo : ui;
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* st = smem + stage * SM::STAGE_BYTES;
                        mbar_expect_tx(&full[stage], SM::STAGE_BYTES);
                        const int k0 = kc * KC;
                        uint8_t* bst = st + (ARES ? 0 : 2 * SM::A_BYTES);
                        if (!ARES) {
                            tma_load_2d(&map_ahi, &full[stage], st, k0, (int)(rt * BM));
                            tma_load_2d(&map_alo, &full[stage], st + SM::A_BYTES, k0, (int)(rt * BM));
                        }
                        if (ARES) {
                            // four 64-row parts (hi 0-63, hi 64-127, lo 0-63, lo 64-127);
                            // cluster CTA r loads parts r, r + CL, ... into every CTA
                            // of the cluster (the centroid tile is shared)
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                if (CL > 1 && (q % CL) != (int)crank) continue;
                                uint8_t* dst = bst + (q >> 1) * SM::B_BYTES + (q & 1) * (SM::B_BYTES / 2);
                                const CUtensorMap* mp = (q >> 1) ? &map_blo : &map_bhi;
                                const int row = ct * BN + (q & 1) * (BN / 2);
                                if (CL > 1) tma_load_2d_mc(mp, &full[stage], dst, k0, row, (uint16_t)((1u << CL) - 1));
                                else tma_load_2d(mp, &full[stage], dst, k0, row);
                            }
                        } else {
                            tma_load_2d(&map_bhi, &full[stage], bst, k0, ct * BN);
                            tma_load_2d(&map_blo, &full[stage], bst + SM::B_BYTES, k0, ct * BN);
                        }
                        if (++stage == SM::STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == MW) {
        // ===== MMA issuer: the whole warp runs the loop (converged, warp-uniform
        // descriptors), one elected lane issues each tcgen05 instruction
        {
            constexpr uint32_t idesc = idesc_tf32(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int it = 0;
            for (; it < n_it; it++) {
                const int64_t rt = blockIdx.x + (int64_t)it * gridDim.x;
                if (ARES) {
                    mbar_wait(afull, it & 1);
                    tc_fence_after();
                }
                // K-outer: both centroid tiles' accumulators stay live across the
                // K loop (buffers 0 and 1), so each A chunk is used twice in a row
                for (int uo = 0; uo < (kouter ? A.n_kc : A.n_ct); uo++) {
                    if (!kouter || uo == 0) {
                        for (int b = 0; b < (kouter ? NBUF : 1); b++)
                            mbar_wait_k(&tempty[kouter ? b : acc], acc_phase ^ 1, A.spin);
                        tc_fence_after();
                    }
                    for (int ui = 0; ui < (kouter ? A.n_ct : A.n_kc); ui++) {
                        const int ct = kouter ? ui : uo;
                        const int kc = kouter ? uo : ui;
                        const uint32_t tmem_d = tmem_base + (kouter ? ct : acc) * NACC * BN;
                        const uint32_t tmem_x = tmem_d + ((SPLIT && !ORD) ? BN : 0);
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        uint8_t* st = smem + stage * SM::STAGE_BYTES;
                        uint8_t* ast = ARES ? abuf : st;
                        uint8_t* bst = st + (ARES ? 0 : 2 * SM::A_BYTES);
                        const uint64_t dahi = umma_desc(ast);
                        const uint64_t dalo = umma_desc(ast + SM::A_BYTES);
                        const uint64_t dbhi = umma_desc(bst);
                        const uint64_t dblo = umma_desc(bst + SM::B_BYTES);
                        if (A.dbg == 2) {
                        } else if (ORD) {
                            // one K chunk: all cross terms, then all hi*hi terms
#pragma unroll
                            for (int k = 0; k < KC / UK; k++) {
                                const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                                mma_tf32(tmem_d, dalo + off, dbhi + off, idesc, k != 0);
                                mma_tf32(tmem_d, dahi + off, dblo + off, idesc, 1);
                            }
#pragma unroll
                            for (int k = 0; k < KC / UK; k++) {
                                const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                                mma_tf32(tmem_d, dahi + off, dbhi + off, idesc, 1);
                            }
                        } else
#pragma unroll
                        for (int k = 0; k < KC / UK; k++) {
                            const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                            if (SPLIT) {
                                // cross terms into their own accumulator, hi*hi alone
                                mma_tf32(tmem_x, dalo + off, dbhi + off, idesc, (kc | k) != 0);
                                mma_tf32(tmem_x, dahi + off, dblo + off, idesc, 1);
                                mma_tf32(tmem_d, dahi + off, dbhi + off, idesc, (kc | k) != 0);
                            } else {
                                // small terms first, then the dominant hi*hi term
                                mma_tf32(tmem_d, dalo + off, dbhi + off, idesc, (kc | k) != 0);
                                mma_tf32(tmem_d, dahi + off, dblo + off, idesc, 1);
                                mma_tf32(tmem_d, dahi + off, dbhi + off, idesc, 1);
                            }
                        }
                        if (CL > 1) mma_commit_mc(&empty[stage], (uint16_t)((1u << CL) - 1));
                        else mma_commit(&empty[stage]);
                        if (++stage == SM::STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (!kouter) {
                        mma_commit(&tfull[acc]);
                        if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
                    } else if (uo == A.n_kc - 1) {
                        for (int b = 0; b < NBUF; b++) mma_commit(&tfull[b]);
                        acc_phase ^= 1;  // (acc stays 0: the row tile used every buffer)
                    }
                }
                if (ARES) mma_commit(aempty);  // the resident A is free once these MMAs finish
            }
        }
    } else {
        // ===== epilogue: warps 0 .. EW-1, lane quarter = warp % 4 (TMEM access rule);
        // SPLIT: two warps per quarter take alternate 64-column halves (half h)
        // and merge their row top-2 through shared memory; the h = 0 warps certify
        const int q = warp & 3;
        const int h = warp >> 2;
        const int row_in_tile = q * 32 + lane;
        const float kappa = ORD ? tc_kappa_ordered(S.d) : SPLIT ? tc_kappa_split(S.d) : tc_kappa(S.d);
        int acc = 0;
        uint32_t acc_phase = 0;
        __shared__ unsigned long long escr[kEpiWarps + 1];
        __shared__ float xb1[2][BM], xb2[2][BM];
        __shared__ int xj1[2][BM];
        int par = 0;
        int it = 0;
        for (; it < n_it; it++) {
            const int64_t rt = blockIdx.x + (int64_t)it * gridDim.x;
            // centered runs: the producer staged this tile's beta row (bfull)
            const int bb = it & 1;
            const float* beta;
            if (A.sbeta) {
                mbar_wait(&bfull[bb], (it >> 1) & 1);
                beta = sbeta + bb * S.kpad;
            } else {
                beta = rt < n_rt ? beta_src(rt) : S.cn2;
            }
            const int64_t r = rt * BM + row_in_tile;
            const bool valid = r < m;
            // centered top-2 runs index-free chains (three FMNMX per column);
            // a lane searches a 64-column chunk for its column only when the
            // chunk takes the running minimum below bv.  bv starts at an upper
            // bound on the TC value of the row's own label column (rows of the
            // tile's label: D'_a = ||x'||^2 - R up to the dot error), so the
            // search runs about once per row instead of once per improvement.
            // A row whose minimum was never searched is left ambiguous.
            float bv = INFINITY;
            int bj = -1;
            // (rowbv: written by k_gather_center for rows of their tile's label)
            if (SPLIT && MODE == kTop2 && A.center && A.fast && valid) bv = __ldcs(S.rowbv + r);
            // MODE_TOP2: running top-2 of D' = |c|^2 - 2 x.c (ties keep the lower index)
            // MODE_COLLECT: every j with D' <= thr goes into the row's candidate slots
            float b1 = INFINITY, b2 = INFINITY;
            int j1 = 0;
            // SPLIT top-2: four chains over columns of residue e mod 4, merged below
            float cb1[4], cb2[4];
            int cj1[4];
#pragma unroll
            for (int e = 0; e < 4; e++) { cb1[e] = INFINITY; cb2[e] = INFINITY; cj1[e] = 0x7fffffff; }
            float thr = -INFINITY;
            int cnt = 0;
            int* slots = nullptr;
            // SPLIT collect: half h fills slots [h * kHalfCand, (h + 1) * kHalfCand)
            constexpr int kHalfCand = kMaxCand / 2;
            const int cap = (SPLIT && MODE == kCollect) ? kHalfCand : kMaxCand;
            if (MODE == kCollect && valid) {
                thr = A.thr[r];
                slots = A.slots + r * kMaxCand + ((SPLIT && h) ? kHalfCand : 0);
            }
            for (int ct = 0; ct < A.n_ct; ct++) {
                mbar_wait_k(&tfull[acc], acc_phase, A.spin);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * NACC * BN;
                const int jbase = ct * BN;
                if (A.dbg == 1) {
                } else if (SPLIT && MODE == kCollect) {
                    // this warp's 64 columns: every j under the row's threshold
                    const int c0 = h * 64;
                    uint32_t r0[32], r1[32], x0[32], x1[32];
                    tmem_ld32_async(taddr + c0, r0);
                    tmem_ld32_async(taddr + c0 + 32, r1);
                    if (!ORD) {  // (ORD: one accumulator, the cross arrays stay unused)
                        tmem_ld32_async(taddr + BN + c0, x0);
                        tmem_ld32_async(taddr + BN + c0 + 32, x1);
                    }
                    const int jb = jbase + c0;
                    const float4* cp = reinterpret_cast<const float4*>(S.cn2 + jb);
                    tmem_wait_ld();
                    unsigned hit0 = 0, hit1 = 0;  // columns under the threshold
#pragma unroll
                    for (int c4 = 0; c4 < 16; c4++) {
                        const float4 cv = __ldg(cp + c4);
                        const float cc[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const int col = c4 * 4 + e;
                            const float vh = __uint_as_float(col < 32 ? r0[col & 31] : r1[col & 31]);
                            const float vx = ORD ? 0.f : __uint_as_float(col < 32 ? x0[col & 31] : x1[col & 31]);
                            const bool in = (ORD ? fmaf(-2.0f, vh, cc[e]) : fmaf(-2.0f, vh + vx, cc[e])) <= thr;
                            if (col < 32) hit0 |= (unsigned)in << (col & 31);
                            else hit1 |= (unsigned)in << (col & 31);
                        }
                    }
                    if (valid) {
                        for (unsigned m = hit0; m; m &= m - 1) {
                            if (cnt < cap) slots[cnt] = col_id(S, jb + __ffs(m) - 1);
                            cnt++;
                        }
                        for (unsigned m = hit1; m; m &= m - 1) {
                            if (cnt < cap) slots[cnt] = col_id(S, jb + 32 + __ffs(m) - 1);
                            cnt++;
                        }
                    }
                }
                if (SPLIT && MODE == kTop2 && A.dbg != 1) {
                    // this warp's 64 columns of both accumulators: four loads in
                    // flight, one wait; four independent top-2 chains (ILP)
                    const int c0 = h * 64;
                    uint32_t r0[32], r1[32], x0[32], x1[32];
                    tmem_ld32_async(taddr + c0, r0);
                    tmem_ld32_async(taddr + c0 + 32, r1);
                    if (!ORD) {
                        tmem_ld32_async(taddr + BN + c0, x0);
                        tmem_ld32_async(taddr + BN + c0 + 32, x1);
                    }
                    const int jb = jbase + c0;
                    const float4* cp = reinterpret_cast<const float4*>(beta + jb);
                    // staged beta: explicit shared-memory loads (a select between a
                    // shared and a global pointer compiles to slow generic loads)
                    const uint32_t sb = smem_u32(sbeta + bb * S.kpad + jb);
                    tmem_wait_ld();
                    auto chunk_dp = [&](int c4, float (&dpv)[4]) {
                        float4 cv;
                        if (A.sbeta) {
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(cv.x), "=f"(cv.y), "=f"(cv.z), "=f"(cv.w)
                                         : "r"(sb + 16 * c4));
                        } else {
                            cv = __ldg(cp + c4);
                        }
                        const float cc[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                        for (int e = 0; e < 4; e += 2) {
                            const int col = c4 * 4 + e;
                            const float vh0 = __uint_as_float(col < 32 ? r0[col & 31] : r1[col & 31]);
                            const float vh1 = __uint_as_float(col < 32 ? r0[(col + 1) & 31] : r1[(col + 1) & 31]);
                            if (ORD) {
                                dp2s(vh0, vh1, cc[e], cc[e + 1], dpv[e], dpv[e + 1]);
                            } else {
                                const float vx0 = __uint_as_float(col < 32 ? x0[col & 31] : x1[col & 31]);
                                const float vx1 = __uint_as_float(col < 32 ? x0[(col + 1) & 31] : x1[(col + 1) & 31]);
                                dp2(vh0, vh1, vx0, vx1, cc[e], cc[e + 1], dpv[e], dpv[e + 1]);
                            }
                        }
                    };
                    if (A.center && A.fast) {
                        // the chunk's 64 values, their minimum (FMNMX3 tree); the
                        // lane's running (b1, b2) = (cb1[0], cb2[0]) changes only when
                        // the chunk holds a value below b2, which after the first
                        // chunks is rare for every row of a (single-cluster) tile:
                        // the exact top-2 update runs only then, warp-uniformly
                        float dv[64];
#pragma unroll
                        for (int c4 = 0; c4 < 16; c4++) {
                            float dpv[4];
                            chunk_dp(c4, dpv);
#pragma unroll
                            for (int e = 0; e < 4; e++) dv[c4 * 4 + e] = dpv[e];
                        }
                        float m21[22];
#pragma unroll
                        for (int i = 0; i < 21; i++) m21[i] = fmin3(dv[3 * i], dv[3 * i + 1], dv[3 * i + 2]);
                        m21[21] = dv[63];
                        float m8[8];
#pragma unroll
                        for (int i = 0; i < 7; i++) m8[i] = fmin3(m21[3 * i], m21[3 * i + 1], m21[3 * i + 2]);
                        m8[7] = m21[21];
                        const float mc = fmin3(fmin3(m8[0], m8[1], m8[2]), fmin3(m8[3], m8[4], m8[5]),
                                               fminf(m8[6], m8[7]));
                        if (__any_sync(LK_FULL_MASK, mc < cb2[0])) {
                            // exact top-2 over the pairs, two chains
                            float a1 = cb1[0], a2 = cb2[0], c1 = INFINITY, c2 = INFINITY;
#pragma unroll
                            for (int pp = 0; pp < 32; pp += 2) {
                                const float lo0 = fminf(dv[2 * pp], dv[2 * pp + 1]);
                                const float hi0 = fmaxf(dv[2 * pp], dv[2 * pp + 1]);
                                a2 = fmin3(fmaxf(a1, lo0), a2, hi0);
                                a1 = fminf(a1, lo0);
                                const float lo1 = fminf(dv[2 * pp + 2], dv[2 * pp + 3]);
                                const float hi1 = fmaxf(dv[2 * pp + 2], dv[2 * pp + 3]);
                                c2 = fmin3(fmaxf(c1, lo1), c2, hi1);
                                c1 = fminf(c1, lo1);
                            }
                            cb2[0] = fmin3(fmaxf(a1, c1), a2, c2);
                            cb1[0] = fminf(a1, c1);
                            const bool imp = cb1[0] < bv;
                            if (__any_sync(LK_FULL_MASK, imp)) {
                                // the lowest column holding the new minimum
                                int found = -1;
#pragma unroll
                                for (int e = 63; e >= 0; e--)
                                    if (dv[e] == cb1[0]) found = jb + e;
                                if (imp) {
                                    bv = cb1[0];
                                    bj = found;
                                }
                            }
                        }
                    } else {
#pragma unroll
                        for (int c4 = 0; c4 < 16; c4++) {
                            float dpv[4];
                            chunk_dp(c4, dpv);
#pragma unroll
                            for (int e = 0; e < 4; e++) {
                                const int col = c4 * 4 + e;
                                const float dp = dpv[e];
                                if (dp < cb1[e]) { cb2[e] = cb1[e]; cb1[e] = dp; cj1[e] = jb + col; }
                                else cb2[e] = fminf(cb2[e], dp);
                            }
                        }
                    }
                }
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    if (SPLIT) break;  // handled above
                    float v[32];
                    tmem_ld32(taddr + c0, v);
                    if (SPLIT) {
                        float vx[32];
                        tmem_ld32(taddr + BN + c0, vx);
#pragma unroll
                        for (int e = 0; e < 32; e++) v[e] += vx[e];
                    }
                    const int jb = jbase + c0;
                    // cn2 is padded with +inf beyond k (zero-filled B rows give v = 0)
                    const float4* cp = reinterpret_cast<const float4*>(S.cn2 + jb);
#pragma unroll
                    for (int c4 = 0; c4 < 8; c4++) {
                        const float4 cv = __ldg(cp + c4);
                        const float cc[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const float dp = fmaf(-2.0f, v[c4 * 4 + e], cc[e]);
                            if (MODE == kTop2) {
                                if (dp < b1) { b2 = b1; b1 = dp; j1 = jb + c4 * 4 + e; }
                                else b2 = fminf(b2, dp);
                            } else {
                                if (valid && dp <= thr) {
                                    if (cnt < cap) slots[cnt] = col_id(S, jb + c4 * 4 + e);
                                    cnt++;
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
            }
            if (A.sbeta && lane == 0) mbar_arrive(&bempty[bb]);  // this tile's beta row is free
            if (A.dbg) continue;  // timing probe: no certification
            if (MODE == kCollect) {
                if (SPLIT) {
                    // the h = 0 warp appends the other half's slots after its own
                    if (h == 1) xj1[par][row_in_tile] = cnt;
                    asm volatile("bar.sync 2, %0;" ::"r"(EW * 32) : "memory");
                    const int cur = par;
                    par ^= 1;
                    if (h == 1) continue;
                    const int c1 = xj1[cur][row_in_tile];
                    if (valid && cnt <= kHalfCand && c1 <= kHalfCand) {
                        int* row_slots = A.slots + r * kMaxCand;
                        for (int e = 0; e < c1; e++) row_slots[cnt + e] = row_slots[kHalfCand + e];
                    }
                    cnt += c1;
                    if (cnt <= kMaxCand && (cnt - c1 > kHalfCand || c1 > kHalfCand))
                        cnt = kMaxCand + 1;  // a half overflowed its slots
                }
                if (valid) A.cnt[r] = cnt;
                continue;
            }
            if (SPLIT) {
                // merge the four chains, then the two halves, in (value, index) order
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if (cb1[e] < b1 || (cb1[e] == b1 && cj1[e] < j1)) {
                        b2 = fminf(b1, cb2[e]);
                        b1 = cb1[e];
                        j1 = cj1[e];
                    } else {
                        b2 = fminf(b2, cb1[e]);
                    }
                }
                // index-free chains: the searched column holds the minimum, or none is known
                if (A.center && A.fast) j1 = (bj >= 0 && bv == b1) ? bj : -1;
                if (h == 1) {
                    xb1[par][row_in_tile] = b1;
                    xb2[par][row_in_tile] = b2;
                    xj1[par][row_in_tile] = j1;
                }
                asm volatile("bar.sync 2, %0;" ::"r"(EW * 32) : "memory");
                const int cur = par;
                par ^= 1;
                if (h == 1) continue;
                const float ob1 = xb1[cur][row_in_tile], ob2 = xb2[cur][row_in_tile];
                const int oj1 = xj1[cur][row_in_tile];
                if (ob1 < b1 || (ob1 == b1 && oj1 < j1)) {
                    b2 = fminf(b1, ob2);
                    b1 = ob1;
                    j1 = oj1;
                } else {
                    b2 = fminf(b2, ob1);
                }
            }
            // certify this row; ambiguous rows get a candidate threshold
            int64_t row = 0;
            bool moved = false, amb = false;
            int old = 0;
            float thr_out = 0.f, lb_out = 0.f;
            if (valid) {
                if (S.colperm && j1 >= 0) j1 = col_id(S, j1);  // (a column of the group tiles)
                row = A.rowlist ? (int64_t)A.rowlist[r] : r;
                const float xn2 = A.center ? S.rowxn2[r] : S.xn2[row];  // (contiguous copy when gathered)
                const float xn = sqrtf(xn2) * (1.0f + 2 * kU32);
                const float cn1 = j1 >= 0 ? S.cnorm[j1] : S.scal[0];  // (unknown column: max |c|)
                const float cmax = S.scal[0];
                if (A.center) {
                    // D_j = R + D'_j with D'_j = beta_j - 2 x'.c_j (x' = x - o).  Errors:
                    // the dot, kappa |x'| |c_j|; beta (fp32 difference form),
                    // (d + 4) u beta_j with beta_j <= |D'_j| + 2 |x'| |c_j|; the final
                    // FFMA, u |D'_j|; and x' = fl(x - o) moves the point by
                    // delta <= 2^-24 |x'|: |dD| <= delta (2 sqrt(D) + delta).
                    // L2 is evaluated at the second-smallest D'~ (the lower bound
                    // over j != j1 is increasing in D'~_j).
                    const double R = S.rowR[r];
                    const double xo = (double)S.rowxo[r];
                    const double gb = (double)(S.d + 4) * 5.9604644775390625e-08;
                    const double e1 = (double)kappa * xo * cn1 + gb * (fabs((double)b1) + 2.0 * xo * cn1) +
                                      2.0 * 5.9604644775390625e-08 * fabs((double)b1);
                    const double eo = (double)kappa * xo * cmax + gb * (fabs((double)b2) + 2.0 * xo * cmax) +
                                      2.0 * 5.9604644775390625e-08 * fabs((double)b2);
                    const double ex = isinf(b2) ? 0.0
                                      : 2.384185791015625e-07 * xo * (sqrt(fmax(R + b2 + eo, 0.0)) + xo);
                    const double U = (R + b1 + e1 + ex) * (1.0 + 1e-12) + 1e-300;
                    const double L2 = isinf(b2) ? INFINITY : (R + b2 - eo - ex) - fabs(R) * 1e-12;
                    if (L2 > U && j1 >= 0) {
                        old = S.rowlab[r];
                        moved = old != j1;
                        if (moved) S.labels[row] = j1;
                        if (S.strategy != LK_STRAT_LLOYD) {
                            S.ub[row] = store_ub(S, __double2float_ru(sqrt(fmax(U, 0.0)) * (1.0 + 1e-12)), j1);
                            write_lb_all(S, row, isinf(L2) ? INFINITY
                                                            : __double2float_rd(sqrt(fmax(L2, 0.0)) * (1.0 - 1e-12)));
                        }
                    } else {
                        // thresholds of the (uncentered) collect pass: D'unc_j = ||c_j||^2
                        // - 2 x.c_j; every possible winner has D_j <= U, so
                        // D'unc~_j <= U - ||x||^2 + e_unc
                        amb = true;
                        const double eunc = (double)kappa * xn * cmax + 8.0 * 5.9604644775390625e-08 *
                                            ((double)xn2 + (double)cmax * cmax);
                        const double thr = (U - (double)xn2 * (1.0 - 2.384185791015625e-07) + eunc) *
                                           (1.0 + 1e-9) + 1e-30;
                        thr_out = __double2float_ru(thr);
                        lb_out = __double2float_rd(sqrt(fmax(U, 0.0)) * (1.0 - 1e-12));
                    }
                } else {
                const float e1 = kappa * xn * cn1 + 8.0f * kU32 * (xn2 + cn1 * cn1);
                const float eo = kappa * xn * cmax + 8.0f * kU32 * (xn2 + cmax * cmax);
                const float U = (xn2 + b1) + e1;
                const float L2 = (xn2 + b2) - eo;
                if (L2 > U) {
                    old = S.labels[row];
                    moved = old != j1;
                    S.labels[row] = j1;
                    if (S.strategy != LK_STRAT_LLOYD) {
                        S.ub[row] = store_ub(S, __fsqrt_ru(fmaxf(U, 0.f)), j1);
                        write_lb_all(S, row, isinf(L2) ? INFINITY : __fsqrt_rd(fmaxf(L2, 0.f)));
                    }
                } else {
                    // any possible winner j has D'_j <= U - xn2 + e_j <= thr
                    amb = true;
                    thr_out = (b1 + e1 + eo) * (1.0f + 4 * kU32) + fabsf(b1) * 4 * kU32 + 1e-30f;
                    lb_out = __fsqrt_rd(fmaxf(U, 0.f));
                }
                }
            }
            // 128-thread aggregated appends across the epilogue warps (named barrier 1)
            int64_t pos = epi_append(moved, (unsigned long long*)(stat + LK_STAT_CHANGED), escr, warp);
            if (moved) S.moved[pos] = make_int2((int)row, old);
            int64_t cpos = epi_append(amb, (unsigned long long*)(stat + LK_STAT_CANDIDATE), escr, warp);
            if (amb) {
                S.cand_rows[cpos] = (int)row;
                S.cand_thr[cpos] = thr_out;
                S.cand_lb[cpos] = lb_out;
            }
        }
    }
    __syncthreads();
    if (CL > 1) cluster_sync();  // no CTA leaves while a peer may still write its shared memory
    if (warp == MW) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(NBUF * NACC * BN));
    }
}

// ---- d <= 32: two row tiles per centroid tile ---------------------------------
//
// With one K chunk (d <= 32) a 128 x 128 tile is 12 MMAs (~800 clk) against a
// 32 KB centroid tile (hi + lo) from L2; the TMA round trip under full load
// (~2.5-3 us) then bounds the single-row-tile pipeline at ~1.4 us per tile
// (measured: a no-MMA / no-epilogue probe of k_assign_tc ran 62 ms on cfg5).
// Here each CTA holds two row tiles (256 rows, A resident: 64 KB) against every
// staged centroid tile, so the same bytes in flight feed twice the MMA work.
// Epilogue warps own whole rows (warp w: lane quarter w % 4 of row tile w / 4),
// top-2 by chunk minima (FMNMX3) with the exact update only for chunks that
// reach a row's second-best; certification as in k_assign_tc.

struct Tc2Smem {
    static constexpr int B_BYTES = 128 * KC * 4;       // 16 KB (hi or lo)
    static constexpr int STAGE_BYTES = 2 * B_BYTES;     // 32 KB
    static constexpr int STAGES = 3;
    static constexpr int A_BYTES = BM * KC * 4;         // 16 KB per row tile and half
    static constexpr int A_OFF = STAGES * STAGE_BYTES;  // 96 KB
    static constexpr int BAR_OFF = A_OFF + 4 * A_BYTES; // + 64 KB
    static constexpr int BETA_OFF = BAR_OFF + 256;      // + 2 x kpad floats (the pair's beta rows)
    static constexpr int TOTAL = BETA_OFF + 1024;       // (+ 8 * kpad at launch)
};

// Certify one row from its top-2 D'~ (b1 at column j1 >= 0, b2), exactly as
// the k_assign_tc epilogue does.  Outputs: the global row, moved / old label,
// or an ambiguous row's collect threshold and lower bound.
__device__ __forceinline__ void tc_certify(const DevState& S, const TcArgs& A, float kappa, int64_t r,
                                           float b1, float b2, int j1, int64_t& row, bool& moved,
                                           int& old, bool& amb, float& thr_out, float& lb_out) {
    row = A.rowlist ? (int64_t)A.rowlist[r] : r;
    const float xn2 = A.center ? S.rowxn2[r] : S.xn2[row];
    const float xn = sqrtf(xn2) * (1.0f + 2 * kU32);
    const float cmax = S.scal[0];
    const float cn1 = j1 >= 0 ? S.cnorm[j1] : cmax;  // (unknown column: max |c|)
    if (A.center) {
        const double R = S.rowR[r];
        const double xo = (double)S.rowxo[r];
        const double gb = (double)(S.d + 4) * 5.9604644775390625e-08;
        const double e1 = (double)kappa * xo * cn1 + gb * (fabs((double)b1) + 2.0 * xo * cn1) +
                          2.0 * 5.9604644775390625e-08 * fabs((double)b1);
        const double eo = (double)kappa * xo * cmax + gb * (fabs((double)b2) + 2.0 * xo * cmax) +
                          2.0 * 5.9604644775390625e-08 * fabs((double)b2);
        const double ex = isinf(b2) ? 0.0 : 2.384185791015625e-07 * xo * (sqrt(fmax(R + b2 + eo, 0.0)) + xo);
        const double U = (R + b1 + e1 + ex) * (1.0 + 1e-12) + 1e-300;
        const double L2 = isinf(b2) ? INFINITY : (R + b2 - eo - ex) - fabs(R) * 1e-12;
        if (L2 > U && j1 >= 0) {
            old = S.rowlab[r];
            moved = old != j1;
            if (moved) S.labels[row] = j1;
            if (S.strategy != LK_STRAT_LLOYD) {
                S.ub[row] = store_ub(S, __double2float_ru(sqrt(fmax(U, 0.0)) * (1.0 + 1e-12)), j1);
                write_lb_all(S, row, isinf(L2) ? INFINITY : __double2float_rd(sqrt(fmax(L2, 0.0)) * (1.0 - 1e-12)));
            }
        } else {
            amb = true;
            const double eunc = (double)kappa * xn * cmax + 8.0 * 5.9604644775390625e-08 *
                                ((double)xn2 + (double)cmax * cmax);
            const double thr = (U - (double)xn2 * (1.0 - 2.384185791015625e-07) + eunc) * (1.0 + 1e-9) + 1e-30;
            thr_out = __double2float_ru(thr);
            lb_out = __double2float_rd(sqrt(fmax(U, 0.0)) * (1.0 - 1e-12));
        }
    } else {
        const float e1 = kappa * xn * cn1 + 8.0f * kU32 * (xn2 + cn1 * cn1);
        const float eo = kappa * xn * cmax + 8.0f * kU32 * (xn2 + cmax * cmax);
        const float U = (xn2 + b1) + e1;
        const float L2 = (xn2 + b2) - eo;
        if (L2 > U && j1 >= 0) {
            old = S.labels[row];
            moved = old != j1;
            S.labels[row] = j1;
            if (S.strategy != LK_STRAT_LLOYD) {
                S.ub[row] = store_ub(S, __fsqrt_ru(fmaxf(U, 0.f)), j1);
                write_lb_all(S, row, isinf(L2) ? INFINITY : __fsqrt_rd(fmaxf(L2, 0.f)));
            }
        } else {
            amb = true;
            thr_out = (b1 + e1 + eo) * (1.0f + 4 * kU32) + fabsf(b1) * 4 * kU32 + 1e-30f;
            lb_out = __fsqrt_rd(fmaxf(U, 0.f));
        }
    }
}

// Aggregated append over the 8 epilogue warps (named barrier 1, 256 threads).
__device__ __forceinline__ int64_t epi_append8(bool pred, unsigned long long* counter,
                                               unsigned long long* scr, int ew) {
    unsigned msk = __ballot_sync(LK_FULL_MASK, pred);
    if (lane_id() == 0) scr[ew] = __popc(msk);
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (ew == 0 && lane_id() == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < 8; w++) {
            unsigned long long c = scr[w];
            scr[w] = tot;
            tot += c;
        }
        scr[8] = tot ? atomicAdd(counter, tot) : 0ull;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    int64_t pos = pred ? (int64_t)(scr[8] + scr[ew] + __popc(msk & lanemask_lt())) : -1;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    return pos;
}

__global__ void __launch_bounds__(320, 1)
    k_assign_tc2(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                 const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                 DevState S, TcArgs A, int64_t* stat) {
    if (*S.done) return;
    if (A.gate && ((*A.gate_cnt > A.gate_thr) != (A.gate == 1))) return;  // (launch_assign_tc_adaptive)
    using SM = Tc2Smem;
    constexpr int BN = 128, NBUF = 2, PW = 8, MW = 9;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* abuf = smem + SM::A_OFF;  // [row tile s][hi, lo]
    uint64_t* full = (uint64_t*)(smem + SM::BAR_OFF);
    uint64_t* empty = full + SM::STAGES;
    uint64_t* tfull = empty + SM::STAGES;  // [NBUF]
    uint64_t* tempty = tfull + NBUF;       // [NBUF]
    uint64_t* afull = tempty + NBUF;
    uint64_t* aempty = afull + 1;
    uint64_t* bfull = aempty + 1;   // the pair's beta rows staged
    uint64_t* bempty = bfull + 1;   // ... and released by the epilogue
    uint32_t* tmem_slot = (uint32_t*)(bempty + 1);
    float* sbeta = (float*)(smem + SM::BETA_OFF);  // [2][kpad]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m = A.rowcount ? *A.rowcount : A.m;
    const int64_t n_rt = (m + BM - 1) / BM;
    const int64_t n_rp = (n_rt + 1) / 2;  // row-tile pairs
    // beta row of row tile t: ||c_j||^2, or ||c_j - o||^2 of its centroid o (centered)
    auto beta_of = [&](int64_t t_) -> const float* {
        if (!A.center || t_ >= n_rt) return S.cn2;
        const int at = S.tile_lab[t_];
        return at >= 0 ? S.ptab + (int64_t)at * S.kpad : S.cn2;
    };
    const int n_it = (int)(n_rp > (int64_t)blockIdx.x ? (n_rp - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < SM::STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);
        }
        mbar_init(afull, 1);
        mbar_init(aempty, 1);
        mbar_init(bfull, 1);
        mbar_init(bempty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_map(&map_ahi);
        prefetch_map(&map_alo);
        prefetch_map(&map_bhi);
        prefetch_map(&map_blo);
    }
    if (warp == MW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == PW) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int it = 0; it < n_it; it++) {
                const int64_t rp = blockIdx.x + (int64_t)it * gridDim.x;
                // the pair's beta rows (single buffer: after the epilogue's last use)
                mbar_wait(bempty, (it & 1) ^ 1);
                mbar_expect_tx(bfull, (uint32_t)S.kpad * 8);
                bulk_load(sbeta, beta_of(2 * rp), (uint32_t)S.kpad * 4, bfull);
                bulk_load(sbeta + S.kpad, beta_of(2 * rp + 1), (uint32_t)S.kpad * 4, bfull);
                mbar_wait(aempty, (it & 1) ^ 1);
                mbar_expect_tx(afull, 4 * SM::A_BYTES);
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    const int row0 = (int)((2 * rp + s) * BM);  // past the end: zero fill
                    tma_load_2d(&map_ahi, afull, abuf + s * 2 * SM::A_BYTES, 0, row0);
                    tma_load_2d(&map_alo, afull, abuf + s * 2 * SM::A_BYTES + SM::A_BYTES, 0, row0);
                }
                for (int ct = 0; ct < A.n_ct; ct++) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* bst = smem + stage * SM::STAGE_BYTES;
                    mbar_expect_tx(&full[stage], SM::STAGE_BYTES);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        uint8_t* dst = bst + (q >> 1) * SM::B_BYTES + (q & 1) * (SM::B_BYTES / 2);
                        tma_load_2d((q >> 1) ? &map_blo : &map_bhi, &full[stage], dst, 0,
                                    ct * BN + (q & 1) * (BN / 2));
                    }
                    if (++stage == SM::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == MW) {
        // ===== MMA issuer (whole warp, one elected lane issues) =====
        constexpr uint32_t idesc = idesc_tf32(BM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int it = 0; it < n_it; it++) {
            mbar_wait(afull, it & 1);
            tc_fence_after();
            for (int ct = 0; ct < A.n_ct; ct++) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                uint8_t* bst = smem + stage * SM::STAGE_BYTES;
                const uint64_t dbhi = umma_desc(bst);
                const uint64_t dblo = umma_desc(bst + SM::B_BYTES);
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    const uint32_t tmem_d = tmem_base + acc * 2 * BN + s * BN;
                    const uint64_t dahi = umma_desc(abuf + s * 2 * SM::A_BYTES);
                    const uint64_t dalo = umma_desc(abuf + s * 2 * SM::A_BYTES + SM::A_BYTES);
                    // one accumulator: every cross term, then every hi*hi term (ORD)
#pragma unroll
                    for (int k = 0; k < KC / UK; k++) {
                        const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                        mma_tf32(tmem_d, dalo + off, dbhi + off, idesc, k != 0);
                        mma_tf32(tmem_d, dahi + off, dblo + off, idesc, 1);
                    }
#pragma unroll
                    for (int k = 0; k < KC / UK; k++) {
                        const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                        mma_tf32(tmem_d, dahi + off, dbhi + off, idesc, 1);
                    }
                }
                mma_commit(&empty[stage]);
                if (++stage == SM::STAGES) { stage = 0; phase ^= 1; }
                mma_commit(&tfull[acc]);
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
            }
            mma_commit(aempty);  // both resident row tiles are free once these MMAs finish
        }
    } else {
        // ===== epilogue: warp w = rows 32 (w % 4) .. of row tile w / 4 =====
        const int q = warp & 3, s = warp >> 2;
        const float kappa = tc_kappa_ordered(S.d);
        __shared__ unsigned long long escr[9];
        int acc = 0;
        uint32_t acc_phase = 0;
        // search thresholds (rowbv, written by k_gather_center) one pair ahead
        auto load_bv = [&](int it_) -> float {
            if (!A.center || it_ >= n_it) return INFINITY;
            const int64_t r_ = (2 * (blockIdx.x + (int64_t)it_ * gridDim.x) + s) * BM + q * 32 + lane;
            return r_ < m ? __ldcs(S.rowbv + r_) : INFINITY;
        };
        float bv_next = load_bv(0);
        for (int it = 0; it < n_it; it++) {
            const int64_t rp = blockIdx.x + (int64_t)it * gridDim.x;
            const int64_t rt = 2 * rp + s;
            const int64_t r = rt * BM + q * 32 + lane;
            const bool valid = r < m;
            float b1 = INFINITY, b2 = INFINITY, bv = bv_next;
            int bj = -1;
            bv_next = load_bv(it + 1);
            mbar_wait(bfull, it & 1);
            const uint32_t sb0 = smem_u32(sbeta + s * S.kpad);
            for (int ct = 0; ct < A.n_ct; ct++) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 2 * BN + s * BN;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 64) {
                    uint32_t r0[32], r1[32];
                    tmem_ld32_async(taddr + c0, r0);
                    tmem_ld32_async(taddr + c0 + 32, r1);
                    const int jb = ct * BN + c0;
                    const uint32_t sb = sb0 + 4 * jb;
                    float4 cv[16];
#pragma unroll
                    for (int c4 = 0; c4 < 16; c4++)
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(cv[c4].x), "=f"(cv[c4].y), "=f"(cv[c4].z), "=f"(cv[c4].w)
                                     : "r"(sb + 16 * c4));
                    tmem_wait_ld();
                    float dv[64];
#pragma unroll
                    for (int c4 = 0; c4 < 16; c4++) {
                        const float cc[4] = {cv[c4].x, cv[c4].y, cv[c4].z, cv[c4].w};
#pragma unroll
                        for (int e = 0; e < 4; e += 2) {
                            const int col = c4 * 4 + e;
                            const float v0 = __uint_as_float(col < 32 ? r0[col & 31] : r1[col & 31]);
                            const float v1 = __uint_as_float(col < 32 ? r0[(col + 1) & 31] : r1[(col + 1) & 31]);
                            dp2s(v0, v1, cc[e], cc[e + 1], dv[col], dv[col + 1]);
                        }
                    }
                    float m21[22];
#pragma unroll
                    for (int i = 0; i < 21; i++) m21[i] = fmin3(dv[3 * i], dv[3 * i + 1], dv[3 * i + 2]);
                    m21[21] = dv[63];
                    float m8[8];
#pragma unroll
                    for (int i = 0; i < 7; i++) m8[i] = fmin3(m21[3 * i], m21[3 * i + 1], m21[3 * i + 2]);
                    m8[7] = m21[21];
                    const float mc = fmin3(fmin3(m8[0], m8[1], m8[2]), fmin3(m8[3], m8[4], m8[5]),
                                           fminf(m8[6], m8[7]));
                    // (as in k_assign_tgy: a chunk that does not beat the row's best
                    // only offers its minimum as a second best; the chunk's exact
                    // top-2, a merge tree, runs only under a new best)
                    if (!__any_sync(LK_FULL_MASK, mc < b1)) {
                        b2 = fminf(b2, mc);
                    } else {
                        float g1v[8], g2v[8];
#pragma unroll
                        for (int g8 = 0; g8 < 8; g8++) {
                            float lo[4], hi[4];
#pragma unroll
                            for (int pp = 0; pp < 4; pp++) {
                                lo[pp] = fminf(dv[8 * g8 + 2 * pp], dv[8 * g8 + 2 * pp + 1]);
                                hi[pp] = fmaxf(dv[8 * g8 + 2 * pp], dv[8 * g8 + 2 * pp + 1]);
                            }
                            const float l01 = fminf(lo[0], lo[1]), h01 = fmin3(fmaxf(lo[0], lo[1]), hi[0], hi[1]);
                            const float l23 = fminf(lo[2], lo[3]), h23 = fmin3(fmaxf(lo[2], lo[3]), hi[2], hi[3]);
                            g1v[g8] = fminf(l01, l23);
                            g2v[g8] = fmin3(fmaxf(l01, l23), h01, h23);
                        }
#pragma unroll
                        for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
                            for (int pp = 0; pp < w2; pp++) {
                                const float l = fminf(g1v[pp], g1v[pp + w2]);
                                g2v[pp] = fmin3(fmaxf(g1v[pp], g1v[pp + w2]), g2v[pp], g2v[pp + w2]);
                                g1v[pp] = l;
                            }
                        if (g1v[0] < b1) {
                            b2 = fminf(b1, g2v[0]);
                            b1 = g1v[0];
                        } else {
                            b2 = fminf(b2, g1v[0]);
                        }
                        const bool imp = b1 < bv;
                        if (__any_sync(LK_FULL_MASK, imp)) {
                            int found = -1;
#pragma unroll
                            for (int e = 63; e >= 0; e--)
                                if (dv[e] == b1) found = jb + e;
                            if (imp) {
                                bv = b1;
                                bj = found;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bempty);  // this warp is done with the pair's beta rows
            const int j1 = (bj >= 0 && bv == b1) ? col_id(S, bj) : -1;
            int64_t row = 0;
            bool moved = false, amb = false;
            int old = 0;
            float thr_out = 0.f, lb_out = 0.f;
            if (valid) tc_certify(S, A, kappa, r, b1, b2, j1, row, moved, old, amb, thr_out, lb_out);
            int64_t pos = epi_append8(moved, (unsigned long long*)(stat + LK_STAT_CHANGED), escr, warp);
            if (moved) S.moved[pos] = make_int2((int)row, old);
            int64_t cpos = epi_append8(amb, (unsigned long long*)(stat + LK_STAT_CANDIDATE), escr, warp);
            if (amb) {
                S.cand_rows[cpos] = (int)row;
                S.cand_thr[cpos] = thr_out;
                S.cand_lb[cpos] = lb_out;
            }
        }
    }
    __syncthreads();
    if (warp == MW) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

// ---- Yinyang on the tensor cores: block-sparse (row-tile pair x group tile) --
//
// Reference: Yinyang.assign_pass (pruners.py:438-497) -- the global gate, the
// per-group scans against the running best, the group-bound rewrite and the
// old-group fix-up -- for d <= 32 on the k_assign_tc2 pipeline.  The B operand
// holds the centroids in group order (column 128 g + member rank: group g is
// centroid tile g, S.colperm maps columns back to ids).  k_filter_tgy lists the
// rows whose bounds fail together with their failing groups plus the group of
// their label; the rows are label-sorted into 256-row pairs and a pair runs
// only the centroid tiles in the union of its rows' masks (pmask).
//
// The epilogue keeps each row's top-2 over the scanned tiles and every scanned
// tile's minimum.  A row is certified iff the winner's upper bound is below the
// second-best's lower bound AND below the lower bound of every unscanned group
// (rowlun); it then rewrites ub, the global bound and each scanned group's
// bound (lazy encoding).  Ambiguous rows take the collect pass
// over all k and the exact fp64 recheck, as on the full path.

// Certified lower bound (distance) on every column whose TC value D'~ >= v, for
// a centered row (R, |x'| = xo): the L2 expression of tc_certify evaluated at
// v, with the square root rounded down.
__device__ __forceinline__ float tgy_lower(double R, double xo, double kx_cmax, double gb, double cmax,
                                           float v) {
    if (isinf(v)) return INFINITY;
    const double av = fabs((double)v);
    const double eo = kx_cmax + gb * (av + 2.0 * xo * cmax) + 2.0 * 5.9604644775390625e-08 * av;
    const float sr = __fsqrt_ru(__double2float_ru(fmax(R + (double)v + eo, 0.0)));
    const double ex = 2.384185791015625e-07 * xo * ((double)sr + xo);
    const double L = (R + (double)v - eo - ex) - fabs(R) * 1e-12;
    return __fsqrt_rd(__double2float_rd(fmax(L, 0.0)));
}

// The same lower bound in fp32 with directed rounding (the per-group rewrite of
// k_assign_tgy: fp64 and its conversions dominated the pair's tail).  Every
// step rounds toward a smaller result: R_lo <= R, the error terms are rounded
// up, the sums / differences down, so the value never exceeds the fp64 form's
// exact counterpart; it is a little weaker (an fp32 rounding of R + v).
struct TgyLow {
    float R_lo, R_hi;   // R rounded down / up
    float xo;           // |x'| (already rounded up)
    float kxc;          // kappa |x'| cmax, rounded up
    float gbx;          // gb * 2 |x'| cmax, rounded up
    float gb;           // (d + 4) u
    float slack;        // |R| 1e-12 + 2^-126, rounded up
};

__device__ __forceinline__ TgyLow tgy_low_setup(double R, double xo, float kappa, float cmax, int d) {
    TgyLow t;
    t.R_lo = __double2float_rd(R);
    t.R_hi = __double2float_ru(R);
    t.xo = (float)xo;  // (xo holds an fp32 value)
    t.kxc = __fmul_ru(__fmul_ru(kappa, t.xo), cmax);
    t.gb = (float)(d + 4) * 5.9604644775390625e-08f;
    t.gbx = __fmul_ru(t.gb, __fmul_ru(__fmul_ru(2.0f, t.xo), cmax));
    t.slack = __fmaf_ru(fabsf(t.R_hi), 1e-12f, 1.2e-38f);
    return t;
}

// Square roots bounded from below / above, cheaper than the directed-rounding
// __fsqrt_rd / __fsqrt_ru sequences (and than sqrtf's Newton step and slow path).
// (sqrt.approx.f32: one MUFU op, relative error <= 2^-23 over the positive
// finite range, subnormals included; the bounds take 2^-21 of margin)
__device__ __forceinline__ float sqrt_mufu(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_lo(float x) {
    if (!(x > 0.f)) return 0.f;
    return __fmul_rd(sqrt_mufu(x), 1.0f - 4.76837158203125e-07f);  // (+inf stays +inf)
}
__device__ __forceinline__ float sqrt_hi(float x) {
    if (!(x > 0.f)) return 0.f;
    return __fmul_ru(sqrt_mufu(x), 1.0f + 4.76837158203125e-07f);
}

__device__ __forceinline__ float tgy_lower32(const TgyLow& t, float v) {
    if (isinf(v)) return INFINITY;
    const float av = fabsf(v);
    // eo = kappa |x'| cmax + gb (|v| + 2 |x'| cmax) + 2u |v|   (rounded up)
    const float eo = __fadd_ru(__fadd_ru(t.kxc, __fmaf_ru(t.gb, av, t.gbx)), __fmul_ru(1.1920928955078125e-07f, av));
    // ex = 2^-22 |x'| (sqrt(R + v + eo) + |x'|)                  (rounded up)
    const float sr = sqrt_hi(__fadd_ru(__fadd_ru(t.R_hi, v), eo));
    const float ex = __fmul_ru(__fmul_ru(2.384185791015625e-07f, t.xo), __fadd_ru(sr, t.xo));
    // L = R + v - eo - ex - slack                               (rounded down)
    const float L = __fsub_rd(__fsub_rd(__fsub_rd(__fadd_rd(t.R_lo, v), eo), ex), t.slack);
    return sqrt_lo(L);
}

// Shared memory of k_assign_tgy: the k_assign_tc2 stages and resident A (the
// tf32 hi / lo operands of the pair's two row tiles), a staging buffer for the
// next pair's centered rows (fp32, as the sort wrote them), a ring of per-tile
// beta slices (the two row tiles' 128 offsets of the staged centroid tile: the
// producer never waits for a whole pair's epilogue), the cumulative group
// drifts.
struct TgySmem {
    static constexpr int B_BYTES = 128 * KC * 4;
    static constexpr int STAGE_BYTES = 2 * B_BYTES;
    static constexpr int STAGES = 3;
    static constexpr int NBB = 4;                        // beta ring slots
    static constexpr int A_BYTES = BM * KC * 4;
    static constexpr int A_OFF = STAGES * STAGE_BYTES;
    static constexpr int XS_OFF = A_OFF + 4 * A_BYTES;   // staging: [row tile][128 rows] x' (fp32)
    static constexpr int BAR_OFF = XS_OFF + 2 * A_BYTES;
    static constexpr int RING_OFF = BAR_OFF + 256;
    static constexpr int DG_OFF = RING_OFF + NBB * 1024;
    static constexpr int TOTAL = DG_OFF + 32 * 4 + 1024; // (+ kpad * 4 at launch: the column norms)
};

// Phase clocks of k_assign_tgy (debug knob LK_TGY_PROF): cycles each role spends
// waiting on each barrier / computing, summed over lane 0 of the role warps.
enum TgyProf {
    TP_P_AEMPTY, TP_P_EMPTY, TP_P_REMPTY, TP_P_TOTAL, TP_M_AFULL, TP_M_TEMPTY, TP_M_FULL, TP_M_TOTAL,
    TP_E_TFULL, TP_E_RFULL, TP_E_TILES, TP_E_TAIL, TP_E_TOTAL, TP_PAIRS, TP_TILES,
    TP_T_CERT, TP_T_GROUPS, TP_T_STORES, TP_T_APPEND,
#ifdef LK_TGY_PROF_CHUNKS
    TP_C_LOAD, TP_C_FAST, TP_C_SLOW, TP_C_MINE, TP_C_SLOWN,
#endif
    TP_N
};
#define TGY_W(idx, call)                                        \
    do {                                                        \
        if (prof_on) {                                          \
            const long long t0_ = clock64();                    \
            call;                                               \
            pc[idx] += clock64() - t0_;                         \
        } else {                                                \
            call;                                               \
        }                                                       \
    } while (0)

// A pair's centroid tiles run starting from the group of its first row tile's
// label (then in increasing group order, wrapping): rows mostly belong to that
// group, so their running top-2 is tight after the first tile and the exact
// update of later chunks rarely triggers.  All three roles derive the same
// order from the same loads.
__device__ __forceinline__ int tgy_rot(const DevState& S, int64_t rt) {
    const int a = __ldg(S.tile_lab + rt);
    return a >= 0 ? __ldg(S.group_of + a) : 0;
}
__device__ __forceinline__ uint32_t rotr32(uint32_t m, int r) {
    return r ? (m >> r) | (m << (32 - r)) : m;
}

// One row tile of the pair's 3xTF32 split, staging -> A operands: hi =
// trunc_tf32(x'), lo = x' - hi (exact), elementwise (the 128B swizzle moves all
// three buffers alike).  Waits for the staged rows and for the previous pair's
// MMAs (the A operands are free), then arrives on sdone.
__device__ __forceinline__ void tgy_split_tile(const uint8_t* xs, uint8_t* abuf, int s_, uint64_t* sfull,
                                               uint64_t* aempty, uint64_t* sdone, int it, int lane) {
    constexpr int A_BYTES = TgySmem::A_BYTES;
    mbar_wait(sfull, it & 1);
    if (it > 0) mbar_wait(aempty, (it - 1) & 1);
    tc_fence_after();
    const float4* xp = reinterpret_cast<const float4*>(xs + s_ * A_BYTES);
    float4* hp = reinterpret_cast<float4*>(abuf + s_ * 2 * A_BYTES);
    float4* lp = reinterpret_cast<float4*>(abuf + s_ * 2 * A_BYTES + A_BYTES);
#pragma unroll 8
    for (int e = lane; e < A_BYTES / 16; e += 32) {
        const float4 x = xp[e];
        const float4 h = make_float4(tf32_trunc(x.x), tf32_trunc(x.y), tf32_trunc(x.z), tf32_trunc(x.w));
        hp[e] = h;
        lp[e] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
    }
    // generic-proxy writes -> visible to the tensor cores' async proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(sdone);
}

__global__ void __launch_bounds__(352, 1)
    k_assign_tgy(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                 const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                 DevState S, TcArgs A, int64_t* stat) {
    if (*S.done) return;
    using SM = TgySmem;
    constexpr int BN = 128, NBUF = 2, PW = 8, MW = 9, LW = 10, NBB = SM::NBB;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* abuf = smem + SM::A_OFF;
    uint64_t* full = (uint64_t*)(smem + SM::BAR_OFF);
    uint64_t* empty = full + SM::STAGES;
    uint64_t* tfull = empty + SM::STAGES;
    uint64_t* tempty = tfull + NBUF;
    uint64_t* sfull = tempty + NBUF;  // the next pair's x' staged (TMA)
    uint64_t* aempty = sfull + 1;     // the pair's MMAs are done (A operands free)
    uint64_t* sdone = aempty + 1;     // both row tiles split (staging free, A ready)
    uint64_t* rfull = sdone + 1;      // [NBB] beta slices staged
    uint64_t* rempty = rfull + NBB;   // [NBB] ... and released by the 8 epilogue warps
    uint32_t* tmem_slot = (uint32_t*)(rempty + NBB);
    float* ring = (float*)(smem + SM::RING_OFF);  // [NBB][2][128]
    float* sdg = (float*)(smem + SM::DG_OFF);     // [32] cumulative group drifts
    float* scn = sdg + 32;                        // [kpad] |c| of each B column (+inf padding)
    uint8_t* xs = smem + SM::XS_OFF;              // [2][A_BYTES] staged x'

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = S.t_groups;
    const int64_t m = *A.rowcount;
    const bool prof_on = A.prof != nullptr;
    long long pc[TP_N];
#ifdef LK_TGY_PROF_CHUNKS
    uint32_t pcc[5] = {0, 0, 0, 0, 0};  // chunk-level clocks of epilogue warp 0 (build-time probe)
#endif
#pragma unroll
    for (int e = 0; e < TP_N; e++) pc[e] = 0;
    const long long tk0 = prof_on ? clock64() : 0;
    const int64_t n_rt = (m + BM - 1) / BM;
    const int64_t n_rp = (n_rt + 1) / 2;
    auto beta_of = [&](int64_t t_) -> const float* {
        if (t_ >= n_rt) return S.cn2;
        const int at = S.tile_lab[t_];
        return at >= 0 ? S.ptab + (int64_t)at * S.kpad : S.cn2;
    };
    const int n_it = (int)(n_rp > (int64_t)blockIdx.x ? (n_rp - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < SM::STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NBUF; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);
        }
        for (int b = 0; b < NBB; b++) {
            mbar_init(&rfull[b], 1);
            mbar_init(&rempty[b], 8);
        }
        mbar_init(sfull, 1);
        mbar_init(aempty, 1);
        mbar_init(sdone, 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_map(&map_ahi);
        prefetch_map(&map_alo);
        prefetch_map(&map_bhi);
        prefetch_map(&map_blo);
    }
    if (threadIdx.x < 32) sdg[threadIdx.x] = threadIdx.x < G ? S.dgcum[threadIdx.x] : 0.f;
    for (int c = threadIdx.x; c < S.kpad; c += blockDim.x) {
        const int j = col_id(S, c);
        scn[c] = j >= 0 ? S.cnorm[j] : S.scal[0];
    }
    if (warp == MW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == PW) {
        // ===== TMA producer: per pair the A tiles (as soon as the previous
        // pair's MMAs are done), then per masked centroid tile its B operand
        // and the two row tiles' beta slices
        if (lane == 0) {
            int stage = 0, rs = 0;
            uint32_t phase = 0, rphase = 0;
            int4 pi_n = n_it > 0 ? __ldg(S.pinfo + blockIdx.x) : make_int4(0, 0, 0, 0);  // (one pair ahead)
            for (int it = 0; it < n_it; it++) {
                const int64_t rp = blockIdx.x + (int64_t)it * gridDim.x;
                const int4 pi = pi_n;
                if (it + 1 < n_it) pi_n = __ldg(S.pinfo + rp + gridDim.x);
                const uint32_t pm = (uint32_t)pi.x | (uint32_t)pi.y;
                const int l0 = (pi.w & 0xffff) - 1, l1 = ((unsigned)pi.w >> 16) - 1;
                const float* bt0 = l0 >= 0 ? S.ptab + (int64_t)l0 * S.kpad : S.cn2;
                const float* bt1 = l1 >= 0 ? S.ptab + (int64_t)l1 * S.kpad : S.cn2;
                const int g0 = pi.z & 31;
                for (uint32_t mm = rotr32(pm, g0); mm; mm &= mm - 1) {
                    const int ct = (__ffs(mm) - 1 + g0) & 31;
                    TGY_W(TP_P_EMPTY, mbar_wait(&empty[stage], phase ^ 1));
                    uint8_t* bst = smem + stage * SM::STAGE_BYTES;
                    mbar_expect_tx(&full[stage], SM::STAGE_BYTES);
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        uint8_t* dst = bst + (q >> 1) * SM::B_BYTES + (q & 1) * (SM::B_BYTES / 2);
                        tma_load_2d((q >> 1) ? &map_blo : &map_bhi, &full[stage], dst, 0,
                                    ct * BN + (q & 1) * (BN / 2));
                    }
                    if (++stage == SM::STAGES) { stage = 0; phase ^= 1; }
                    TGY_W(TP_P_REMPTY, mbar_wait(&rempty[rs], rphase ^ 1));
                    mbar_expect_tx(&rfull[rs], 1024);
                    bulk_load(ring + rs * 256, bt0 + ct * BN, 512, &rfull[rs]);
                    bulk_load(ring + rs * 256 + 128, bt1 + ct * BN, 512, &rfull[rs]);
                    if (++rs == NBB) { rs = 0; rphase ^= 1; }
                }
            }
        }
    } else if (warp == MW) {
        // ===== MMA issuer (ordered single accumulator, as k_assign_tc2) =====
        constexpr uint32_t idesc = idesc_tf32(BM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        int64_t n_dist = 0;
        int4 pi_n = n_it > 0 ? __ldg(S.pinfo + blockIdx.x) : make_int4(0, 0, 0, 0);  // (one pair ahead)
        for (int it = 0; it < n_it; it++) {
            const int64_t rp = blockIdx.x + (int64_t)it * gridDim.x;
            const int4 pi = pi_n;
            if (it + 1 < n_it) pi_n = __ldg(S.pinfo + rp + gridDim.x);
            // each row tile runs only the centroid tiles of its own mask
            const uint32_t m0 = (uint32_t)pi.x, m1 = (uint32_t)pi.y;
            const uint32_t pm = m0 | m1;
            const int64_t r0n = m - 2 * rp * BM < BM ? m - 2 * rp * BM : BM;
            const int64_t r1n = m - (2 * rp + 1) * BM < BM ? (m - (2 * rp + 1) * BM > 0 ? m - (2 * rp + 1) * BM : 0) : BM;
            n_dist += 128 * (r0n * __popc(m0) + r1n * __popc(m1));
            // row tile 1's split (the loader warp splits row tile 0), then both
            TGY_W(TP_M_AFULL, tgy_split_tile(xs, abuf, 1, sfull, aempty, sdone, it, lane));
            TGY_W(TP_M_AFULL, mbar_wait(sdone, it & 1));
            tc_fence_after();
            const int g0 = pi.z & 31;
            for (uint32_t mm = rotr32(pm, g0); mm; mm &= mm - 1) {
                TGY_W(TP_M_TEMPTY, mbar_wait(&tempty[acc], acc_phase ^ 1));
                tc_fence_after();
                TGY_W(TP_M_FULL, mbar_wait(&full[stage], phase));
                tc_fence_after();
                uint8_t* bst = smem + stage * SM::STAGE_BYTES;
                const uint64_t dbhi = umma_desc(bst);
                const uint64_t dblo = umma_desc(bst + SM::B_BYTES);
                const int ct = (__ffs(mm) - 1 + g0) & 31;
#pragma unroll
                for (int s = 0; s < 2; s++) {
                    if (!((((s ? m1 : m0)) >> ct) & 1u)) continue;  // (warp-uniform)
                    const uint32_t tmem_d = tmem_base + acc * 2 * BN + s * BN;
                    const uint64_t dahi = umma_desc(abuf + s * 2 * SM::A_BYTES);
                    const uint64_t dalo = umma_desc(abuf + s * 2 * SM::A_BYTES + SM::A_BYTES);
#pragma unroll
                    for (int k = 0; k < KC / UK; k++) {
                        const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                        mma_tf32(tmem_d, dalo + off, dbhi + off, idesc, k != 0);
                        mma_tf32(tmem_d, dahi + off, dblo + off, idesc, 1);
                    }
#pragma unroll
                    for (int k = 0; k < KC / UK; k++) {
                        const uint64_t off = (uint64_t)((k * UK * 4) >> 4);
                        mma_tf32(tmem_d, dahi + off, dbhi + off, idesc, 1);
                    }
                }
                mma_commit(&empty[stage]);
                if (++stage == SM::STAGES) { stage = 0; phase ^= 1; }
                mma_commit(&tfull[acc]);
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
            }
            mma_commit(aempty);
        }
        if (lane == 0 && n_dist) atomicAdd((unsigned long long*)(stat + LK_STAT_DIST), (unsigned long long)n_dist);
    } else if (warp == LW) {
        // ===== A loader: the next pair's centered rows x' (fp32) into the
        // staging buffer while the current pair runs; row tile 0's split.  The
        // split waits only for the previous pair's MMAs, not for an HBM load.
        if (n_it > 0 && lane == 0) {
            mbar_expect_tx(sfull, 2 * SM::A_BYTES);
            tma_load_2d(&map_ahi, sfull, xs, 0, (int)(2 * (int64_t)blockIdx.x * BM));
            tma_load_2d(&map_ahi, sfull, xs + SM::A_BYTES, 0, (int)((2 * (int64_t)blockIdx.x + 1) * BM));
        }
        for (int it = 0; it < n_it; it++) {
            tgy_split_tile(xs, abuf, 0, sfull, aempty, sdone, it, lane);
            mbar_wait(sdone, it & 1);  // (both halves read: the staging buffer is free)
            if (it + 1 < n_it && lane == 0) {
                const int64_t rp = blockIdx.x + (int64_t)(it + 1) * gridDim.x;
                mbar_expect_tx(sfull, 2 * SM::A_BYTES);
                tma_load_2d(&map_ahi, sfull, xs, 0, (int)(2 * rp * BM));
                tma_load_2d(&map_ahi, sfull, xs + SM::A_BYTES, 0, (int)((2 * rp + 1) * BM));
            }
            __syncwarp();
        }
    } else {
        // ===== epilogue: warp w = rows 32 (w % 4) .. of row tile w / 4 =====
        const int q = warp & 3, s = warp >> 2;
        const float kappa = tc_kappa_ordered(S.d);
        const float dm = S.scal[4];
        const float cmax_f = S.scal[0];
        int acc = 0, rs = 0;
        uint32_t acc_phase = 0, rphase = 0;
        const int rloc0 = s * BM + q * 32;   // this warp's first row in the pair
        const int rloc = rloc0 + lane;
        // the rows' certification records (and labels) are loaded one pair ahead
        int4 mw0 = make_int4(0, 0, 0, 0), mw1 = mw0;
        int old_n = 0;
        auto load_meta = [&](int it_) {
            const int64_t r_ = (2 * (blockIdx.x + (int64_t)it_ * gridDim.x) + s) * BM + q * 32 + lane;
            if (it_ < n_it && r_ < m) {
                const int4* src = reinterpret_cast<const int4*>(S.tmeta + r_);
                mw0 = __ldcs(src);
                mw1 = __ldcs(src + 1);
            }
        };
        load_meta(0);
        int4 pi_n = n_it > 0 ? __ldg(S.pinfo + blockIdx.x) : make_int4(0, 0, 0, 0);  // (one pair ahead)
        for (int it = 0; it < n_it; it++) {
            const int64_t rp = blockIdx.x + (int64_t)it * gridDim.x;
            const int4 pi = pi_n;
            if (it + 1 < n_it) pi_n = __ldg(S.pinfo + rp + gridDim.x);
            // the pair's tiles stream in for the union of the two row tiles'
            // masks; this row tile evaluates only its own (ms)
            const uint32_t ms = (uint32_t)(s ? pi.y : pi.x);
            const uint32_t pm = (uint32_t)pi.x | (uint32_t)pi.y;
            const int64_t rt = 2 * rp + s;
            const int64_t r = rt * BM + q * 32 + lane;
            const bool valid = r < m;
            float b1 = INFINITY, b2 = INFINITY, bv = INFINITY;
            int bj = -1;
            // the row's certification record, loaded while the tiles stream
            int64_t row = 0;
            double R = 0.0, xo = 0.0;
            float lun = 0.f, xn2 = 0.f;
            int old = 0;
            if (valid) {
                int4 w[2] = {mw0, mw1};
                const TgyMeta& t = *reinterpret_cast<const TgyMeta*>(w);
                row = t.row;
                R = t.R;
                xo = (double)t.xo;
                lun = t.lun;
                xn2 = t.xn2;
                bv = t.bv;
                old = S.labels[row];  // (used in the tail only)
            }
            load_meta(it + 1);
            // the fp32 lower-bound setup of the row (tgy_lower32): each scanned
            // group's bound is formed and stored as soon as its tile is done
            const TgyLow tl = tgy_low_setup(R, xo, kappa, cmax_f, S.d);
            float* lbr = S.lb + row * S.nlb;
            const int g0 = pi.z & 31;
            // the B column of this row tile's label: its 64-column chunk runs
            // first (it sets the rows' best, so the tile's other chunk seldom
            // needs the exact top-2)
            const int acol = (int)(((unsigned)pi.z >> (s ? 18 : 5)) & 0x1fffu) - 1;
            for (uint32_t mm = rotr32(pm, g0); mm; mm &= mm - 1) {
                const int ct = (__ffs(mm) - 1 + g0) & 31;
                TGY_W(TP_E_TFULL, mbar_wait(&tfull[acc], acc_phase));
                tc_fence_after();
                TGY_W(TP_E_RFULL, mbar_wait(&rfull[rs], rphase));
                const long long tt0 = prof_on ? clock64() : 0;
                pc[TP_TILES]++;
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 2 * BN + s * BN;
                const uint32_t sb0 = smem_u32(ring + rs * 256 + s * 128);
                float gmin = INFINITY;
                const bool mine = (ms >> ct) & 1u;  // (warp-uniform)
                const int cf = (acol >= 0 && (acol >> 7) == ct) ? (acol & 64) : 0;
#pragma unroll 1
                for (int ci = 0; ci < ((mine && A.dbg != 4) ? 2 : 0); ci++) {
                    const int c0 = ci == 0 ? cf : 64 - cf;
                    uint32_t r0[32], r1[32];
#ifdef LK_TGY_PROF_CHUNKS
                    const long long tc0 = prof_on ? clock64() : 0;
#endif
                    tmem_ld32_async(taddr + c0, r0);
                    tmem_ld32_async(taddr + c0 + 32, r1);
                    const int jb = ct * BN + c0;
                    const uint32_t sb = sb0 + 4 * c0;
                    float4 cv[16];
#pragma unroll
                    for (int c4 = 0; c4 < 16; c4++)
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(cv[c4].x), "=f"(cv[c4].y), "=f"(cv[c4].z), "=f"(cv[c4].w)
                                     : "r"(sb + 16 * c4));
                    tmem_wait_ld();
#ifdef LK_TGY_PROF_CHUNKS
                    const long long tc1 = prof_on ? clock64() : 0;
#endif
                    float dv[64];
#pragma unroll
                    for (int c4 = 0; c4 < 16; c4++) {
                        const float cc[4] = {cv[c4].x, cv[c4].y, cv[c4].z, cv[c4].w};
#pragma unroll
                        for (int e = 0; e < 4; e += 2) {
                            const int col = c4 * 4 + e;
                            const float v0 = __uint_as_float(col < 32 ? r0[col & 31] : r1[col & 31]);
                            const float v1 = __uint_as_float(col < 32 ? r0[(col + 1) & 31] : r1[(col + 1) & 31]);
                            dp2s(v0, v1, cc[e], cc[e + 1], dv[col], dv[col + 1]);
                        }
                    }
                    float m21[22];
#pragma unroll
                    for (int i = 0; i < 21; i++) m21[i] = fmin3(dv[3 * i], dv[3 * i + 1], dv[3 * i + 2]);
                    m21[21] = dv[63];
                    float m8[8];
#pragma unroll
                    for (int i = 0; i < 7; i++) m8[i] = fmin3(m21[3 * i], m21[3 * i + 1], m21[3 * i + 2]);
                    m8[7] = m21[21];
                    const float mc = fmin3(fmin3(m8[0], m8[1], m8[2]), fmin3(m8[3], m8[4], m8[5]),
                                           fminf(m8[6], m8[7]));
                    gmin = fminf(gmin, mc);
                    // A chunk whose minimum does not beat the row's best only
                    // offers that minimum as a second best; the chunk's own
                    // second smallest value matters only under a new best
                    // (the first tile of a row, and rows about to move), so the
                    // exact top-2 of the chunk -- a merge tree, no serial chain
                    // -- runs only when some row of the warp has one.
#ifdef LK_TGY_PROF_CHUNKS
                    const long long tc2 = prof_on ? clock64() : 0;
                    if (prof_on) {
                        pcc[0] += (uint32_t)(tc1 - tc0);
                        pcc[1] += (uint32_t)(tc2 - tc1);
                        pcc[3]++;
                    }
#endif
                    if (A.dbg == 1 || !__any_sync(LK_FULL_MASK, mc < b1)) {
                        b2 = fminf(b2, mc);
                    } else {
#ifdef LK_TGY_PROF_CHUNKS
                        pcc[4]++;
#endif
                        float g1v[8], g2v[8];
#pragma unroll
                        for (int g8 = 0; g8 < 8; g8++) {
                            float lo[4], hi[4];
#pragma unroll
                            for (int pp = 0; pp < 4; pp++) {
                                lo[pp] = fminf(dv[8 * g8 + 2 * pp], dv[8 * g8 + 2 * pp + 1]);
                                hi[pp] = fmaxf(dv[8 * g8 + 2 * pp], dv[8 * g8 + 2 * pp + 1]);
                            }
                            const float l01 = fminf(lo[0], lo[1]), h01 = fmin3(fmaxf(lo[0], lo[1]), hi[0], hi[1]);
                            const float l23 = fminf(lo[2], lo[3]), h23 = fmin3(fmaxf(lo[2], lo[3]), hi[2], hi[3]);
                            g1v[g8] = fminf(l01, l23);
                            g2v[g8] = fmin3(fmaxf(l01, l23), h01, h23);
                        }
#pragma unroll
                        for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
                            for (int pp = 0; pp < w2; pp++) {
                                const float l = fminf(g1v[pp], g1v[pp + w2]);
                                g2v[pp] = fmin3(fmaxf(g1v[pp], g1v[pp + w2]), g2v[pp], g2v[pp + w2]);
                                g1v[pp] = l;
                            }
                        // (g1v[0] == mc; g2v[0] the chunk's second smallest)
                        if (g1v[0] < b1) {
                            b2 = fminf(b1, g2v[0]);
                            b1 = g1v[0];
                        } else {
                            b2 = fminf(b2, g1v[0]);
                        }
                        const bool imp = b1 < bv;
                        if (__any_sync(LK_FULL_MASK, imp)) {
                            int found = -1;
#pragma unroll
                            for (int e = 63; e >= 0; e--)
                                if (dv[e] == b1) found = jb + e;
                            if (imp) {
                                bv = b1;
                                bj = found;
                            }
                        }
                    }
#ifdef LK_TGY_PROF_CHUNKS
                    if (prof_on) pcc[2] += (uint32_t)(clock64() - tc2);
#endif
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&tempty[acc]);
                    mbar_arrive(&rempty[rs]);
                }
                // the group's bound (lazy encoding) from its minimum D'~: it bounds
                // all its members, whichever wins (the winner's group is rewritten
                // from the second best in the tail when the row is certified).
                // Every group of the row tile's mask is rewritten, not only the
                // row's own failing groups (measured: the tile's other groups then
                // keep older, weaker bounds and fail later -- 1.3e10 -> 1.75e10
                // products at cfg5 iteration 20).
                if (mine && valid && A.dbg != 2) __stcg(lbr + ct, __fadd_rd(tgy_lower32(tl, gmin), sdg[ct]));
                if (++acc == NBUF) { acc = 0; acc_phase ^= 1; }
                if (++rs == NBB) { rs = 0; rphase ^= 1; }
                if (prof_on) pc[TP_E_TILES] += clock64() - tt0;
            }
            const long long tl0 = prof_on ? clock64() : 0;
            pc[TP_PAIRS]++;
            if (A.dbg == 3) continue;  // (timing probe: no pair tail)
            // the winning column (searched and holding the minimum), its centroid
            // id and cumulative drift: both loads go out before the math
            const int jc = (bj >= 0 && bv == b1) ? bj : -1;
            const int j1 = jc >= 0 ? col_id(S, jc) : -1;
            const float dcj = jc >= 0 ? __ldg(S.dcum_col + jc) : 0.f;
            bool moved = false, amb = false, cert = false;
            float thr_out = 0.f, lb_out = 0.f;
            float L2d = 0.f, Ud = 0.f;
            int g1 = -1;
            if (valid) {
                // certification in fp32 with directed rounding (tgy_lower32's scheme:
                // upper bounds rounded up, lower bounds down; R split into R_lo / R_hi)
                const float cn1 = jc >= 0 ? scn[jc] : cmax_f;  // (|c| of the winner's column)
                const float ab1 = fabsf(b1);
                // e1 = kappa |x'| |c1| + gb (|b1| + 2 |x'| |c1|) + 2u |b1|        (up)
                const float xc1 = __fmul_ru(tl.xo, cn1);
                const float e1 = __fadd_ru(__fadd_ru(__fmul_ru(kappa, xc1),
                                                     __fmul_ru(tl.gb, __fmaf_ru(2.0f, xc1, ab1))),
                                           __fmul_ru(1.1920928955078125e-07f, ab1));
                const float sr1 = sqrt_hi(__fadd_ru(__fadd_ru(tl.R_hi, b1), e1));
                const float ex1 = __fmul_ru(__fmul_ru(2.384185791015625e-07f, tl.xo), __fadd_ru(sr1, tl.xo));
                // U >= (R + b1 + e1 + ex1): the squared distance of the best column, from above
                const float U = __fadd_ru(__fadd_ru(__fadd_ru(__fadd_ru(tl.R_hi, b1), e1), ex1), tl.slack);
                Ud = sqrt_hi(U);
                L2d = tgy_lower32(tl, b2);
                // the winner beats every other scanned column and every unscanned group
                cert = jc >= 0 && L2d > Ud && lun > Ud && !isinf(b1);
                // (the winner's group is its tile: B columns are in group order)
                g1 = cert ? (jc >> 7) : -1;
                if (cert) {
                    moved = old != j1;
                } else {
                    amb = true;
                    // thresholds of the (uncentered) collect pass: every possible winner
                    // has D'unc <= U - |x|^2 + e_unc (tc_certify's bound, rounded up)
                    const float xn = __fmul_ru(sqrtf(xn2), 1.0f + 4 * kU32);
                    const float eunc = __fadd_ru(__fmul_ru(__fmul_ru(kappa, xn), cmax_f),
                                                 __fmul_ru(8.0f * kU32, __fmaf_ru(cmax_f, cmax_f, xn2)));
                    const float thr = __fadd_ru(__fadd_ru(U, -__fmul_rd(xn2, 1.0f - 2.384185791015625e-07f)), eunc);
                    thr_out = __fadd_ru(__fmaf_ru(fabsf(thr), 1e-9f, thr), 1e-30f);
                    lb_out = sqrt_lo(U);
                }
            }
            if (prof_on) pc[TP_T_CERT] += clock64() - tl0;
            // list slots: one atomic per warp and list (no barrier across the
            // epilogue warps), issued before the group-bound work so that their
            // round trips overlap it
            const unsigned mmv = __ballot_sync(LK_FULL_MASK, moved);
            const unsigned mam = __ballot_sync(LK_FULL_MASK, amb);
            unsigned long long bmv = 0, bam = 0;
            if (lane == 0) {
                if (mmv) bmv = atomicAdd((unsigned long long*)(stat + LK_STAT_CHANGED), (unsigned long long)__popc(mmv));
                if (mam) bam = atomicAdd((unsigned long long*)(stat + LK_STAT_CANDIDATE), (unsigned long long)__popc(mam));
            }
            if (valid) {
                if (cert) {
                    // the winner's group: the second best bounds its other members
                    __stcg(lbr + g1, __fadd_rd(L2d, sdg[g1]));
                    if (moved) S.labels[row] = j1;
                    S.ub[row] = __fsub_ru(Ud, dcj);
                    S.glb[row] = __fadd_rd(fminf(L2d, lun), dm);
                }
            }
            if (prof_on) {
                pc[TP_T_GROUPS] += clock64() - tl0;
                pc[TP_T_STORES] += clock64() - tl0;
            }
            bmv = __shfl_sync(LK_FULL_MASK, bmv, 0);
            bam = __shfl_sync(LK_FULL_MASK, bam, 0);
            if (moved) S.moved[bmv + __popc(mmv & lanemask_lt())] = make_int2((int)row, old);
            if (amb) {
                const int64_t cpos = (int64_t)(bam + __popc(mam & lanemask_lt()));
                S.cand_rows[cpos] = (int)row;
                S.cand_thr[cpos] = thr_out;
                S.cand_lb[cpos] = lb_out;
            }
            if (prof_on) {
                pc[TP_E_TAIL] += clock64() - tl0;
                pc[TP_T_APPEND] += clock64() - tl0;
            }
        }
    }
    if (prof_on && lane == 0 && (warp == PW || warp == MW || warp == 0)) {
        const long long tot = clock64() - tk0;
        if (warp == PW) pc[TP_P_TOTAL] = tot;
        if (warp == MW) pc[TP_M_TOTAL] = tot;
        if (warp == 0) pc[TP_E_TOTAL] = tot;
#ifdef LK_TGY_PROF_CHUNKS
        if (warp == 0)
            for (int e = 0; e < 5; e++) pc[TP_C_LOAD + e] = pcc[e];
#endif
        for (int e = 0; e < TP_N; e++)
            if (pc[e]) atomicAdd(A.prof + e, (unsigned long long)pc[e]);
    }
    __syncthreads();
    if (warp == MW) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

// Union of the group masks of each 128-row tile of the sorted worklist (one
// warp per tile; 0 past the last tile).
__global__ void k_pair_mask(DevState S, const int64_t* count, int freq) {
    if (*S.done) return;
    const int64_t m = *count;
    const int64_t nt = (m + 127) / 128 + 1;
    const int lane = threadIdx.x & 31;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < nt;
         p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t v = 0, ve[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int64_t pos = p * 128 + e * 32 + lane;
            ve[e] = pos < m ? __ldcs(&S.tmeta[pos].mask) : 0u;
            v |= ve[e];
        }
        const uint32_t any = __reduce_or_sync(LK_FULL_MASK, v);
        if (lane == 0) S.pmask[p] = any;
        if (freq && any) {
            // how many of the tile's rows scan each group, added to the tile
            // label's frequencies (lane g owns group g)
            const int lab = __ldg(S.tile_lab + p);
            int mine = 0;
            for (uint32_t mm = any; mm; mm &= mm - 1) {
                const int g = __ffs(mm) - 1;
                int c = 0;
#pragma unroll
                for (int e = 0; e < 4; e++) c += __popc(__ballot_sync(LK_FULL_MASK, (ve[e] >> g) & 1));
                if (lane == g) mine = c;
            }
            if (lab >= 0 && mine > 0) atomicAdd(S.gfreq + (int64_t)lab * 32 + lane, mine);
        }
    }
}

// Per row-tile pair of the sorted worklist, everything the pass's three roles
// derive from the pair's tile labels and masks, in one 16-byte record (no
// dependent loads at the start of a pair): x / y the two row tiles' masks,
// z = group of the first tile's label | (B column of tile 0's label + 1) << 5
// | (of tile 1's + 1) << 18, w = (label 0 + 1) | (label 1 + 1) << 16.
__global__ void k_pair_info(DevState S, const int64_t* count) {
    if (*S.done) return;
    const int64_t m = *count;
    const int64_t nt = (m + 127) / 128, np = (nt + 1) / 2;
    for (int64_t rp = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; rp <= np;
         rp += (int64_t)gridDim.x * blockDim.x) {
        int4 v = make_int4(0, 0, 0, 0);
        if (rp < np) {
            const int l0 = 2 * rp < nt ? S.tile_lab[2 * rp] : -1;
            const int l1 = 2 * rp + 1 < nt ? S.tile_lab[2 * rp + 1] : -1;
            v.x = (int)S.pmask[2 * rp];
            v.y = 2 * rp + 1 < nt ? (int)S.pmask[2 * rp + 1] : 0;
            const int g0 = l0 >= 0 ? S.group_of[l0] : 0;
            const int a0 = l0 >= 0 ? S.ginv[l0] : -1, a1 = l1 >= 0 ? S.ginv[l1] : -1;
            v.z = g0 | ((a0 + 1) << 5) | ((a1 + 1) << 18);
            v.w = (l0 + 1) | ((l1 + 1) << 16);
        }
        S.pinfo[rp] = v;
    }
}

// ---- prep kernels -----------------------------------------------------------

// x_lo = x - trunc_tf32(x) (exact in fp32) and ||x||^2 (fp64, rounded to fp32).
__global__ void k_split_points(DevState S) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < S.n; i += nwarps) {
        double s = 0.0;
        for (int z = lane; z < S.ldx; z += 32) {
            float x = z < S.d ? S.X32[i * S.ldx + z] : 0.f;
            float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
            S.Xlo[i * S.ldx + z] = x - hi;
            double xv = S.X64 && z < S.d ? S.X64[i * S.d + z] : (double)x;
            s = fma(xv, xv, s);
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(LK_FULL_MASK, s, o);
        if (lane == 0) S.xn2[i] = (float)s;
    }
}

// Gather worklist rows into the contiguous rescan buffers (hi = x, lo = split).
__global__ void k_gather_rows(DevState S, const int32_t* rows, const int64_t* count,
                              int64_t dense_thr = -1) {
    // rows: worklist of global row ids; count: device length; dense_thr >= 0:
    // nothing to gather when the list is long (the dense pass runs instead)
    if (*S.done) return;
    const int64_t m = *count;
    if (dense_thr >= 0 && m > dense_thr) return;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < m; r += nwarps) {
        const int64_t row = rows[r];
        for (int z = lane * 4; z < S.ldx; z += 128) {
            float4 h = *reinterpret_cast<const float4*>(S.X32 + row * S.ldx + z);
            float4 l = *reinterpret_cast<const float4*>(S.Xlo + row * S.ldx + z);
            *reinterpret_cast<float4*>(S.Xg_hi + r * S.ldx + z) = h;
            *reinterpret_cast<float4*>(S.Xg_lo + r * S.ldx + z) = l;
        }
    }
}

// ---- tile centering -----------------------------------------------------------
//
// The dot-form error scales with |x| |c|.  Rows sorted by label
// make a 128-row tile (mostly) one cluster; shifting the tile by the centroid
// o = c_a of its first row's label gives
//     ||x - c_j||^2 = R(x') + beta_j - 2 x'.c_j,   x' = x - o,
//     R(x') = ||x'||^2 + 2 x'.o,   beta_j = ||c_j - o||^2 = ptab[a][j],
// so the contraction runs on x' (small) against the unshifted centroids (the
// B operand stays shared by every tile) and the error scales with |x'| |c|.

// ptab[a][j] = sum_z (c_a,z - c_j,z)^2 in fp32 difference form (fmaf chain in
// dimension order), +inf for padding columns j >= k.  T x T tiles, 16 x 16
// threads, (T/16)^2 pairs per thread: T = 64 for many centroids, T = 16 when
// the 64-tiles would not fill the SMs (few centroids, long rows: cfg4).
template <int T>
__global__ void __launch_bounds__(256) k_pair_table(DevState S) {
    if (*S.done) return;
    constexpr int P = T / 16;
    __shared__ float ta[32][T + 1];
    __shared__ float tb[32][T + 1];
    const int a0 = blockIdx.y * T, j0 = blockIdx.x * T;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[P][P];
#pragma unroll
    for (int u = 0; u < P; u++)
#pragma unroll
        for (int v = 0; v < P; v++) acc[u][v] = 0.f;
    for (int z0 = 0; z0 < S.d; z0 += 32) {
        __syncthreads();
        for (int e = threadIdx.x; e < T * 32; e += 256) {
            const int r = e / 32, z = e % 32, zz = z0 + z;
            ta[z][r] = (a0 + r < S.k && zz < S.d) ? S.C32[(int64_t)(a0 + r) * S.ldc + zz] : 0.f;
            const int jb = col_id(S, j0 + r);
            tb[z][r] = (jb >= 0 && zz < S.d) ? S.C32[(int64_t)jb * S.ldc + zz] : 0.f;
        }
        __syncthreads();
        const int zn = min(32, S.d - z0);
        for (int z = 0; z < zn; z++) {
#pragma unroll
            for (int u = 0; u < P; u++)
#pragma unroll
                for (int v = 0; v < P; v++) {
                    const float t = ta[z][ty + 16 * u] - tb[z][tx + 16 * v];
                    acc[u][v] = fmaf(t, t, acc[u][v]);
                }
        }
    }
#pragma unroll
    for (int u = 0; u < P; u++) {
        const int a = a0 + ty + 16 * u;
        if (a >= S.k) continue;
#pragma unroll
        for (int v = 0; v < P; v++) {
            const int j = j0 + tx + 16 * v;
            if (j < S.kpad) S.ptab[(int64_t)a * S.kpad + j] = col_id(S, j) >= 0 ? acc[u][v] : INFINITY;
        }
    }
}

// Per-label histogram of a row list (rowlist == nullptr: the label counts of
// the last refinement are used instead).
// Sort key of a label: the label itself, or on the group-tile path its B
// column (labels of one group adjacent, so a pair spanning several labels
// mostly stays inside one group tile).
__device__ __forceinline__ int sort_key(const DevState& S, int lab) {
    return S.colperm ? __ldg(S.ginv + lab) : lab;
}

__global__ void k_label_count(DevState S, const int32_t* rowlist, const int64_t* count) {
    if (*S.done) return;
    const int64_t m = count ? *count : S.n;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(S.lcur + sort_key(S, S.labels[rowlist ? rowlist[p] : p]), 1);
}

// lcur := exclusive prefix of the histogram (from lcur, or from S.counts).
__global__ void __launch_bounds__(1024) k_label_scan(DevState S, int from_counts) {
    if (*S.done) return;
    __shared__ int part[1024];
    const int k = from_counts ? S.k : S.kcols, per = (k + 1023) / 1024;
    const int b = threadIdx.x * per;
    int sum = 0;
    for (int j = b; j < b + per && j < k; j++) sum += from_counts ? (int)S.counts[j] : S.lcur[j];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = part[threadIdx.x] - sum;
    for (int j = b; j < b + per && j < k; j++) {
        const int c = from_counts ? (int)S.counts[j] : S.lcur[j];
        S.lcur[j] = run;
        run += c;
    }
}

// perm[cursor[label]++] = row (order inside a label is arbitrary: labels are
// certified per row, independent of the tiling).
__global__ void k_label_scatter(DevState S, const int32_t* rowlist, const int64_t* count) {
    if (*S.done) return;
    const int64_t m = count ? *count : S.n;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int row = rowlist ? rowlist[p] : (int)p;
        const int lab = S.labels[row];
        const int pos = atomicAdd(S.lcur + sort_key(S, lab), 1);
        S.perm[pos] = row;
        // per sorted position: the row's label, and each tile's (first row's) label
        S.rowlab[pos] = lab;
        if ((pos & 127) == 0) S.tile_lab[pos >> 7] = lab;
    }
}

// Group-tile worklist sort (counting sort by B column of the label, no global
// atomics on the hot keys): each of nb blocks histograms a contiguous chunk of
// the worklist in shared memory, k_sort_offsets turns the [nb, keys] counts
// into per-(block, key) bases, k_sort_scatter places the rows with shared-
// memory cursors.  The order inside a key is arbitrary (labels are certified
// per row, independent of the tiling).
__device__ __forceinline__ void sort_chunk(int64_t m, int nb, int b, int64_t& p0, int64_t& p1) {
    const int64_t per = (m + nb - 1) / nb;
    p0 = (int64_t)b * per;
    p1 = p0 + per < m ? p0 + per : m;
}

// ---- second sort key: the groups a row scans --------------------------------
// A 128-row tile runs the union of its rows' group masks, and rows of one label
// fail different neighbour groups: in label order alone the pass evaluated
// ~1.7x the products of the rows' own masks (cfg5).  So the worklist is first
// partitioned by a bucket key -- the row's mask bits at up to kSelBits groups
// chosen per label (S.gsel: the groups whose separation saves the most tile
// scans, from the previous iteration's per-label frequencies S.gfreq) -- and
// the label sort, which keeps the block order inside a label, then leaves a
// label's rows ordered by bucket (an LSD radix sort with the label as the
// last digit; a block's chunk lies in one bucket but for the ~64 boundaries).
constexpr int kSelBits = 6;
constexpr int kBuckets = 1 << kSelBits;

__device__ __forceinline__ int bucket_key(uint32_t mask, uint32_t sel) {
    int key = 0;
    while (sel) {
        const int b = __ffs(sel) - 1;
        key = (key << 1) | ((mask >> b) & 1);
        sel &= sel - 1;
    }
    return key;
}

// counts `key` over the warp's active lanes with one shared-memory atomic per
// distinct key; returns the lane's slot (base from the atomic + rank)
__device__ __forceinline__ int warp_key_add(int* sh, int key, bool ok) {
    // (whole-warp call; lanes without a row share the key -1 and add nothing)
    const unsigned peers = __match_any_sync(LK_FULL_MASK, ok ? key : -1);
    const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
    int base = 0;
    if (ok && lane == leader) base = atomicAdd(sh + key, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    return base + __popc(peers & lanemask_lt());
}

__global__ void __launch_bounds__(256) k_bucket_hist(DevState S, const int64_t* count) {
    if (*S.done) return;
    __shared__ int sh[kBuckets];
    if (threadIdx.x < kBuckets) sh[threadIdx.x] = 0;
    __syncthreads();
    int64_t p0, p1;
    sort_chunk(*count, gridDim.x, blockIdx.x, p0, p1);
    for (int64_t b = p0; b < p1; b += blockDim.x) {
        const int64_t p = b + threadIdx.x;
        const bool ok = p < p1;
        int key = 0;
        if (ok) {
            const int lab = __float_as_int(__ldg(&S.ylun[p].y));
            key = bucket_key(__ldg(S.ymask + p), __ldg(S.gsel + lab));
        }
        warp_key_add(sh, key, ok);
    }
    __syncthreads();
    if (threadIdx.x < kBuckets) S.bhist[blockIdx.x * kBuckets + threadIdx.x] = sh[threadIdx.x];
}

// per bucket: exclusive prefix over the blocks (in place), then the bucket bases
__global__ void __launch_bounds__(1024) k_bucket_offsets(DevState S, int nb) {
    if (*S.done) return;
    __shared__ int tot[kBuckets];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < kBuckets; j += 32) {
        int run = 0;
        for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            const int v = b < nb ? S.bhist[b * kBuckets + j] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(LK_FULL_MASK, incl, o);
                if (lane >= o) incl += u;
            }
            if (b < nb) S.bhist[b * kBuckets + j] = run + incl - v;
            run += __shfl_sync(LK_FULL_MASK, incl, 31);
        }
        if (lane == 0) tot[j] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int j = 0; j < kBuckets; j++) {
            S.bbase[j] = run;
            run += tot[j];
        }
    }
}

__global__ void __launch_bounds__(256) k_bucket_scatter(DevState S, const int64_t* count) {
    if (*S.done) return;
    __shared__ int sh[kBuckets];
    if (threadIdx.x < kBuckets)
        sh[threadIdx.x] = S.bbase[threadIdx.x] + S.bhist[blockIdx.x * kBuckets + threadIdx.x];
    __syncthreads();
    int64_t p0, p1;
    sort_chunk(*count, gridDim.x, blockIdx.x, p0, p1);
    for (int64_t b = p0; b < p1; b += blockDim.x) {
        const int64_t p = b + threadIdx.x;
        const bool ok = p < p1;
        float2 yl = make_float2(0.f, 0.f);
        uint32_t mask = 0;
        int row = 0, key = 0;
        if (ok) {
            yl = __ldcs(S.ylun + p);
            mask = __ldcs(S.ymask + p);
            row = __ldcs(S.work + p);
            key = bucket_key(mask, __ldg(S.gsel + __float_as_int(yl.y)));
        }
        const int pos = warp_key_add(sh, key, ok);
        if (ok) {
            S.work2[pos] = row;
            S.ymask2[pos] = mask;
            S.ylun2[pos] = yl;
        }
    }
}

// A label's bucket key for the next iteration, from this iteration's listing:
// with p the share of the label's listed rows that scan group g, a tile of 128
// of them scans g with probability 1 - (1 - p)^128 when the rows are mixed and
// p when they are separated; the kSelBits groups with the largest difference
// are selected.  Clears the label's frequencies.
__global__ void k_pick_sel(DevState S) {
    if (*S.done) return;
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= S.k) return;
    const int G = S.t_groups, own = S.group_of[l];
    int* f = S.gfreq + (int64_t)l * 32;
    const float cnt = (float)f[own];
    float sc[32];
#pragma unroll
    for (int g = 0; g < 32; g++) {
        float v = -1.f;
        if (g < G && g != own && cnt > 0.f) {
            const float p = fminf((float)f[g] / cnt, 1.f);
            v = 1.f - __expf(128.f * log1pf(-fminf(p, 0.999999f))) - p;
        }
        sc[g] = v;
        if (g < G) f[g] = 0;
    }
    uint32_t sel = 0;
    for (int r = 0; r < kSelBits; r++) {
        float best = 0.02f;  // (a group nearly every / hardly any row scans is not worth a bit)
        int bg = -1;
#pragma unroll
        for (int g = 0; g < 32; g++)
            if (sc[g] > best) {
                best = sc[g];
                bg = g;
            }
        if (bg < 0) break;
        sel |= 1u << bg;
#pragma unroll
        for (int g = 0; g < 32; g++)
            if (g == bg) sc[g] = -1.f;
    }
    S.gsel[l] = sel;
}

__global__ void __launch_bounds__(256) k_sort_hist(DevState S, const int64_t* count, int* hist,
                                                   const float2* __restrict__ wlun) {
    if (*S.done) return;
    extern __shared__ int sh[];
    const int keys = S.kcols;
    for (int j = threadIdx.x; j < keys; j += blockDim.x) sh[j] = 0;
    __syncthreads();
    int64_t p0, p1;
    sort_chunk(*count, gridDim.x, blockIdx.x, p0, p1);
    for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x)
        atomicAdd(sh + sort_key(S, __float_as_int(__ldcs(&wlun[p].y))), 1);
    __syncthreads();
    int* h = hist + (int64_t)blockIdx.x * keys;
    for (int j = threadIdx.x; j < keys; j += blockDim.x) h[j] = sh[j];
}

// per key: exclusive prefix over the blocks (in place) and the key total (lcur)
__global__ void k_sort_offsets(DevState S, int* hist, int nb) {
    if (*S.done) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S.kcols) return;
    int run = 0;
    for (int b = 0; b < nb; b++) {
        const int v = hist[(int64_t)b * S.kcols + j];
        hist[(int64_t)b * S.kcols + j] = run;
        run += v;
    }
    S.lcur[j] = run;
}

// The label each 128-position tile is centered on: the label of its first
// position (the key whose [base, next base) range holds it).
__global__ void k_tile_labels(DevState S, const int64_t* count) {
    if (*S.done) return;
    const int64_t m = *count;
    const int64_t nt = (m + 127) / 128;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int p = (int)(t * 128);
        int lo = 0, hi = S.kcols;  // first key whose base exceeds p
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(S.lcur + mid) > p) hi = mid;
            else lo = mid + 1;
        }
        S.tile_lab[t] = col_id(S, lo - 1);
    }
}

// Sort and gather in one pass: each worklist row is placed at its sorted
// position by a shared-memory cursor (per-block bases from k_sort_offsets)
// and written there centered on its tile's centroid (x' in fp32, one full
// 128-byte line: the pass splits it for 3xTF32 in shared memory), with its
// certification record (one 32-byte sector).
// Two phases per 1024-row slice of the block's chunk, so that many rows'
// dependent loads are in flight at once:
//   A  a thread per row (4 rows each, loads interleaved): worklist entry ->
//      label -> sort key -> cursor (shared-memory atomic) -> tile label;
//      (row, position, tile label, label, mask, bound) into shared memory
//   B  8 lanes per row (one float4 column each), 4 rows per lane group in
//      flight: the point and its tile centroid, centered split, hi/lo rows,
//      the norms and the record.
constexpr int kSortSlice = 1024;

struct SortStage {
    int row[kSortSlice];
    int pos[kSortSlice];
    int a[kSortSlice];
    int lab[kSortSlice];
    uint32_t mask[kSortSlice];
    float lun[kSortSlice];
};

__global__ void __launch_bounds__(256, 4) k_sort_gather(DevState S, const int64_t* count, const int* hist,
                                                     const int32_t* __restrict__ wrow,
                                                     const uint32_t* __restrict__ wmask,
                                                     const float2* __restrict__ wlun) {
    if (*S.done) return;
    extern __shared__ int sh[];
    __shared__ SortStage st;
    const int keys = S.kcols;
    const int* h = hist + (int64_t)blockIdx.x * keys;
    for (int j = threadIdx.x; j < keys; j += blockDim.x) sh[j] = __ldg(S.lcur + j) + h[j];
    __syncthreads();
    int64_t p0, p1;
    sort_chunk(*count, gridDim.x, blockIdx.x, p0, p1);
    constexpr int L = 8, RPT = kSortSlice / 256;
    const int sub = threadIdx.x & (L - 1), grp = threadIdx.x / L;  // 32 lane groups
    const int c4n = S.ldx / 4;
    const float kap = tc_kappa_ordered(S.d);
    for (int64_t base = p0; base < p1; base += kSortSlice) {
        const int nrow = (int)(p1 - base < kSortSlice ? p1 - base : kSortSlice);
        // ---- A: positions
        int rw[RPT], lb[RPT];
        float ln[RPT];
#pragma unroll
        for (int u = 0; u < RPT; u++) {
            const int e = threadIdx.x + u * 256;
            rw[u] = e < nrow ? __ldcs(wrow + base + e) : 0;
            const float2 yl = e < nrow ? __ldcs(wlun + base + e) : make_float2(0.f, 0.f);
            ln[u] = yl.x;
            lb[u] = __float_as_int(yl.y);  // the row's label (written by the filter)
        }
#pragma unroll
        for (int u = 0; u < RPT; u++) {
            const int e = threadIdx.x + u * 256;
            if (e < nrow) {
                const int pos = atomicAdd(sh + sort_key(S, lb[u]), 1);
                st.row[e] = rw[u];
                st.pos[e] = pos;
                st.lab[e] = lb[u];
                st.a[e] = __ldg(S.tile_lab + (pos >> 7));
                st.mask[e] = __ldcs(wmask + base + e);
                st.lun[e] = ln[u];
            }
        }
        __syncthreads();
        // ---- B: centered split rows and records, 4 rows per lane group at a time
        // (block-uniform trip count: the 8-lane shuffles below need every
        // lane of the warp)
        for (int b0 = 0; b0 < nrow; b0 += 32 * 4) {
            float4 xv[4], ov[4];
            int er[4], ea[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int e = b0 + grp + u * 32;
                er[u] = e < nrow ? e : -1;
                ea[u] = er[u] >= 0 ? st.a[e] : -1;
                const bool ok = er[u] >= 0 && sub < c4n;
                xv[u] = ok ? __ldg(reinterpret_cast<const float4*>(S.X32 + (int64_t)st.row[e] * S.ldx) + sub)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
                ov[u] = (ok && ea[u] >= 0) ? __ldg(reinterpret_cast<const float4*>(S.C32 + (int64_t)ea[u] * S.ldc) + sub)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int e = er[u];
                double x2 = 0.0, xo = 0.0, xx = 0.0;
                const int pos = e >= 0 ? st.pos[e] : 0;
                if (e >= 0 && sub < c4n) {
                    const float xa[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
                    const float oa[4] = {ov[u].x, ov[u].y, ov[u].z, ov[u].w};
                    float xs[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        xs[q] = xa[q] - oa[q];
                        x2 = fma((double)xs[q], (double)xs[q], x2);
                        xo = fma((double)xs[q], (double)oa[q], xo);
                        xx = fma((double)xa[q], (double)xa[q], xx);
                    }
                    // x' itself (the pass splits it for 3xTF32 in shared memory)
                    __stcs(reinterpret_cast<float4*>(S.Xg_hi + (int64_t)pos * S.ldx) + sub,
                           make_float4(xs[0], xs[1], xs[2], xs[3]));
                }
#pragma unroll
                for (int o = L >> 1; o > 0; o >>= 1) {
                    x2 += __shfl_xor_sync(LK_FULL_MASK, x2, o, L);
                    xo += __shfl_xor_sync(LK_FULL_MASK, xo, o, L);
                    xx += __shfl_xor_sync(LK_FULL_MASK, xx, o, L);
                }
                if (e >= 0 && sub == 0) {
                    const int a = ea[u], row = st.row[e];
                    TgyMeta t;
                    t.R = x2 + 2.0 * xo;
                    t.xo = __double2float_ru(sqrt(x2) * (1.0 + 1e-12));
                    t.xn2 = S.X64 ? S.xn2[row] : (float)xx;
                    float bv = INFINITY;
                    if (a >= 0 && st.lab[e] == a) {
                        // upper bound on the TC value of the row's own label column (as k_gather_center)
                        const double xd = (double)t.xo, ca = (double)S.cnorm[a];
                        const double est = xd * xd - t.R;
                        const double gb = (double)(S.d + 4) * 5.9604644775390625e-08;
                        const double eA = (double)kap * xd * ca + gb * (fabs(est) + 2.0 * xd * ca) +
                                          2.0 * 5.9604644775390625e-08 * fabs(est);
                        bv = __double2float_ru(est + 2.0 * eA + 1e-30);
                    }
                    t.bv = bv;
                    t.lun = st.lun[e];
                    t.row = row;
                    t.mask = st.mask[e];
                    const int4* src = reinterpret_cast<const int4*>(&t);
                    int4* dst = reinterpret_cast<int4*>(S.tmeta + pos);
                    __stcs(dst, src[0]);
                    __stcs(dst + 1, src[1]);
                }
            }
        }
        __syncthreads();
    }
}

// Gather the sorted rows, shifted by their tile's centroid, split for 3xTF32;
// per row the fp64 row constant R and |x'| (rounded up); per tile its label.
// L lanes per row (float4 columns), 32 / L rows per warp in flight.
__global__ void __launch_bounds__(256) k_gather_center(DevState S, const int64_t* count, int L) {
    if (*S.done) return;
    const int64_t m = count ? *count : S.n;
    const int lane = threadIdx.x & 31, sub = lane & (L - 1);
    const int rpw = 32 / L;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int c4n = S.ldx / 4;
    const float kap = tc_kappa_ordered(S.d);
    // software pipeline: the next group's row id and labels (written by
    // k_label_scatter per sorted position) load while this group is processed
    int row_n = 0, lab_n = -1, a_n = -1;
    {
        const int64_t p = warp * rpw + lane / L;
        if (p < m) {
            row_n = S.perm[p];
            lab_n = S.rowlab[p];
            a_n = S.tile_lab[p >> 7];
        }
    }
    for (int64_t p0 = warp * rpw; p0 < m; p0 += nwarps * rpw) {
        const int64_t p = p0 + lane / L;
        const bool ok = p < m;
        const int64_t row = row_n;
        const int lab = lab_n, a = a_n;
        {
            const int64_t pn = p + nwarps * rpw;
            if (pn < m) {
                row_n = S.perm[pn];
                lab_n = S.rowlab[pn];
                a_n = S.tile_lab[pn >> 7];
            }
        }
        double x2 = 0.0, xo = 0.0, xx = 0.0;
        if (ok) {
            const float4* xp = reinterpret_cast<const float4*>(S.X32 + row * S.ldx);
            const float4* op = reinterpret_cast<const float4*>(S.C32 + (int64_t)(a >= 0 ? a : 0) * S.ldc);
            float4* hp = reinterpret_cast<float4*>(S.Xg_hi + p * S.ldx);
            float4* lp = reinterpret_cast<float4*>(S.Xg_lo + p * S.ldx);
            for (int c = sub; c < c4n; c += L) {
                const float4 x = __ldcs(xp + c);
                const float4 o = a >= 0 ? __ldg(op + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float xv[4] = {x.x, x.y, x.z, x.w};
                const float xs[4] = {x.x - o.x, x.y - o.y, x.z - o.z, x.w - o.w};
                const float ov[4] = {o.x, o.y, o.z, o.w};
                float h[4], l[4];
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    h[e] = __uint_as_float(__float_as_uint(xs[e]) & 0xFFFFE000u);
                    l[e] = xs[e] - h[e];
                    x2 = fma((double)xs[e], (double)xs[e], x2);
                    xo = fma((double)xs[e], (double)ov[e], xo);
                    xx = fma((double)xv[e], (double)xv[e], xx);
                }
                __stcs(hp + c, make_float4(h[0], h[1], h[2], h[3]));
                __stcs(lp + c, make_float4(l[0], l[1], l[2], l[3]));
            }
        }
        for (int o = L >> 1; o > 0; o >>= 1) {
            x2 += __shfl_xor_sync(LK_FULL_MASK, x2, o);
            xo += __shfl_xor_sync(LK_FULL_MASK, xo, o);
            xx += __shfl_xor_sync(LK_FULL_MASK, xx, o);
        }
        if (ok && sub == 0) {
            const double R = x2 + 2.0 * xo;
            const float xof = __double2float_ru(sqrt(x2) * (1.0 + 1e-12));
            S.rowR[p] = R;
            S.rowxo[p] = xof;
            // contiguous |x|^2 for k_assign_tc2's certification (fp64 sum rounded
            // once: within the 2^-22 the bound allows of k_split_points' value;
            // exact fp64 input keeps that value), and its search threshold: an
            // upper bound on the TC value of the row's own label column (rows of
            // the tile's label: D'_a = ||x'||^2 - R up to the dot error)
            S.rowxn2[p] = S.X64 ? S.xn2[row] : (float)xx;
            float bv = INFINITY;
            if (a >= 0 && lab == a) {
                const double xd = (double)xof, ca = (double)S.cnorm[a];
                const double est = xd * xd - R;
                const double gb = (double)(S.d + 4) * 5.9604644775390625e-08;
                const double ea = (double)kap * xd * ca + gb * (fabs(est) + 2.0 * xd * ca) +
                                  2.0 * 5.9604644775390625e-08 * fabs(est);
                bv = __double2float_ru(est + 2.0 * ea + 1e-30);
            }
            S.rowbv[p] = bv;
        }
    }
}

}  // namespace tc
}  // namespace lk

// ---------------------------------------------------------------------------
// host side: tensor maps through the driver entry point (no -lcuda needed)

namespace lkh {

using namespace lk;
using namespace lk::tc;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

static bool make_map(CUtensorMap* map, const float* base, int64_t rows, int cols, int ld,
                     int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool tc_supported(const DevState& S) {
    return S.Xlo != nullptr && S.d >= 8 && (S.ldx % 4) == 0 && get_encode() != nullptr;
}

static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);  // A/B knobs of the tensor-core pipeline
    return e ? atoi(e) : dflt;
}

static int g_tc_max_dyn = 0;  // dynamic smem limit of the split kernels (device opt-in max)
static int tc_max_dyn_smem() { return g_tc_max_dyn; }
static int g_tgy_max_dyn = 0;
static int tc_max_dyn_smem_tgy() { return g_tgy_max_dyn; }
// k_assign_tgy: the k_assign_tc2 layout + the pair's per-group minima
static int tgy_smem(const DevState& S) { return TgySmem::TOTAL + S.kpad * 4; }

template <int BN, int MODE, bool SPLIT, bool ARES, int CL = 1>
static lk_status tc_attr(int optin) {
    cudaFuncAttributes fa;
    LK_CUDA_CHECK(cudaFuncGetAttributes(&fa, k_assign_tc<BN, MODE, SPLIT, ARES, CL>));
    const int lim = optin - (int)fa.sharedSizeBytes;
    if (SPLIT && (g_tc_max_dyn == 0 || lim < g_tc_max_dyn)) g_tc_max_dyn = lim;
    LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_tc<BN, MODE, SPLIT, ARES, CL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       SPLIT ? lim : Smem<BN>::TOTAL));
    return LK_OK;
}

// Centroid-tile multicast width for d <= 32 (resident A): the B tiles stream
// from L2 once per cluster instead of once per CTA (the L2 -> SM traffic paces
// the d = 32 pass otherwise).  LK_TC_CL = 1 / 2 / 4 (A/B knob).
static int tc_cluster() {
    static const int v = [] {
        const int c = env_int("LK_TC_CL", 1);
        return (c == 1 || c == 2 || c == 4) ? c : 1;
    }();
    return v;
}

lk_status init_tc_attributes() {
    int dev = 0, optin = 0;
    LK_CUDA_CHECK(cudaGetDevice(&dev));
    LK_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    lk_status s = tc_attr<128, kTop2, false, false>(optin);
    if (s == LK_OK) s = tc_attr<128, kCollect, false, false>(optin);
    if (s == LK_OK) s = tc_attr<256, kTop2, false, false>(optin);
    if (s == LK_OK) s = tc_attr<256, kCollect, false, false>(optin);
    if (s == LK_OK) s = tc_attr<128, kTop2, true, false>(optin);
    if (s == LK_OK) s = tc_attr<128, kCollect, true, false>(optin);
    if (s == LK_OK) s = tc_attr<128, kTop2, true, true>(optin);
    if (s == LK_OK) s = tc_attr<128, kCollect, true, true>(optin);
    if (s == LK_OK) {
        LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           optin - 1024));
        cudaFuncAttributes fa;
        LK_CUDA_CHECK(cudaFuncGetAttributes(&fa, k_assign_tgy));
        g_tgy_max_dyn = optin - (int)fa.sharedSizeBytes;
        LK_CUDA_CHECK(cudaFuncSetAttribute(k_assign_tgy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           g_tgy_max_dyn));
    }
    if (s == LK_OK) s = tc_attr<128, kTop2, true, true, 2>(optin);
    if (s == LK_OK) s = tc_attr<128, kCollect, true, true, 2>(optin);
    if (s == LK_OK) s = tc_attr<128, kTop2, true, true, 4>(optin);
    if (s == LK_OK) s = tc_attr<128, kCollect, true, true, 4>(optin);
    return s;
}

// Split accumulators (tighter certification, fewer ambiguous rows) unless
// LK_TC_SPLIT=0 (A/B knob).
static bool tc_split() {
    static const int v = [] {
        const char* e = getenv("LK_TC_SPLIT");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

lk_status launch_tc_prep_points(const DevState& S, int sms, cudaStream_t st) {
    if (!S.Xlo) return LK_OK;
    k_split_points<<<sms * 8, 256, 0, st>>>(S);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

template <int BN, int MODE, bool SPLIT, bool ARES, int CL = 1>
static lk_status launch_bn(const DevState& S, const float* ahi, const float* alo, int64_t a_rows,
                           TcArgs A, int64_t max_rows, int64_t* stat, int sms, cudaStream_t st) {
    CUtensorMap mah, mal, mbh, mbl;
    if (!make_map(&mah, ahi, a_rows, S.d, S.ldx, BM) || !make_map(&mal, alo, a_rows, S.d, S.ldx, BM) ||
        !make_map(&mbh, S.Chi, S.kcols, S.d, S.ldc, ARES ? BN / 2 : BN) ||
        !make_map(&mbl, S.Clo, S.kcols, S.d, S.ldc, ARES ? BN / 2 : BN)) {
        set_error("cuTensorMapEncodeTiled failed");
        return LK_ERR_CUDA;
    }
    A.m = max_rows;
    A.n_ct = (S.kcols + BN - 1) / BN;
    static const int knob_fast = env_int("LK_TC_FAST", 1), knob_spin = env_int("LK_TC_SPIN", 0);
    A.fast = knob_fast;
    A.spin = knob_spin;
    static const int knob_dbg = env_int("LK_TC_DBG", 0);
    static const int knob_kouter = env_int("LK_TC_KOUTER", 1);
    A.kouter = knob_kouter;
    A.dbg = (MODE == kTop2 && A.center) ? knob_dbg : 0;  // (iteration >= 2 only)
    A.n_kc = (S.d + KC - 1) / KC;
    int smem = Smem<BN, ARES>::TOTAL;
    if (A.sbeta) smem += 2 * S.kpad * 4;
    int64_t tiles = (max_rows + BM - 1) / BM;
    int grid = (int)(tiles < sms ? (tiles > 0 ? tiles : 1) : sms);
    auto kern = k_assign_tc<BN, MODE, SPLIT, ARES, CL>;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.blockDim = dim3(TcShape<SPLIT>::THREADS);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    if (CL > 1) {
        // one wave of whole clusters (a GPC with an odd free SM cannot host a pair)
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        static int max_cl[2] = {0, 0};  // per shared-memory variant (sbeta on / off)
        int& mc = max_cl[A.sbeta ? 1 : 0];
        if (mc == 0) {
            cfg.gridDim = dim3((unsigned)(sms / CL * CL));
            LK_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&mc, kern, &cfg));
            if (mc < 1) mc = 1;
        }
        int g = (int)((tiles + CL - 1) / CL);
        if (g > mc) g = mc;
        grid = g * CL;
    }
    cfg.gridDim = dim3((unsigned)grid);
    LK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, mah, mal, mbh, mbl, S, A, stat));
    LK_LAUNCH_CHECK();
    return LK_OK;
}

// d <= 32 top-2 pass: two row tiles per centroid tile (k_assign_tc2) unless
// LK_TC2=0 (A/B knob: the single-row-tile k_assign_tc)
static lk_status launch_tc2(const DevState& S, const float* ahi, const float* alo, TcArgs A,
                            int64_t max_rows, int64_t* stat, int sms, cudaStream_t st) {
    CUtensorMap mah, mal, mbh, mbl;
    if (!make_map(&mah, ahi, S.n, S.d, S.ldx, BM) || !make_map(&mal, alo, S.n, S.d, S.ldx, BM) ||
        !make_map(&mbh, S.Chi, S.kcols, S.d, S.ldc, 64) || !make_map(&mbl, S.Clo, S.kcols, S.d, S.ldc, 64)) {
        set_error("cuTensorMapEncodeTiled failed");
        return LK_ERR_CUDA;
    }
    A.m = max_rows;
    A.n_ct = (S.kcols + 127) / 128;
    A.n_kc = 1;
    A.sbeta = 0;
    const int64_t pairs = ((max_rows + BM - 1) / BM + 1) / 2;
    const int grid = (int)(pairs < sms ? (pairs > 0 ? pairs : 1) : sms);
    const int smem = Tc2Smem::TOTAL + 8 * S.kpad;
    k_assign_tc2<<<grid, 320, smem, st>>>(mah, mal, mbh, mbl, S, A, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

template <int MODE>
static lk_status launch_mode(const DevState& S, const float* ahi, const float* alo, TcArgs A,
                             int64_t max_rows, int64_t* stat, int sms, cudaStream_t st) {
    static const int knob_tc2 = env_int("LK_TC2", 1);
    if (MODE == kTop2 && tc_split() && S.d <= KC && knob_tc2 && Tc2Smem::TOTAL + 8 * S.kpad <= tc_max_dyn_smem())
        return launch_tc2(S, ahi, alo, A, max_rows, stat, sms, st);
    if (tc_split()) {
        // one K chunk (d <= 32): the row tile's A stays resident across centroid tiles
        const bool ares = S.d <= KC;
        const int base = ares ? Smem<128, true>::TOTAL : Smem<128, false>::TOTAL;
        if (A.sbeta && base + 2 * S.kpad * 4 > tc_max_dyn_smem()) A.sbeta = 0;
        if (ares) {
            const int cl = tc_cluster();
            if (cl == 4) return launch_bn<128, MODE, true, true, 4>(S, ahi, alo, S.n, A, max_rows, stat, sms, st);
            if (cl == 2) return launch_bn<128, MODE, true, true, 2>(S, ahi, alo, S.n, A, max_rows, stat, sms, st);
            return launch_bn<128, MODE, true, true>(S, ahi, alo, S.n, A, max_rows, stat, sms, st);
        }
        return launch_bn<128, MODE, true, false>(S, ahi, alo, S.n, A, max_rows, stat, sms, st);
    }
    A.sbeta = 0;
    if (S.k <= 128) return launch_bn<128, MODE, false, false>(S, ahi, alo, S.n, A, max_rows, stat, sms, st);
    return launch_bn<256, MODE, false, false>(S, ahi, alo, S.n, A, max_rows, stat, sms, st);
}

lk_status launch_assign_tc(const DevState& S, const int32_t* rowlist, const int64_t* rowcount,
                           int64_t* stat, int64_t max_rows, int sms, cudaStream_t st) {
    TcArgs A = {};
    A.rowlist = rowlist;
    A.rowcount = rowcount;
    if (rowlist) {
        // gather the worklist into contiguous rescan buffers first
        k_gather_rows<<<sms * 8, 256, 0, st>>>(S, rowlist, rowcount);
        LK_LAUNCH_CHECK();
        return launch_mode<kTop2>(S, S.Xg_hi, S.Xg_lo, A, max_rows, stat, sms, st);
    }
    return launch_mode<kTop2>(S, S.X32, S.Xlo, A, max_rows, stat, sms, st);
}

lk_status launch_pair_table(const DevState& S, cudaStream_t st) {
    if (!S.center) return LK_OK;
    const int64_t tiles64 = (int64_t)(S.kpad / 64) * ((S.k + 63) / 64);
    if (tiles64 >= 148) {
        const dim3 g((unsigned)(S.kpad / 64), (unsigned)((S.k + 63) / 64));
        k_pair_table<64><<<g, 256, 0, st>>>(S);
    } else {
        const dim3 g((unsigned)(S.kpad / 16), (unsigned)((S.k + 15) / 16));
        k_pair_table<16><<<g, 256, 0, st>>>(S);
    }
    LK_LAUNCH_CHECK();
    return LK_OK;
}

// Tensor-core assignment of a row list (nullptr: every row) on label-sorted,
// centroid-shifted tiles.  Labels must be valid (iteration >= 2).
lk_status launch_assign_tc_centered(const DevState& S, const int32_t* rowlist,
                                    const int64_t* rowcount, int64_t* stat, int64_t max_rows,
                                    bool counts_are_local, int sms, cudaStream_t st) {
    if (!S.center || !tc_split()) return launch_assign_tc(S, rowlist, rowcount, stat, max_rows, sms, st);
    const int grid = sms * 8;
    if (rowlist == nullptr && counts_are_local) {
        k_label_scan<<<1, 1024, 0, st>>>(S, 1);  // the label counts are the histogram
        LK_LAUNCH_CHECK();
    } else {
        LK_CUDA_CHECK(cudaMemsetAsync(S.lcur, 0, (size_t)(S.kcols + 1) * 4, st));
        // (every local row of a shard: its counts are global, histogram the labels)
        k_label_count<<<grid, 256, 0, st>>>(S, rowlist, rowcount);
        LK_LAUNCH_CHECK();
        k_label_scan<<<1, 1024, 0, st>>>(S, 0);
        LK_LAUNCH_CHECK();
    }
    k_label_scatter<<<grid, 256, 0, st>>>(S, rowlist, rowcount);
    LK_LAUNCH_CHECK();
    int L = 1;
    while (L < 32 && L * 2 <= S.ldx / 4) L *= 2;
    k_gather_center<<<sms * 8, 256, 0, st>>>(S, rowcount, L);
    LK_LAUNCH_CHECK();
    TcArgs A = {};
    A.rowlist = S.perm;
    A.rowcount = rowcount;
    A.center = 1;
    A.sbeta = 1;  // (dropped by launch_mode when the double buffer does not fit)
    return launch_mode<kTop2>(S, S.Xg_hi, S.Xg_lo, A, max_rows, stat, sms, st);
}

// Rescan of the bound filter's worklist, or -- when most rows failed their
// bounds (d = 128 Gaussian-mixture rows: every row) -- one dense pass over all
// rows without the gather: both are launched, the device count picks (a pass
// over rows whose bounds held re-certifies them: same labels, fresh bounds).
// Worklist pass up to 70% of the rows (gather + 0.7 pass ~ one dense pass).
lk_status launch_assign_tc_adaptive(const DevState& S, const int32_t* rowlist, const int64_t* rowcount,
                                    int64_t* stat, int64_t max_rows, int sms, cudaStream_t st) {
    const int64_t thr = (S.n * 7) / 10;
    k_gather_rows<<<sms * 8, 256, 0, st>>>(S, rowlist, rowcount, thr);
    LK_LAUNCH_CHECK();
    TcArgs A = {};
    A.rowlist = rowlist;
    A.rowcount = rowcount;
    A.gate_cnt = rowcount;
    A.gate_thr = thr;
    A.gate = 2;
    lk_status s = launch_mode<kTop2>(S, S.Xg_hi, S.Xg_lo, A, max_rows, stat, sms, st);
    if (s != LK_OK) return s;
    TcArgs B = {};
    B.gate_cnt = rowcount;
    B.gate_thr = thr;
    B.gate = 1;
    return launch_mode<kTop2>(S, S.X32, S.Xlo, B, S.n, stat, sms, st);
}

// LK_TGY_PROF=1 (debug knob): k_assign_tgy accumulates its phase clocks into a
// managed buffer, printed to stderr at exit (tgy_prof_dump).
static unsigned long long* g_tgy_prof = nullptr;
static void tgy_prof_dump() {
    if (!g_tgy_prof) return;
    cudaDeviceSynchronize();
    static const char* names[] = {"P_aempty", "P_empty", "P_rempty", "P_total", "M_afull", "M_tempty",
                                  "M_full", "M_total", "E_tfull", "E_rfull", "E_tiles", "E_tail",
                                  "E_total", "pairs(warp0)", "tiles(warp0)", "T_cert", "T_groups",
                                  "T_stores", "T_append",
#ifdef LK_TGY_PROF_CHUNKS
                                  "C_load", "C_fast", "C_slow", "chunks(warp0)", "slow_chunks(warp0)"
#endif
    };
    fprintf(stderr, "k_assign_tgy phase clocks (sum over CTAs, lane 0 of producer / MMA / epilogue warp 0):");
    for (int e = 0; e < TP_N; e++) fprintf(stderr, " %s=%llu", names[e], g_tgy_prof[e]);
    fprintf(stderr, "\n");
}
static unsigned long long* tgy_prof_buffer() {
    static const int on = env_int("LK_TGY_PROF", 0);
    if (!on) return nullptr;
    if (!g_tgy_prof) {
        if (cudaMallocManaged(&g_tgy_prof, 64 * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
        memset(g_tgy_prof, 0, 64 * sizeof(unsigned long long));
        atexit(tgy_prof_dump);
    }
    return g_tgy_prof;
}

// Block-sparse Yinyang pass over the filter's worklist (stat[LK_STAT_WORK]
// rows, masks in S.ymask): label sort, pair masks, centered gather, then the
// (row-tile pair x group tile) MMAs of k_assign_tgy.
// the worklist is partitioned by mask bucket before the label sort
// (LK_TGY_BUCKET, A/B knob, default 0: sort by label alone.  Measured on cfg5:
// the pass evaluates 13% fewer products, not the 35% the tile unions alone
// predict -- a row also has the bounds of its tile's other groups refreshed, so
// wider unions list fewer rows and leave fewer ambiguous -- and the partition
// costs more than the pass saves)
bool tgy_bucket_on(const DevState& S) {
    static const int bucket = env_int("LK_TGY_BUCKET", 0);
    return bucket != 0 && S.work2 != nullptr;
}

lk_status launch_sort_tgy(const DevState& S, int64_t* stat, int sms, cudaStream_t st) {
    const int64_t* count = stat + LK_STAT_WORK;
    const int nb = tgy_sort_blocks(sms);
    const size_t hs = (size_t)S.kcols * 4;
    const bool bucket = tgy_bucket_on(S);
    const int32_t* wrow = S.work;
    const uint32_t* wmask = S.ymask;
    const float2* wlun = S.ylun;
    if (bucket) {
        k_bucket_hist<<<nb, 256, 0, st>>>(S, count);
        LK_LAUNCH_CHECK();
        k_bucket_offsets<<<1, 1024, 0, st>>>(S, nb);
        LK_LAUNCH_CHECK();
        k_bucket_scatter<<<nb, 256, 0, st>>>(S, count);
        LK_LAUNCH_CHECK();
        wrow = S.work2;
        wmask = S.ymask2;
        wlun = S.ylun2;
    }
    k_sort_hist<<<nb, 256, hs, st>>>(S, count, S.shist, wlun);
    LK_LAUNCH_CHECK();
    k_sort_offsets<<<(S.kcols + 255) / 256, 256, 0, st>>>(S, S.shist, nb);
    LK_LAUNCH_CHECK();
    k_label_scan<<<1, 1024, 0, st>>>(S, 0);
    LK_LAUNCH_CHECK();
    k_tile_labels<<<sms * 2, 256, 0, st>>>(S, count);
    LK_LAUNCH_CHECK();
    // (d <= 32: at most 8 float4 columns per row)
    // (the row's chain of dependent loads -- worklist, label, cursor, tile
    // label, point -- is the limit, not the bytes: see k_sort_gather)
    k_sort_gather<<<nb, 256, hs, st>>>(S, count, S.shist, wrow, wmask, wlun);
    LK_LAUNCH_CHECK();
    k_pair_mask<<<sms * 4, 256, 0, st>>>(S, count, bucket ? 1 : 0);
    LK_LAUNCH_CHECK();
    k_pair_info<<<sms, 256, 0, st>>>(S, count);
    LK_LAUNCH_CHECK();
    if (bucket) {
        k_pick_sel<<<(S.k + 127) / 128, 128, 0, st>>>(S);
        LK_LAUNCH_CHECK();
    }
    return LK_OK;
}

lk_status launch_assign_tgy(const DevState& S, int64_t* stat, int64_t max_rows, int sms,
                            cudaStream_t st) {
    const int64_t* count = stat + LK_STAT_WORK;
    CUtensorMap mah, mal, mbh, mbl;
    if (!make_map(&mah, S.Xg_hi, S.n, S.d, S.ldx, BM) || !make_map(&mal, S.Xg_lo, S.n, S.d, S.ldx, BM) ||
        !make_map(&mbh, S.Chi, S.kcols, S.d, S.ldc, 64) || !make_map(&mbl, S.Clo, S.kcols, S.d, S.ldc, 64)) {
        set_error("cuTensorMapEncodeTiled failed");
        return LK_ERR_CUDA;
    }
    TcArgs A = {};
    A.m = max_rows;
    A.rowcount = count;
    A.rowlist = S.perm;
    A.center = 1;
    A.n_kc = 1;
    A.n_ct = S.t_groups;
    A.prof = tgy_prof_buffer();
    {
        // LK_TGY_DBG=v LK_TGY_DBG_AT=N (timing probes, wrong results): launch N
        // (1-based; 0: every launch) runs without 1 the chunks' exact top-2,
        // 2 the per-tile group bounds, 3 the pair tail, 4 the chunk math
        static int dbg_launch = 0;
        static const int dbg = env_int("LK_TGY_DBG", 0), dbg_at = env_int("LK_TGY_DBG_AT", 0);
        dbg_launch++;
        A.dbg = (dbg && (dbg_at == 0 || dbg_at == dbg_launch)) ? dbg : 0;
    }
    {
        // LK_TGY_PROF_SKIP=N: the first N launches run without the clocks
        static int launches = 0;
        static const int skip = env_int("LK_TGY_PROF_SKIP", 0);
        if (launches++ < skip) A.prof = nullptr;
    }
    const int smem = tgy_smem(S);
    if (smem > tc_max_dyn_smem_tgy()) {
        set_error("group-tile pass: %d B of shared memory needed (k = %d)", smem, S.k);
        return LK_ERR_UNSUPPORTED;
    }
    k_assign_tgy<<<sms, 352, smem, st>>>(mah, mal, mbh, mbl, S, A, stat);
    LK_LAUNCH_CHECK();
    return LK_OK;
}

// Second pass over the ambiguous rows: collect every centroid under the row's
// certified threshold into cand_slots (count in cand_cnt; > LK_MAX_CAND =
// overflow, decided by the full fp64 recheck).
lk_status launch_collect_tc(const DevState& S, int64_t* stat, int64_t max_rows, int sms,
                            cudaStream_t st) {
    TcArgs A = {};
    A.rowlist = S.cand_rows;
    A.rowcount = stat + LK_STAT_CANDIDATE;
    A.thr = S.cand_thr;
    A.slots = S.cand_slots;
    A.cnt = S.cand_cnt;
    k_gather_rows<<<sms * 8, 256, 0, st>>>(S, S.cand_rows, stat + LK_STAT_CANDIDATE);
    LK_LAUNCH_CHECK();
    return launch_mode<kCollect>(S, S.Xg_hi, S.Xg_lo, A, max_rows, stat, sms, st);
}

}  // namespace lkh
