// lk_internal.h -- launchers shared between the kernel translation units and
// the C ABI (lk_api.cu).  Not part of the public boundary.
#pragma once

#include "lk_common.cuh"

namespace lkh {

lk_status launch_assign_simt(const lk::DevState& S, const int32_t* rowlist,
                             const int64_t* rowcount, int64_t* stat, int64_t max_rows, int sms,
                             cudaStream_t st);
// a short device-counted row list (d <= 32: one warp per row)
lk_status launch_assign_short(const lk::DevState& S, const int32_t* rowlist,
                              const int64_t* rowcount, int64_t* stat, int64_t max_rows, int sms,
                              cudaStream_t st);
// qscale_inline: also add the refinement deltas of the rows it moves
lk_status launch_recheck(const lk::DevState& S, int64_t* stat, int64_t max_rows, int sms,
                         cudaStream_t st, const double* qscale_inline = nullptr);
lk_status launch_recheck_cand(const lk::DevState& S, int64_t* stat, int64_t max_rows, int sms,
                              cudaStream_t st);
lk_status launch_filter_hamerly(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st);
lk_status launch_refine(const lk::DevState& S, int64_t* stat, const double* qscale,
                        int64_t max_rows, int sms, cudaStream_t st);
lk_status launch_update(const lk::DevState& S, const double* qscale, const double* qinv,
                        double* sse_part, bool need_half, cudaStream_t st);
lk_status launch_log_history(const lk::DevState& S, int sms, cudaStream_t st);
lk_status init_simt_attributes();
lk_status launch_d2_update(const float* x32, const double* x64, int64_t n, int d, int64_t ldx,
                           const double* c, double* d2, int first, const lk::PwProg& prog,
                           cudaStream_t st);
lk_status init_tc_attributes();
lk_status init_yy_attributes();
lk_status launch_scan_exp(const lk::DevState& S, int sms, cudaStream_t st);

// debug shadow check of the stored bounds (lk_validate.cu): worst overshoot
// per kind into host_out[0 .. nout) (ub, lb_global, lb_group[g]); synchronous
lk_status launch_validate(const lk::DevState& S, int decayed, double* host_out, int nout,
                          double* dev_scratch, cudaStream_t st);
bool yy_masked(const lk::DevState& S);
// one-kernel Yinyang iteration (lk_yy_fused.cu), d <= 32 and t <= 32
bool yy_fused_ok(const lk::DevState& S);
lk_status init_fused_attributes();
lk_status launch_yy_fused(const lk::DevState& S, int64_t* stat, const double* qscale, int sms,
                          cudaStream_t st);
lk_status launch_yy_seed(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st);
// full_only: every row failing the bounds is rescanned in full (tensor-core runs with d > 32)
lk_status launch_yy_filter(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st,
                           bool full_only);
lk_status launch_yy_pairs(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st,
                          bool full_only);
lk_status launch_yy_merge(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st,
                          bool full_only);

// tcgen05 path (lk_tc.cu): full-scan assignment with 3xTF32 products.
bool tc_supported(const lk::DevState& S);
lk_status launch_tc_prep_points(const lk::DevState& S, int sms, cudaStream_t st);
// tile centering: the k x k table of squared centroid distances (after every
// centroid update) and the centered full pass / rescan (iteration >= 2)
lk_status launch_pair_table(const lk::DevState& S, cudaStream_t st);
lk_status launch_assign_tc_centered(const lk::DevState& S, const int32_t* rowlist,
                                    const int64_t* rowcount, int64_t* stat, int64_t max_rows,
                                    bool counts_are_local, int sms, cudaStream_t st);
lk_status launch_collect_tc(const lk::DevState& S, int64_t* stat, int64_t max_rows, int sms,
                            cudaStream_t st);
// block-sparse Yinyang on the tensor cores (group tiles, d <= 32): the bound
// filter (lk_tgy.cu) and the sorted, masked tcgen05 pass over its worklist
// Elkan's per-centroid bounds (lk_elkan.cu): half-distance table + assignment
lk_status launch_elkan(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st);
// Regroup (lk_regroup.cu): the per-iteration regrouping and bound remap
lk_status launch_regroup(const lk::DevState& S, int32_t* scr, double* means, int sms, cudaStream_t st);
lk_status launch_filter_tgy(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st);
lk_status launch_sort_tgy(const lk::DevState& S, int64_t* stat, int sms, cudaStream_t st);
bool tgy_bucket_on(const lk::DevState& S);  // 4 more launches in launch_sort_tgy
lk_status launch_assign_tgy(const lk::DevState& S, int64_t* stat, int64_t max_rows, int sms,
                            cudaStream_t st);
// worklist rescan or, when the list holds most rows, one dense pass (device-chosen)
lk_status launch_assign_tc_adaptive(const lk::DevState& S, const int32_t* rowlist,
                                    const int64_t* rowcount, int64_t* stat, int64_t max_rows, int sms,
                                    cudaStream_t st);
lk_status launch_assign_tc(const lk::DevState& S, const int32_t* rowlist,
                           const int64_t* rowcount, int64_t* stat, int64_t max_rows, int sms,
                           cudaStream_t st);

}  // namespace lkh
