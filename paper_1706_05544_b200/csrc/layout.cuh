// layout.cuh -- host launchers of layout.cu (setup, reductions, model assembly) and predict.cu.
#pragma once

#include <algorithm>

#include "svm_internal.cuh"

cudaError_t lay_check_finite(const float* p, int64_t n, int* d_bad, cudaStream_t st);
cudaError_t lay_check_csr(const int64_t* indptr, const int32_t* idx, int64_t n, int64_t d,
                          int64_t nnz, int* d_bad, cudaStream_t st);
// CSR rows in slices of 32 (SmoArgs::sell_*): group counts per slice, then the packed copy
cudaError_t lay_sell_len(const int64_t* indptr, int64_t n, int64_t R, int spc, int64_t ns,
                         int64_t* len, cudaStream_t st);
cudaError_t lay_sell_fill(const int64_t* indptr, const int32_t* idx, const float* vals, int64_t n,
                          int64_t d, int64_t R, int spc, int64_t ns, const int64_t* gptr, uint2* sidx,
                          float4* sval, cudaStream_t st);
cudaError_t lay_rowmajor_to_XT(const float* X, int64_t n, int64_t d, float* XT, int64_t n_pad,
                               cudaStream_t st);
cudaError_t lay_colmajor_to_XT(const float* X, int64_t n, int64_t d, float* XT, int64_t n_pad,
                               cudaStream_t st);
cudaError_t lay_XT_to_rowmajor(const float* XT, int64_t n, int64_t d, int64_t n_pad, float* X,
                               cudaStream_t st);
cudaError_t lay_norms_XT(const float* XT, int64_t n, int64_t d, int64_t n_pad, float* xnorm,
                         cudaStream_t st);
cudaError_t lay_norms_csr(const int64_t* indptr, const float* vals, int64_t n, int64_t n_pad,
                          float* xnorm, cudaStream_t st);
cudaError_t lay_init_state(const float* yv, int64_t n, int64_t n_pad, int ncopy, double eps,
                           double C, double* alpha, float* G, uint8_t* status, cudaStream_t st);
cudaError_t lay_exclude_fold(const int32_t* fold, int32_t held, int64_t n, int64_t n_pad,
                             int ncopy, uint8_t* status, cudaStream_t st);
cudaError_t lay_status_from_alpha(const double* alpha, int64_t n, int64_t n_pad, int ncopy,
                                  double C, uint8_t* status, cudaStream_t st);
cudaError_t lay_pack_state(const double* alpha, const float* G, int64_t n, int64_t n_pad,
                           int ncopy, double* a_out, float* g_out, cudaStream_t st);
cudaError_t lay_unpack_state(const double* a_in, const float* g_in, int64_t n, int64_t n_pad,
                             int ncopy, double* alpha, float* G, cudaStream_t st);
cudaError_t lay_reduce_state(const double* alpha, const float* G, const uint8_t* status,
                             const float* yv, int64_t n, int64_t n_pad, int ncopy, double eps,
                             double C, double* d_out5, cudaStream_t st);
cudaError_t lay_coef(const double* alpha, const uint8_t* status, int64_t n, int64_t n_pad,
                     int ncopy, double C, double* coef, uint8_t* svflag, cudaStream_t st);
// incremental re-certification: delta = coef - coef_prev, flag = delta != 0, coef_prev = coef;
// a += b (fp64)
cudaError_t lay_coef_delta(const double* coef, double* coef_prev, int64_t n, double* delta,
                           uint8_t* flag, cudaStream_t st);
cudaError_t lay_add_f64(double* a, const double* b, int64_t n, cudaStream_t st);
cudaError_t lay_count_flags(const uint8_t* flag, int64_t n, int32_t* cnt, int* nblk_out,
                            cudaStream_t st);
cudaError_t lay_scatter_flags(const uint8_t* flag, int64_t n, const int64_t* offs, int64_t* out,
                              cudaStream_t st);
cudaError_t lay_gather_sv(const float* XT, int64_t n_pad, int64_t d, const float* xnorm,
                          const int64_t* sv_idx, int64_t nsv, int64_t nsv_pad, float* SVT,
                          float* svnorm, cudaStream_t st);
cudaError_t lay_csr_to_XT(const int64_t* indptr, const int32_t* idx, const float* vals,
                          const int64_t* rows, int64_t nrows, int64_t row_base, float* XT,
                          int64_t ld, cudaStream_t st);
cudaError_t lay_gather_coef(const double* coef_rows, const int64_t* sv_idx, int64_t nsv,
                            int64_t nsv_pad, double* coef_sv, cudaStream_t st);

// ---- sharded path (peer pointers of every rank, mapped with cudaIpcOpenMemHandle) ----------
#define XCH_K 64
struct XchgPeers {
    double* buf[SVM_MAX_RANKS];     // [2][world][XCH_K] doubles on each rank
    uint32_t* flags[SVM_MAX_RANKS]; // [world] tags on each rank
};
struct SvPeers {
    int world;
    int64_t off[SVM_MAX_RANKS + 1];   // global SV offsets per rank
    int64_t n_local[SVM_MAX_RANKS], row0[SVM_MAX_RANKS];
    const float* XR[SVM_MAX_RANKS];   // dense rows (NULL for CSR)
    const int64_t* indptr[SVM_MAX_RANKS];
    const int32_t* indices[SVM_MAX_RANKS];
    const float* vals[SVM_MAX_RANKS];
    const float* norms[SVM_MAX_RANKS];
    const int64_t* svidx[SVM_MAX_RANKS];  // local SV row indices per rank
    const double* coefx[SVM_MAX_RANKS];   // per-row coefficients [nprob][n_local] per rank
};
cudaError_t lay_xchg(const double* vals, int K, int rank, int world, const XchgPeers& P,
                     uint32_t tag, double* out, uint64_t timeout_ns, int* err, cudaStream_t st);
cudaError_t lay_gather_global_sv(const SvPeers& P, int64_t nsv, int64_t nsv_pad, int64_t d,
                                 int nprob, float* SVT, float* svn, double* coef, int64_t* grow,
                                 cudaStream_t st);

// predict.cu: F[q * ldf + p] (+)= sum_s coef[p * nsv_pad + s] K(sv_s, x_q) (+ b[p]) in fp64 for
// queries in feature-major [d][nq_pad] and SVs in feature-major [d][nsv_pad].
cudaError_t pred_decision(const float* XqT, const float* qnorm, int64_t nq, int64_t nq_pad,
                          const float* SVT, const float* svnorm, int64_t nsv, int64_t nsv_pad,
                          int64_t d, const double* coef, int n_out, const KParams& kp,
                          double* F, cudaStream_t st, const float* SVtc = nullptr, bool f16_any_d = false);
// (f16_any_d: use the fp16-split tcgen05 kernel for every d -- predict; the certification keeps the
// 3xTF32 kernel for d <= 128, whose measured violations decide the resume of the loop)
// tcgen05 predict (d <= 128): SV tiles [nsv_pad / 64][hi | lo][64 * dp] in the K-major core
// layout (dp = pred_tc_dp(d)); 0 when the tensor-core path does not apply
int64_t pred_tc_dp(int64_t d);
int64_t pred_sv_tiles_floats(int64_t nsv_pad, int64_t d, int n_out);   // tiles + fp32 coefficients
cudaError_t pred_sv_tiles(const float* SVT, int64_t nsv_pad, int64_t d, const double* coef, int n_out,
                          float* out, cudaStream_t st);
// G refresh from raw decision sums (certification, a4): G_c(i) = p_c(i) + y_c * F[i]
cudaError_t pred_refresh_G(const double* F, const float* yv, const uint8_t* status, int64_t n,
                           int64_t n_pad, int ncopy, double eps, float* G, cudaStream_t st);
// labels / values from decision values (+ b)
cudaError_t pred_finalize(const double* F, int64_t nq, int n_out, const double* b, int mode,
                          const double* labels, double first_label, float* decision, float* out,
                          cudaStream_t st);
