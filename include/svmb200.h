/*
 * svmb200.h -- C ABI of the B200-native working-set SVM library (libsvmb200.so).
 *
 * The library implements one path of Rgtsvm (arXiv 1706.05544): the working-set dual
 * decomposition of Eq. 2 for C-classification and eps-regression (Eq. 1,
 * P:59-63; "substituting the generalized linear term p"), iterated as P:53 describes --
 * "iteratively optimizing 16 heuristically selected dual space coefficients ... Each iteration
 * starts by calculating the gradient for all dual space coefficients, followed by picking 16
 * dual space coefficients ... The 16 dual space coefficients are then optimized based on the
 * local gradient" -- plus the decision-function predict the benchmark of P:92/P:96 times.
 * The call shape follows the e1071-compatible interface the paper claims:
 * svm(x, y, type, kernel, cost, gamma, degree, coef0, epsilon, tolerance).
 * (P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n; readings in DESIGN.md.)
 *
 * Conventions for every entry point
 *   - Every function returns an int status: SVM_OK (0) or a negative SVM_E* code; none throws
 *     or aborts.  On error, svm_last_error() returns a thread-local, human-readable message and
 *     all output pointers are left untouched (model handles: *out is set to NULL).
 *   - Array arguments may live in host memory or in device memory of the current CUDA device;
 *     the library detects which with cudaPointerGetAttributes.  They are BORROWED for the call
 *     only: read (or written, for outputs) during the call, never freed or retained
 *     ("Efficient memory handling": the library takes addresses, never owns user data).
 *   - Dense matrices are n x d fp32 in `layout` order: SVM_ROW_MAJOR (C order, row i contiguous)
 *     or SVM_COL_MAJOR (R / Fortran order, feature k contiguous).
 *   - CSR matrices: indptr int64[n+1] (indptr[0] = 0, non-decreasing), indices int32[nnz]
 *     strictly increasing within a row and < d, data fp32[nnz].
 *   - All work is ordered on params->stream (a cudaStream_t, NULL = the legacy default stream);
 *     functions return after their results are in the caller's buffers.
 */
#ifndef SVMB200_H
#define SVMB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ----------------------------------------------------------------------- */
#define SVM_OK 0
#define SVM_EINVAL (-1)       /* bad argument: shapes, parameters, CSR invariants, d mismatch */
#define SVM_EDEGENERATE (-2)  /* classification labels with a single class            */
#define SVM_ENONFINITE (-3)   /* a non-finite value in X or y                    */
#define SVM_ENOMEM (-4)       /* device or host allocation failed                              */
#define SVM_ECUDA (-5)        /* a CUDA runtime error (message carries cudaGetErrorString)     */
#define SVM_EPEER (-6)        /* sharded run: peer-memory mapping / rank exchange failed       */
#define SVM_ETIMEOUT (-7)     /* sharded run: a rank stopped publishing working-set candidates */
#define SVM_ENCCL (-8)        /* svm_train_sharded*: NCCL could not be loaded or a call failed  */

/* ---- enums (e1071 numbering) ------------------------------------------------------------- */
#define SVM_C_CLASSIFICATION 0 /* e1071 type = "C-classification"  (P:75 item 1)            */
#define SVM_EPS_REGRESSION 3   /* e1071 type = "eps-regression"    (Eq. 1)         */

#define SVM_LINEAR 0     /* u.v                        */
#define SVM_POLYNOMIAL 1 /* (gamma u.v + coef0)^degree                                        */
#define SVM_RADIAL 2     /* exp(-gamma |u - v|^2)                                             */
#define SVM_SIGMOID 3    /* tanh(gamma u.v + coef0)                                           */

#define SVM_ROW_MAJOR 0
#define SVM_COL_MAJOR 1

/* ---- training parameters (e1071 argument names) ------------------------------ */
typedef struct svm_params {
    int32_t type;        /* SVM_C_CLASSIFICATION | SVM_EPS_REGRESSION                           */
    int32_t kernel;      /* SVM_LINEAR | SVM_POLYNOMIAL | SVM_RADIAL | SVM_SIGMOID              */
    double cost;         /* C > 0, the box bound of Eq. 1/2;                     default 1      */
    double gamma;        /* kernel gamma; <= 0 selects 1/d;               default 1/d    */
    int32_t degree;      /* polynomial degree >= 1;                              default 3      */
    double coef0;        /* polynomial / sigmoid offset;                         default 0      */
    double epsilon;      /* eps-SVR tube half-width >= 0 (Eq. 1);                default 0.1    */
    double tolerance;    /* stop when m_up - M_low <= tolerance (KKT reading of P:53);
                            > 0;                                                 default 1e-3   */
    int32_t working_set; /* |W|, even, 2..16 ("16 ... coefficients");      default 16     */
    int64_t max_iter;    /* outer-iteration cap per binary problem; <= 0 selects max(10 m, 1e4)
                            (S:41).  Hitting it is not an error: info.converged = 0.    */
    int32_t layout;      /* SVM_ROW_MAJOR | SVM_COL_MAJOR for dense X                           */
    int32_t certify;     /* after the loop, recompute G = Q a + p from the support vectors with
                            fp64 accumulation and resume if the violation exceeds tolerance:
                            1 = always, 0 = never, -1 = auto (when n * n_SV * d <= 2e15)  */
    void* stream;        /* cudaStream_t, or NULL for the legacy default stream                 */
} svm_params;

/* Fills *p with the defaults above for d features.  Returns SVM_EINVAL if p is NULL or d < 1. */
int svm_params_default(svm_params* p, int64_t d);

/* ---- model ------------------------------------------------------------------------------- */
typedef struct svm_model svm_model; /* opaque; owns device + host memory until svm_free_model */

typedef struct svm_model_info {
    int32_t type, kernel, degree;
    double gamma, coef0;
    int64_t n_features;   /* d                                                                */
    int64_t n_train;      /* training rows                                                    */
    int64_t n_sv;         /* support vectors: rows with any |coef| > 1e-12 C           */
    int32_t n_class;      /* 2 for binary, k for one-vs-rest, 0 for regression                */
    int32_t n_problem;    /* binary problems solved: 1, or k for one-vs-rest                  */
    double labels[64];    /* class labels in first-appearance order; first n_class    */
    double b[64];         /* bias per problem (sign-corrected)              */
    int64_t iterations;   /* total outer iterations over all problems                         */
    double violation;     /* largest final m_up - M_low over problems (fp32 G, after certify) */
    int32_t converged;    /* 1 if every problem reached tolerance                             */
    int32_t certified;    /* 1 if the final violation was re-measured from scratch (certify)   */
    double dual_objective;/* sum over problems of 1/2 a'(G + p)                       */
    double train_ms;      /* svm_train* wall time, entry to return                            */
    double loop_ms;       /* time inside the working-set loop (device events)                 */
    double setup_ms, certify_ms;
    int64_t passes;       /* passes of the dominant X-pass kernel in the loop: the iterations of  */
                          /* the persistent kernel, or the k_ovr_pass launches (batched OvR)      */
    double pass_ms;       /* their device time: loop_ms (persistent), or for the batched one-vs- */
                          /* rest passes the mean of CUDA event pairs around every 8th k_ovr_pass */
                          /* launch times the launch count                                        */
    int32_t batched;      /* 1 if the one-vs-rest problems iterated together      */
    double exchange_ms;   /* part of loop_ms the persistent kernel spent in the per-iteration    */
                          /* candidate exchange (a1), measured on CTA 0 of this rank: from its  */
                          /* publish until every CTA's (every rank's, when sharded) keys are    */
                          /* staged -- transport latency plus the wait for the slowest CTA.     */
                          /* 0 for the batched one-vs-rest passes.                               */
    double exchange_p50_us; /* median and 99th percentile of that per-iteration exchange latency */
    double exchange_p99_us; /* (histogram of 512-cycle bins, converted at the loop's clock)       */
    int64_t cache_passes;   /* iterations whose W rows were all in the kernel-column cache (SURVEY */
                            /* 8(f) #3): their pass read K columns instead of X                  */
    int32_t certifications; /* certification passes run over all problems (a resumed loop is     */
                            /* certified again, from the rows whose coefficient changed only)    */
} svm_model_info;

/*
 * svm_train -- fit on dense X (n x d fp32, params->layout order) and labels / targets y (fp32[n]).
 *   C-classification: y holds class codes.  Exactly {-1,+1}: used as-is.  Two other values: the
 *   first-appearing label maps to +1.  k > 2 values: k one-vs-rest problems on the shared X
 *   (BASELINE config 3; the paper names multi-class but not its scheme).
 *   eps-regression: y = z, the responses of Eq. 1.
 * Writes a new model to *out (caller frees with svm_free_model).
 * Errors: SVM_EINVAL (n < 2, d < 1, cost <= 0, gamma < 0 is treated as default, degree < 1,
 *   epsilon < 0, tolerance <= 0, working_set odd / < 2 / > 16, k > 64 classes, NULL pointers),
 *   SVM_ENONFINITE, SVM_EDEGENERATE (one class), SVM_ENOMEM, SVM_ECUDA.
 */
int svm_train(const float* X, const float* y, int64_t n, int64_t d, const svm_params* params,
              svm_model** out);

/* svm_train_csr -- as svm_train, X in CSR form (the sparse-input path). */
int svm_train_csr(const int64_t* indptr, const int32_t* indices, const float* data,
                  const float* y, int64_t n, int64_t d, const svm_params* params, svm_model** out);

/*
 * svm_predict -- decision values f(x) = sum_s coef_s K(sv_s, x) + b for nq dense
 * query rows (nq x d fp32 in `layout`).
 *   decision: fp32[nq * n_problem], row-major (query-major); may be NULL.
 *   out:      fp32[nq]: SVC label (sign(f), f = 0 -> the first class; one-vs-rest: label of
 *             argmax_c f_c, ties -> lowest c) or the SVR value f; may be NULL.
 * Errors: SVM_EINVAL (NULL model, d != model d, nq < 0), SVM_ENOMEM, SVM_ECUDA.
 */
int svm_predict(const svm_model* model, const float* Xq, int64_t nq, int64_t d, int32_t layout,
                float* decision, float* out);

/* svm_predict_csr -- as svm_predict with CSR queries. */
int svm_predict_csr(const svm_model* model, const int64_t* indptr, const int32_t* indices,
                    const float* data, int64_t nq, int64_t d, float* decision, float* out);

/* Model accessors.  svm_model_get_sv writes, for each support vector s < n_sv, its training-row
 * index (int64, may be NULL) and its coefficients coef[p * n_sv + s] for every problem p
 * (fp64[n_problem * n_sv], may be NULL): y_i a_i for SVC, a*_i - a_i for SVR. */
int svm_model_get_info(const svm_model* model, svm_model_info* info);
int svm_model_get_sv(const svm_model* model, int64_t* sv_index, double* coef);
void svm_free_model(svm_model* model);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* svm_last_error(void);

/* Number of CUDA kernels this library has launched since it was loaded (diagnostics: the bench
 * reports the launches inside its timed region from the difference of two calls). */
int64_t svm_launch_count(void);

/* ---- K-fold cross validation over a (gamma, C) grid ---------
 * For every grid cell g (gammas[g], costs[g]; NULL arrays = params' value) and fold f, the model of
 * the training split (rows with fold[i] != f) is trained exactly as svm_train would train it on
 * those rows (same label map from ALL of y, same one-vs-rest split for k > 2 classes) and
 * evaluated on the held-out rows.  All problems share one device copy of X: held-out rows leave a
 * problem through their status, classification problems run 16 at a time through the batched
 * tcgen05 pass (one X pass per iteration for all of them, per-problem gamma and C), eps-SVR ones
 * on the persistent kernel.  The held-out decision values come from the certified G (recomputed
 * from the fold model's support vectors, fp64 sums).
 *   fold: int32[n] fold id in [0, nfold) per row (host or device), or NULL for i mod nfold.
 *   results: [ngrid] -- metric = mean accuracy (classification) or mean MSE (regression) over the
 *            folds that did not fail (a training split with one class fails), pearson =
 *            mean Pearson correlation (regression; NaN when undefined), plus the cell's gamma, C,
 *            total iterations and whether every fold problem converged.
 *   cv_decision: optional fp64 [ngrid][n][n_problem] (host or device): each row's decision value
 *            from the model of the fold that held it out (n_problem = k for one-vs-rest, else 1).
 * Errors: those of svm_train, SVM_EINVAL (nfold outside [2, n], a fold id out of range, an empty
 * fold, ngrid < 1, a non-positive gamma or C). */
typedef struct svm_cv_result {
    int32_t nfold, failed;   /* folds; folds whose training split had a single class            */
    double metric;           /* mean accuracy (classification) or MSE (regression)              */
    double pearson;          /* regression: mean Pearson correlation; 0 for classification       */
    double gamma, cost;      /* the grid cell                                                     */
    int64_t iterations;      /* outer iterations summed over the cell's problems                  */
    int32_t converged;       /* 1 if every problem of the cell converged                          */
} svm_cv_result;
int svm_cross_validate(const float* X, const float* y, int64_t n, int64_t d,
                       const svm_params* params, int32_t nfold, const int32_t* fold,
                       int32_t ngrid, const double* gammas, const double* costs,
                       svm_cv_result* results, double* cv_decision);

/* ---- solver-state API: one binary problem, stepwise (parity tests and drivers) -------------
 * A solver owns the device state of one Eq. 2 instance built from (X, y, params) exactly as
 * svm_train builds it (labels: binary only -- exactly two classes, mapped as svm_train maps them).
 * Dual variables are indexed as the oracle indexes them: SVC i = row; SVR i < n is the positive
 * copy (alpha*) of row i, i >= n the negative copy (alpha) of row i - n (Eq. 1). */
typedef struct svm_solver svm_solver;

typedef struct svm_solver_stats {
    int64_t iterations;   /* outer iterations executed by the last svm_solver_run             */
    double m_up, M_low;   /* violation pair measured at the last selection (fp32 G)           */
    int32_t converged;    /* m_up - M_low <= tolerance at the last selection                   */
    int32_t last_nw;      /* |W| of the last iteration executed                                */
    int64_t last_w[16];   /* its working set (dual indices, ascending)                         */
    double last_dalpha[16]; /* alpha change of each last_w entry                               */
    int32_t last_inner;   /* inner pair steps of the last subproblem                           */
    double loop_ms;       /* device time of the last run                                       */
    int64_t cache_passes; /* iterations of the last run served by the kernel-column cache       */
} svm_solver_stats;

int svm_solver_create(const float* X, const float* y, int64_t n, int64_t d,
                      const svm_params* params, svm_solver** out);
int svm_solver_create_csr(const int64_t* indptr, const int32_t* indices, const float* data,
                          const float* y, int64_t n, int64_t d, const svm_params* params,
                          svm_solver** out);
/* m = number of dual variables (n or 2n). */
int svm_solver_size(const svm_solver* s, int64_t* m);
/* Replace (alpha, G): host or device fp64[m] and fp32[m].  alpha must lie in [0, C]. */
int svm_solver_set_state(svm_solver* s, const double* alpha, const float* G);
/* Read (alpha fp64[m], G fp32[m]); either pointer may be NULL. */
int svm_solver_get_state(const svm_solver* s, double* alpha, float* G);
/* Run up to max_iter outer iterations from the current state (selection a1, subproblem a2,
 * fused kernel-row + gradient pass a3), stopping early at tolerance.  max_iter = 0 only
 * measures the violation.  Fills *stats (may be NULL). */
int svm_solver_run(svm_solver* s, int64_t max_iter, svm_solver_stats* stats);
/* Debug view of the fused pass's kernel rows: K[i * nr + r] = K(x_i, x_rows[r]) for all n
 * training rows i, through the same dot-product and kernel code as the pass (nr <= 16). */
int svm_solver_kernel_rows(svm_solver* s, const int64_t* rows, int32_t nr, float* K);
/* Virtual ranks: subsequent svm_solver_run calls split the
 * solver's nblk CTAs into vranks ranks of nblk / vranks CTAs inside ONE launch on this GPU.  Each
 * virtual rank owns the rows its CTAs own in a one-rank launch, keeps its own exchange buffer,
 * merges its CTAs' lists, publishes one 8+8 list per rank, gathers W rows / payloads from their
 * owner rank -- the code path of a multi-GPU run.  Per-row arithmetic and the merges are exact,
 * so alpha, G and the iteration count must equal vranks = 1 bit for bit.  vranks = 1 restores
 * the one-rank launch.  SVM_EINVAL unless 1 <= vranks <= 8 and vranks divides nblk. */
int svm_solver_set_ranks(svm_solver* s, int32_t vranks);
/* Launch geometry of the solver: CTAs of the persistent kernel and training rows per CTA. */
int svm_solver_geometry(const svm_solver* s, int32_t* nblk, int64_t* rows_per_cta);
/* Pass-only diagnostic of the fused kernel-row + gradient step (a3) in its production launch
 * configuration: `passes` repetitions of { for every training row i: K(x_i, x_rows[r]) for the
 * nr <= 16 distinct rows, G_i += y_i sum_r coef[r] K_ir, new candidate keys, CTA top-8 lists },
 * with W fixed (no exchange, no subproblem).  rows: int64[nr] training-row indices, coef:
 * fp32[nr] (host or device).  *ms receives the device time of the launch (CUDA events on the
 * solver's stream).  The solver's G is modified (G += passes x the update): restore it with
 * svm_solver_set_state before training further.  Single-rank solvers only. */
int svm_solver_pass_bench(svm_solver* s, const int64_t* rows, int32_t nr, const float* coef,
                          int64_t passes, double* ms);
void svm_solver_free(svm_solver* s);

/* ---- batched solver: P binary C-SVC problems on one dense X, stepwise -------
 * The machinery svm_train uses for one-vs-rest (and svm_cross_validate for folds / grids): each
 * iteration is one k_ovr_solve launch (per problem: selection, stop test, fp64 subproblem, its 16
 * U columns) and one k_ovr_pass launch (tcgen05 D = X X_U^T for all problems at once, kernel
 * values, G update, candidates).  Y: fp32 [nprob][n] labels +-1 (host or device); 2 <= nprob <=
 * 16.  Dual variables indexed by row (as svm_solver).  svm_batch_run executes up to max_iter
 * iterations per problem from the current state (a problem stops early at tolerance) and writes
 * each problem's iteration count (may be NULL).  SVM_EINVAL when d or the shared-memory plan is
 * not covered by the batched pass. */
typedef struct svm_batch svm_batch;
int svm_batch_create(const float* X, const float* Y, int32_t nprob, int64_t n, int64_t d,
                     const svm_params* params, svm_batch** out);
int svm_batch_set_state(svm_batch* b, int32_t p, const double* alpha, const float* G);
int svm_batch_get_state(const svm_batch* b, int32_t p, double* alpha, float* G);
int svm_batch_run(svm_batch* b, int64_t max_iter, int64_t* iterations);
void svm_batch_free(svm_batch* b);

/* ---- row-sharded training over several GPUs (one process per GPU) --------------------------
 * Rank r holds training rows [row0, row0 + n_local) of an n_global-row problem (contiguous
 * blocks).  Every iteration each CTA of a rank publishes its 8+8 working-set
 * candidates into its rank's own buffer; every CTA merges the rank's lists; CTA 0 of every rank
 * then writes the rank's merged 8+8 list straight into every rank's buffer over NVLink peer
 * memory (a one-shot all-gather of one list per rank, fused into the pass); every CTA merges the
 * `world` lists identically, so all ranks pick the same W and solve the same subproblem
 * redundantly.  Working-set rows are read from their owner over
 * NVLink.  Setup is two-phase because peer mappings need an exchange of opaque handles between
 * processes, which the caller performs (e.g. torch.distributed all_gather_object):
 *   svm_shard_create   allocates this rank's state and its exported buffers;
 *   svm_shard_handle   writes SVM_SHARD_HANDLE_BYTES describing them (cudaIpc handles);
 *   svm_shard_connect  takes all `world` handles (rank-major, world * HANDLE_BYTES), maps peers;
 *   svm_shard_train    trains; every rank returns the identical model (SV rows gathered over
 *                      NVLink).  All ranks must call it; it begins with a device-side barrier.
 * y_global: labels / targets of ALL n_global rows (fp32, host or device) -- the class map must be
 * identical on every rank.  X_local: dense n_local x d (params->layout).  world = 1 is valid and
 * runs the same kernels as svm_train.  Errors: SVM_EINVAL (world > 8, rank out of range, rows
 * outside [0, n_global)), SVM_EPEER (handle mismatch or cudaIpc failure), SVM_ETIMEOUT (a peer
 * stopped publishing for 60 s), plus those of svm_train. */
#define SVM_SHARD_HANDLE_BYTES 1024
typedef struct svm_shard svm_shard;

int svm_shard_create(const float* X_local, int64_t n_local, int64_t d, int64_t row0,
                     const float* y_global, int64_t n_global, int32_t rank, int32_t world,
                     const svm_params* params, svm_shard** out);
int svm_shard_create_csr(const int64_t* indptr, const int32_t* indices, const float* data,
                         int64_t n_local, int64_t d, int64_t row0, const float* y_global,
                         int64_t n_global, int32_t rank, int32_t world, const svm_params* params,
                         svm_shard** out);
int svm_shard_handle(const svm_shard* sh, void* handle /* SVM_SHARD_HANDLE_BYTES */);
int svm_shard_connect(svm_shard* sh, const void* all_handles /* world * HANDLE_BYTES */);
int svm_shard_train(svm_shard* sh, svm_model** out);
void svm_shard_free(svm_shard* sh);

/* One-call sharded training: create + handle exchange + connect + train + free.
 * nccl_unique_id: the 128-byte ncclUniqueId rank 0 obtained (svm_nccl_unique_id) and shared with
 * every rank by the caller (e.g. torch.distributed.broadcast_object_list).  All `world` ranks call
 * it collectively with the same id; the handles are all-gathered over a communicator created from
 * the id (NCCL is loaded at first use: libnccl.so.2, the host framework's when one is loaded) and
 * destroyed before returning.  Arguments and results as svm_shard_create* / svm_shard_train:
 * every rank returns the identical model.  Errors: those of the shard API, SVM_ENCCL. */
int svm_nccl_unique_id(void* id /* 128 bytes, out */);
int svm_train_sharded(const float* X_local, int64_t n_local, int64_t d, int64_t row0,
                      const float* y_global, int64_t n_global, int32_t rank, int32_t world,
                      const void* nccl_unique_id, const svm_params* params, svm_model** out);
int svm_train_sharded_csr(const int64_t* indptr, const int32_t* indices, const float* data,
                          int64_t n_local, int64_t d, int64_t row0, const float* y_global,
                          int64_t n_global, int32_t rank, int32_t world, const void* nccl_unique_id,
                          const svm_params* params, svm_model** out);

#ifdef __cplusplus
}
#endif
#endif /* SVMB200_H */
