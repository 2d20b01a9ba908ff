// svm_internal.cuh -- device-side structures and helpers shared by the CUDA translation units of
// libsvmb200.so (the product path).  Nothing here is shared with oracle/ (the test oracle).
//
// Paper: Rgtsvm, arXiv 1706.05544 (P:n = PAPER.md line n).  The hot path is the working-set
// iteration of P:53 on the Eq. 2 dual, with eps-SVR through Eq. 1's doubled problem
// (P:59-69).  Layout and kernel design are in DESIGN.md.
#pragma once

#include <cuda.h>   // CUtensorMap (the TMA descriptor type; encoded through the runtime's driver entry point)
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#define SVM_MAX_RANKS 8
#define SVM_WS 16           // maximum |W| ("16 dual space coefficients")
#define SMO_THREADS 512     // persistent CTA size: 16 warps
#define SMO_WARPS (SMO_THREADS / 32)

// ---- kernel functions (P:77 names; S:116 formulas; e1071 parameterisation) -------------------
struct KParams {
    int32_t kernel;  // 0 linear, 1 polynomial, 2 radial, 3 sigmoid
    int32_t degree;
    float gamma;
    float coef0;
    double gamma64;  // the same parameters in fp64 for the fp64 subproblem matrix Q_WW
    double coef064;
};

// K from the fp32 dot product u.v and the squared norms |u|^2, |v|^2.  RBF uses
// |u - v|^2 = |u|^2 + |v|^2 - 2 u.v clamped at 0 (reading R11), so K <= 1.
__device__ __forceinline__ float kernel_from_dot(const KParams& kp, float dot, float nu, float nv)
{
    if (kp.kernel == 2) {
        float d2 = fmaxf(fmaf(-2.0f, dot, nu + nv), 0.0f);
        return __expf(-kp.gamma * d2);
    }
    if (kp.kernel == 0) return dot;
    float z = fmaf(kp.gamma, dot, kp.coef0);
    if (kp.kernel == 1) {
        float r = 1.0f;
        for (int e = 0; e < kp.degree; ++e) r *= z;
        return r;
    }
    return tanhf(z);
}

// fp64 kernel between two rows held in shared memory as columns a, b of a [d][16] tile;
// used for the 16x16 subproblem matrix Q_WW (direct difference for RBF, as the definition).
__device__ __forceinline__ double kernel_fp64_from(double dot_or_dist, const KParams& kp)
{
    if (kp.kernel == 2) return exp(-kp.gamma64 * dot_or_dist);
    if (kp.kernel == 0) return dot_or_dist;
    double z = kp.gamma64 * dot_or_dist + kp.coef064;
    if (kp.kernel == 1) {
        double r = 1.0;
        for (int e = 0; e < kp.degree; ++e) r *= z;
        return r;
    }
    return tanh(z);
}

// Sequential fp32 squared norm with explicit fmaf, so every unit that needs |x|^2 (layout
// kernel, CSR norms, the in-CTA recompute for working-set rows) gets bit-identical values.
__device__ __forceinline__ float sqnorm_step(float acc, float v) { return fmaf(v, v, acc); }

// ---- status byte per dual variable ---------------------------------------------------------
// bit0: y = +1;  bit1: alpha == 0 (lower bound);  bit2: alpha == C (upper bound).
#define ST_YPOS 1u
#define ST_LOW 2u
#define ST_UPP 4u

__device__ __forceinline__ bool st_in_up(uint32_t st)
{   // I_up = {y=+1, a<C} u {y=-1, a>0}
    return (st & ST_YPOS) ? !(st & ST_UPP) : !(st & ST_LOW);
}
__device__ __forceinline__ bool st_in_low(uint32_t st)
{   // I_low = {y=+1, a>0} u {y=-1, a<C}
    return (st & ST_YPOS) ? !(st & ST_LOW) : !(st & ST_UPP);
}
__host__ __device__ __forceinline__ uint8_t make_status(int y, double a, double C)
{
    return (uint8_t)((y > 0 ? ST_YPOS : 0u) | (a <= 0.0 ? ST_LOW : 0u) | (a >= C ? ST_UPP : 0u));
}

// ---- candidate keys --------------------------------------------------------------------------
// 64-bit key, larger = better: high word = order-preserving image of the fp32 score, low word =
// ~dual_index so equal scores prefer the lower index.  0 = no candidate.
__device__ __forceinline__ uint32_t ord_f32(float f)
{
    uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t u)
{
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ __forceinline__ uint64_t make_key(float score, uint64_t gidx)
{
    return ((uint64_t)ord_f32(score) << 32) | (uint64_t)(0xffffffffu - (uint32_t)gidx);
}
__device__ __forceinline__ uint64_t key_index(uint64_t key) { return 0xffffffffu - (uint32_t)key; }

// Exchange words ("LL" format: every 8-byte word carries its own 16-bit tag, so a reader never
// needs a fence or a separate flag -- it polls the words until their tags match).  Per CTA slot
// and iteration: 16 key words [tag16 | ord(score) 32 | pos16] (8 up, 8 low; pos = c * rows_per_cta
// + local row, score 0 = no candidate) and 16 x 3 payload words carrying the candidate's alpha
// (fp64), G (fp32) and status byte.
#define XW_PER_SLOT 64
// Per-rank exchange buffer = [rank level: 2 parities x SVM_MAX_RANKS x XW_RANK_SLOT words]
// followed by [local level: 2 parities x nblk CTA slots x XW_PER_SLOT words].  The local level is
// the all-to-all of the rank's own CTAs (every CTA merges the rank's nblk lists); with world > 1
// CTA 0 of every rank then publishes the rank's merged 8 + 8 list into every rank's rank level
// (2 words per candidate: [tag | ord(score) 32 | CTA slot 16] and [tag | candidate 16 | pos 16]),
// so the lists a CTA stages and merges number nblk + world, not world x nblk (SURVEY 8(e):
// one 8+8 list per rank).  Payload words stay in the owner's local level, read over NVLink.
#define XW_RANK_SLOT 32
#define XW_RANK_WORDS (2 * SVM_MAX_RANKS * XW_RANK_SLOT)
__host__ __device__ __forceinline__ uint64_t tag16_of(uint32_t tag) { return (uint64_t)(tag % 65535u + 1u) << 48; }

// Histogram of the per-iteration exchange latency (cycles): 64 bins of 512 cycles below 32768,
// then 64 bins of 4096 cycles (the last one open) -- p50 / p99 for the scaling report.
#define SMO_EXCH_BINS 128
__host__ __device__ __forceinline__ int exch_bin(uint32_t c)
{
    const uint32_t hi = (c - 32768u) >> 12;
    return c < 32768u ? (int)(c >> 9) : 64 + (int)(hi < 63u ? hi : 63u);
}
__host__ __device__ __forceinline__ double exch_bin_mid(int b)
{
    return b < 64 ? 512.0 * b + 256.0 : 32768.0 + 4096.0 * (b - 64) + 2048.0;
}

// Device-side result record of the persistent loop (written by CTA 0 of rank 0).
struct SmoInfo {
    int64_t iterations;      // iterations completed in this launch
    double m_up, M_low;      // at the last selection
    int32_t converged;
    int32_t error;           // 0, or 1 = timeout waiting for candidates
    int32_t last_nw;
    int32_t last_inner;
    int64_t last_w[SVM_WS];
    double last_dalpha[SVM_WS];
    int64_t inner_total;
    int64_t cache_lookups, cache_hits, cache_allhit;   // kernel-column cache dry run (statistics)
    int64_t phase_cycles[16]; // CTA 0: clock64 per phase (solver [0,8), worker warp 0 [8,16))
    int64_t exch_cycles;      // CTA 0, thread 0: clock64 from its publish to all slots staged
    int64_t loop_cycles;      // CTA 0, thread 0: clock64 over the whole loop (prologue excluded)
    uint32_t exch_hist[SMO_EXCH_BINS];   // per-iteration exchange cycles (exch_bin)
};

// All arguments of the persistent working-set kernel (passed by value).
struct SmoArgs {
    // local training rows [row0, row0 + n_local) of an n_global-row problem
    const float* XT;          // dense: feature-major [d][n_pad]; NULL for CSR
    const int64_t* indptr;    // CSR (local rows); NULL for dense
    const int32_t* indices;
    const float* vals;
    const float* xnorm;       // [n_pad] squared norms
    int64_t n_local, n_pad, d, row0, n_global;
    int64_t rows_per_cta;     // multiple of 4
    int32_t ncopy;            // 1 = SVC (m = n), 2 = eps-SVR (m = 2n, Eq. 1)
    int32_t rpt;              // rows per thread in the dense pass: 1, 2 or 4
    // per-dual state of the local rows, copy-major: dual (c, i) at c * n_pad + i
    double* alpha;
    float* G;
    uint8_t* status;
    double C, tol, inner_tol;
    int32_t inner_max;
    int32_t q;                // |W| requested (even, <= 16)
    KParams kp;
    // ranks (world = 1 for single-GPU training).  virt = 1: all `world` ranks run inside this
    // one launch (virtual ranks on one GPU, `nblk` CTAs each; rank r = blockIdx.x / nblk owns rows
    // [rank_row0[r], rank_row0[r + 1]) of the arrays above, which then hold ALL rows) -- the
    // multi-rank exchange, owner and peer-gather code runs exactly as across GPUs.
    int32_t rank, world, nblk, virt;
    int32_t rank_nblk[SVM_MAX_RANKS];         // CTAs of each rank
    int64_t rank_row0[SVM_MAX_RANKS + 1];
    const float* peer_XR[SVM_MAX_RANKS];      // dense row-major rows of each rank
    const float* peer_xnorm[SVM_MAX_RANKS];   // squared norms of each rank's rows
    const int64_t* peer_indptr[SVM_MAX_RANKS];
    const int32_t* peer_indices[SVM_MAX_RANKS];
    const float* peer_vals[SVM_MAX_RANKS];
    int64_t rank_rpc[SVM_MAX_RANKS];          // rows_per_cta of each rank
    uint64_t* peer_xw[SVM_MAX_RANKS];         // exchange buffers (XW_RANK_WORDS + 2 nblk XW_PER_SLOT)
    uint32_t tag0;            // epoch: this launch publishes tags tag0+1, tag0+2, ...
    int64_t max_iter;         // iterations allowed in this launch
    uint64_t timeout_ns;
    SmoInfo* info;
    int32_t x_in_smem;        // 1: this CTA's slice of X^T is staged once into shared memory
    int32_t overlap;          // 2: solver's sub-partition warps defer phase A; 1: all warps
    int32_t dbuf_rows;        // rows whose 16 dot products are buffered in shared memory
    int32_t wide;             // 1: CTA-wide bulk-copy pipeline for wide streamed rows (one row
                              //    block per consumer warp, dots in registers across all features)
    int32_t wide_kc;          //    features per pipeline stage (8 stages)
    int32_t nslice;           // > 1: phase A splits the features of each chunk into nslice items
                              //      (partials [nslice][16][dbuf_rows], summed in slice order)
    int32_t x_ring;           // streamed X through a per-lane cp.async ring (RPT >= 2)
    // pass-only diagnostic (svm_solver_pass_bench): max_iter repetitions of the fused a3 pass +
    // CTA selection with a FIXED working set (local rows pass_rows[0..pass_nr), coefficients
    // pass_c), no exchange and no subproblem -- the same device code, timed in isolation
    int32_t pass_only, pass_nr;
    const int64_t* pass_rows;
    const float* pass_c;
    // streamed dense X through the TMA engine (x_tma = 1): chunk j of a CTA (32 RPT rows x all d
    // features of X^T) is one 2D tensor copy (boxes of <= 256 features) into a tma_ns-slot
    // mbarrier ring; the warp that consumes chunk T refills its slot with chunk T + tma_ns (the ring
    // runs ahead across iterations: X does not depend on W).  xmap: 2D map over X^T [d][n_pad]
    // (dim 0 = rows, contiguous), box {32 RPT, min(d, 256)}.
    int32_t x_tma, tma_ns;
    int32_t chunk_rows;       // rows per warp work item (multiple of 4, <= 32 rpt; 0 = 32 rpt)
    int32_t qww_mma;          // 1: K_WW from the fp64 tensor-core Gram (dense X)
    // kernel-column cache (SPEC KernelRowCache S:105-110): cache_slots columns of
    // K(x_i, x_r) over the local rows ([slot][n_pad] fp32), per-CTA 4-way set-associative LRU tags
    // and stamps ([nblk][cache_slots]); 0 slots = off
    int32_t cache_slots;
    float* cache_data;
    int32_t* cache_tag;
    uint32_t* cache_stamp;
    // CSR rows in slices of 32 for the pass (layout.cu k_sell_fill): slice
    // s = g * sell_spc + c holds rows g R + 32 c + l of global CTA g (l = lane); group j of slice s
    // (4 consecutive nonzeros of every lane's row) at [(sell_gptr[s] + j) * 32 + l]: 4 u16 column
    // indices packed in a uint2 (padding past a row's end: index d, value 0), the 4 values in a
    // float4.  NULL: per-warp shared-memory staging.
    const uint2* sell_idx;
    const float4* sell_val;
    const int64_t* sell_gptr;  // [slices + 1] group offsets
    int32_t sell_spc;          // slices per CTA = ceil(rows_per_cta / 32)
    alignas(64) CUtensorMap xmap;
};

// Batched one-vs-rest: P <= 16 binary problems on the same dense X, one X pass per
// iteration for all of them.  The union U of the problems' working sets (16 slots per problem,
// column p * 16 + slot) is the B operand of a tcgen05 3xTF32 product D[rows x NU] = X_rows X_U^T.
constexpr int OVR_MAXP = 16;
constexpr int OVR_KCH = 32;   // features per K-chunk of the batched pass (two kind::f16 k-steps)
struct OvrArgs {
    const float* XT;           // [d][n_pad] feature-major
    const float* XR;           // [n][d] row-major (working-set row gathers)
    const float* xnorm;        // [n_pad]
    int64_t n, n_pad, d;
    int P;                     // problems
    double* alpha[OVR_MAXP];   // per problem [n_pad]
    float* G[OVR_MAXP];
    uint8_t* status[OVR_MAXP];
    double tol, inner_tol;
    int inner_max;
    int64_t max_iter;
    KParams kpp[OVR_MAXP];     // per problem: kernel parameters (gamma grids share the X pass)
    double Cp[OVR_MAXP];       // per problem: box bound C
    int NU;                    // 16 * P (MMA N)
    int kch, nkc;              // features per K-chunk (multiple of 8), number of chunks
    uint16_t* Uh;              // [nkc][hi | lo][NU x KCH] fp16 K-major core tiles (k_ovr_solve)
    uint16_t* XH;              // [nct][nkc][hi | lo][128 x KCH] fp16 K-major core tiles of sigma X
    float sigma, inv_sigma2;   // power-of-two operand scale and 1 / sigma^2
    float* unorm;              // [NU] |x_u|^2 (0 for empty slots)
    float* ucoef;              // [NU] c_r of slot r of problem p (0 = no update)
    uint64_t* cand;            // [P][2 sides][nct][8] per-row-tile top-8 keys
    int nct;                   // row tiles of 128 (pass CTAs)
    int32_t* done;             // [P] 1 once problem p stopped
    int64_t* iters;            // [P]
    double* mup;               // [P] m_up, M_low at the stop
    double* mlow;
    int64_t* inner_total;      // [P]
    int na, nb;                // k_ovr_pass ring depths (set at launch)
    long long* prof;           // optional [warps][3] cycle counters of CTA 0's roles (profiling)
};
int ovr_pass_smem(const OvrArgs& a);
cudaError_t launch_ovr_pass(const OvrArgs& a, cudaStream_t st);
cudaError_t launch_ovr_solve(const OvrArgs& a, cudaStream_t st);
cudaError_t ovr_prepare(OvrArgs& a, unsigned int* scratch, cudaStream_t st);
cudaError_t launch_ovr_solve_prepare(const OvrArgs& a);   // kernel attribute of k_ovr_solve
// atomicMax of max |X[0 .. count)| as float bits into *out (caller zeroes *out)
cudaError_t launch_absmax(const float* X, int64_t count, unsigned int* out, cudaStream_t st);

// Count of CUDA kernels launched by this library (svm_launch_count in the C ABI).
void svm_note_launches(int k);
// The library's private stream-ordered memory pool of the current device (capi.cu): every
// scratch buffer is allocated from it on the caller's stream and freed on that stream at the end
// of the call -- no scratch is shared between calls, threads or devices.
cudaMemPool_t svm_mem_pool();
inline cudaError_t svm_scratch_alloc(void** p, size_t bytes, cudaStream_t st)
{
    cudaMemPool_t pool = svm_mem_pool();
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}
inline int svm_device_sms()
{
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

cudaError_t launch_smo(const SmoArgs& a, int smem_bytes, cudaStream_t st);
int smo_dyn_smem_cap(const SmoArgs& a);   // dynamic shared memory the selected variant may use
void smo_l2_restore();   // after the launch's loop: the caller's persisting-L2 limit back
int smo_smem_bytes(int64_t d, int world, int nblk, int64_t x_rows);
int smo_ring_bytes(int rpt);
int smo_csr_stage_bytes();
int smo_sell_bytes(int spc, int64_t d);   // slice offsets + group masks of one CTA (SELL CSR pass)
int smo_csr_w_extra_bytes(int64_t d);
cudaError_t launch_kernel_rows(const SmoArgs& a, const int64_t* rows, int nr, float* K,
                               cudaStream_t st);
// ---- tcgen05 TF32 operands (predict.cu, the batched one-vs-rest pass in smo.cu) -------------
// K-major SWIZZLE_NONE canonical layout: core matrix = 8 rows x 4 consecutive k (16 B per row),
// at ((row / 8) * KC + k / 4) * 128 B with KC = (k extent) / 4; LBO (next k chunk) = 128 B,
// SBO (next 8-row group) = KC * 128 B.  kind::tf32 reads the top 19 bits of each fp32 operand,
// so operands are split x = hi + lo, hi = rna_tf32(x), lo = x - hi (exact, |lo| <= 2^-11 |x|).
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// x = hi + lo with hi = rna_tf32(x) (|lo| <= 2^-11 |x|, exact in fp32)
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo)
{
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
    hi = __uint_as_float(h);
    lo = x - hi;
}
__device__ __forceinline__ int kmaj_off(int r, int k, int KC) { return ((r >> 3) * KC + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }

// ---- fp16-split tensor-core operands (the batched pass in smo.cu, the d > 128 decision kernel in
// predict.cu).  x is pre-split once into an fp16 pair with a power-of-two scale sigma:
//   xs = sigma x,  h = fp16_rn(xs),  l = fp16_rn(xs - h)        (xs - h is exact in fp32)
// and D = hA hB + hA lB + lA hB (three kind::f16 MMAs, fp32 accumulation) ~= sigma^2 x.u with the
// error of the dropped lA lB term (~2^-24 relative, the 3xTF32 level); products of two 11-bit
// significands are exact in fp32.  sigma puts max|x| sigma below 2^13 (fp16 range, no overflow).
// Layout: K-major SWIZZLE_NONE core matrices of 8 rows x 8 k (128 B), KC8 = (k extent) / 8 per
// 8-row group; LBO 128 B, SBO = KC8 x 128 B; one K = 16 MMA step advances 256 B.
__device__ __forceinline__ void f16_split(float x, float sigma, uint16_t& h, uint16_t& l)
{
    const float xs = x * sigma;
    const __half hh = __float2half_rn(xs);
    const float r = xs - __half2float(hh);
    h = __half_as_ushort(hh);
    l = __half_as_ushort(__float2half_rn(r));
}
__device__ __forceinline__ int kmaj16_off_kc(int r, int k, int KC8)
{
    return ((r >> 3) * KC8 + (k >> 3)) * 64 + (r & 7) * 8 + (k & 7);
}
// sigma = 2^e with mx sigma < 2^13 (mx = max |x| over both operands), and 1 / sigma^2
inline void f16_sigma(float mx, float* sigma, float* inv_sigma2)
{
    int ex = 0;
    if (mx > 0) frexpf(mx, &ex);
    int sh = 14 - ex - 1;
    sh = sh < -100 ? -100 : (sh > 100 ? 100 : sh);
    *sigma = ldexpf(1.0f, sh);
    *inv_sigma2 = ldexpf(1.0f, -2 * sh);
}
