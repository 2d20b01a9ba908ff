// layout.cu -- setup (a0) and bookkeeping kernels of the working-set path.
//   a0: the Eq. 2 instance: y, p, alpha = 0, G = p, laid out per dual in
//       copy-major order (eps-SVR's positive copy alpha* first, Eq. 1);
//       X re-laid feature-major [d][n_pad] (the streamed operand of the fused pass) with its
//       squared norms; input validation (finite values).
//   a4: violation, bias sums (sign-corrected) and dual objective reductions.
//   a5: per-row coefficients and stream compaction of the support vectors.
#include "layout.cuh"

#include <math.h>

namespace {

// ---- validation -------------------------------------------------------------------------------
__global__ void k_check_finite(const float* __restrict__ p, int64_t n, int* bad)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int local = 0;
    for (; i < n; i += stride) local |= !isfinite(p[i]);
    if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}

__global__ void k_check_csr(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                            int64_t n, int64_t d, int64_t nnz, int* bad)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t b = indptr[i], e = indptr[i + 1];
    if (b > e || b < 0 || e > nnz) { atomicOr(bad, 1); return; }
    int prev = -1;
    for (int64_t p = b; p < e; ++p) {
        int k = idx[p];
        if (k <= prev || k >= d) { atomicOr(bad, 2); return; }
        prev = k;
    }
}

// ---- X -> feature-major X^T [d][n_pad] (32x32 smem tile transpose, coalesced both sides) -------
__global__ void k_rowmajor_to_XT(const float* __restrict__ X, int64_t n, int64_t d,
                                 float* __restrict__ XT, int64_t n_pad)
{
    __shared__ float tile[32][33];
    int64_t i0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int64_t i = i0 + r, k = k0 + threadIdx.x;
        tile[r][threadIdx.x] = (i < n && k < d) ? X[i * d + k] : 0.0f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int64_t k = k0 + r, i = i0 + threadIdx.x;
        if (k < d && i < n_pad) XT[k * n_pad + i] = tile[threadIdx.x][r];
    }
}

// column-major (R / Fortran) X[k * n + i] -> X^T with padded stride (zero tail)
__global__ void k_colmajor_to_XT(const float* __restrict__ X, int64_t n, int64_t d,
                                 float* __restrict__ XT, int64_t n_pad)
{
    int64_t total = d * n_pad;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t k = t / n_pad, i = t - k * n_pad;
        XT[t] = i < n ? X[k * n + i] : 0.0f;
    }
}

// X^T [d][n_pad] -> row-major X [n][d] (used when the input was column-major).  Row tiles on
// grid.x (2^31 - 1 blocks), feature tiles on grid.y (d <= 2,097,120 features).
__global__ void k_XT_to_rowmajor(const float* __restrict__ XT, int64_t n, int64_t d, int64_t n_pad,
                                 float* __restrict__ X)
{
    __shared__ float tile[32][33];
    int64_t k0 = (int64_t)blockIdx.y * 32, i0 = (int64_t)blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int64_t k = k0 + r, i = i0 + threadIdx.x;
        tile[r][threadIdx.x] = (k < d && i < n) ? XT[k * n_pad + i] : 0.0f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int64_t i = i0 + r, k = k0 + threadIdx.x;
        if (i < n && k < d) X[i * d + k] = tile[threadIdx.x][r];
    }
}

// |x_i|^2 in feature order with fmaf (bit-identical to every other norm in the library)
__global__ void k_norms_XT(const float* __restrict__ XT, int64_t n, int64_t d, int64_t n_pad,
                           float* __restrict__ xnorm)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    float acc = 0.0f;
    if (i < n)
        for (int64_t k = 0; k < d; ++k) acc = sqnorm_step(acc, XT[k * n_pad + i]);
    xnorm[i] = acc;
}

__global__ void k_norms_csr(const int64_t* __restrict__ indptr, const float* __restrict__ vals,
                            int64_t n, int64_t n_pad, float* __restrict__ xnorm)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    float acc = 0.0f;
    if (i < n)
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) acc = sqnorm_step(acc, vals[p]);
    xnorm[i] = acc;
}

// ---- a0: alpha = 0, G = p, status (Eq. 1 / Eq. 2 linear terms) -------------
// yv: +-1 labels (SVC) or z (SVR).  Dual (c, i) lives at c * n_pad + i.
__global__ void k_init_state(const float* __restrict__ yv, int64_t n, int64_t n_pad, int ncopy,
                             double eps, double C, double* __restrict__ alpha, float* __restrict__ G,
                             uint8_t* __restrict__ status)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_pad) return;
    for (int c = 0; c < ncopy; ++c) {
        int64_t idx = (int64_t)c * n_pad + i;
        alpha[idx] = 0.0;
        if (i >= n) {                 // padding rows: never candidates (at both bounds)
            G[idx] = 0.0f;
            status[idx] = ST_LOW | ST_UPP | ST_YPOS;
            continue;
        }
        int y;
        double p;
        if (ncopy == 1) { y = yv[i] > 0.0f ? 1 : -1; p = -1.0; }          // p = -e
        else if (c == 0) { y = 1; p = eps - (double)yv[i]; }              // alpha*: eps - z
        else { y = -1; p = eps + (double)yv[i]; }                          // alpha:  eps + z
        G[idx] = (float)p;
        status[idx] = make_status(y, 0.0, C);
    }
}

// status from a given alpha (solver set_state); y recovered from the existing status
__global__ void k_status_from_alpha(const double* __restrict__ alpha, int64_t n, int64_t n_pad,
                                    int ncopy, double C, uint8_t* __restrict__ status)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int c = 0; c < ncopy; ++c) {
        int64_t idx = (int64_t)c * n_pad + i;
        int y = (status[idx] & ST_YPOS) ? 1 : -1;
        status[idx] = make_status(y, alpha[idx], C);
    }
}

// Cross-validation folds: rows whose fold id equals `held` leave the problem.
// Their status gets both bound bits (alpha = 0 and alpha = C at once, which no live variable can
// have), so they are in neither I_up nor I_low: never selected, alpha stays 0, and they add
// nothing to Q alpha, the bias, the dual or the model -- the Eq. 2 instance of the training split.
// G keeps being updated for them, so after certification y_i (G_i - p_i) is the fold model's
// decision value (without b) on the held-out row.
__global__ void k_exclude_fold(const int32_t* __restrict__ fold, int32_t held, int64_t n,
                               int64_t n_pad, int ncopy, uint8_t* __restrict__ status)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || fold[i] != held) return;
    for (int c = 0; c < ncopy; ++c) {
        const int64_t idx = (int64_t)c * n_pad + i;
        status[idx] = (uint8_t)((status[idx] & ST_YPOS) | ST_LOW | ST_UPP);
    }
}

// copy-major device state <-> dual-indexed host order (dual (c,i) <-> c*n + i)
__global__ void k_pack_state(const double* __restrict__ alpha, const float* __restrict__ G,
                             int64_t n, int64_t n_pad, int ncopy, double* __restrict__ a_out,
                             float* __restrict__ g_out)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * ncopy) return;
    int64_t c = t / n, i = t - c * n;
    if (a_out) a_out[t] = alpha[c * n_pad + i];
    if (g_out) g_out[t] = G[c * n_pad + i];
}

__global__ void k_unpack_state(const double* __restrict__ a_in, const float* __restrict__ g_in,
                               int64_t n, int64_t n_pad, int ncopy, double* __restrict__ alpha,
                               float* __restrict__ G)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * ncopy) return;
    int64_t c = t / n, i = t - c * n;
    alpha[c * n_pad + i] = a_in[t];
    G[c * n_pad + i] = g_in[t];
}

// ---- a4 reductions ------------------------------------------------------------------------------
// out[0] = m_up = max_{I_up} s, out[1] = M_low = min_{I_low} s (s = -y G, fp32 G), out[2] = sum of
// s over free duals (0 < alpha < C), out[3] = count of free duals, out[4] = sum alpha (G + p) / 2
// needs p: computed as (G - Qa) is not available, so the dual uses G and the stored p.
__device__ __forceinline__ double atomicMaxD(double* addr, double v)
{
    unsigned long long* a = (unsigned long long*)addr;
    unsigned long long old = *a, assumed;
    while (__longlong_as_double(old) < v) {
        assumed = old;
        old = atomicCAS(a, assumed, __double_as_longlong(v));
        if (old == assumed) break;
    }
    return __longlong_as_double(old);
}
__device__ __forceinline__ double atomicMinD(double* addr, double v)
{
    unsigned long long* a = (unsigned long long*)addr;
    unsigned long long old = *a, assumed;
    while (__longlong_as_double(old) > v) {
        assumed = old;
        old = atomicCAS(a, assumed, __double_as_longlong(v));
        if (old == assumed) break;
    }
    return __longlong_as_double(old);
}

__global__ void k_reduce_state(const double* __restrict__ alpha, const float* __restrict__ G,
                               const uint8_t* __restrict__ status, const float* __restrict__ yv,
                               int64_t n, int64_t n_pad, int ncopy, double eps, double C,
                               double* __restrict__ out)
{
    double up = -INFINITY, low = INFINITY, fsum = 0.0, fcnt = 0.0, dual = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * ncopy;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = t / n, i = t - c * n;
        int64_t idx = c * n_pad + i;
        uint32_t st = status[idx];
        double y = (st & ST_YPOS) ? 1.0 : -1.0;
        double g = (double)G[idx];
        double s = -y * g;
        double a = alpha[idx];
        if (st_in_up(st)) up = fmax(up, s);
        if (st_in_low(st)) low = fmin(low, s);
        if (a > 0.0 && a < C) { fsum += s; fcnt += 1.0; }
        double p = ncopy == 1 ? -1.0 : (c == 0 ? eps - (double)yv[i] : eps + (double)yv[i]);
        dual += a * (g + p);
    }
    for (int off = 16; off; off >>= 1) {
        up = fmax(up, __shfl_xor_sync(0xffffffffu, up, off));
        low = fmin(low, __shfl_xor_sync(0xffffffffu, low, off));
        fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
        fcnt += __shfl_xor_sync(0xffffffffu, fcnt, off);
        dual += __shfl_xor_sync(0xffffffffu, dual, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMaxD(out + 0, up);
        atomicMinD(out + 1, low);
        atomicAdd(out + 2, fsum);
        atomicAdd(out + 3, fcnt);
        atomicAdd(out + 4, 0.5 * dual);
    }
}

__global__ void k_init_reduce(double* out)
{
    out[0] = -INFINITY;
    out[1] = INFINITY;
    out[2] = out[3] = out[4] = 0.0;
}

// ---- a5: coefficients per training row and SV flags -----------------------------------------
// SVC coef_i = y_i alpha_i; SVR beta_i = alpha*_i - alpha_i; |coef| <= 1e-12 C -> 0.
__global__ void k_coef(const double* __restrict__ alpha, const uint8_t* __restrict__ status,
                       int64_t n, int64_t n_pad, int ncopy, double C, double* __restrict__ coef,
                       int64_t coef_stride_unused, uint8_t* __restrict__ svflag)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double c;
    if (ncopy == 1) c = ((status[i] & ST_YPOS) ? 1.0 : -1.0) * alpha[i];
    else c = alpha[i] - alpha[n_pad + i];
    if (fabs(c) <= 1e-12 * C) c = 0.0;
    coef[i] = c;
    if (c != 0.0) svflag[i] = 1;
}

// Incremental re-certification: delta = coef - coef_prev (flag where nonzero), and F += dF.
__global__ void k_coef_delta(const double* __restrict__ coef, double* __restrict__ coef_prev,
                             int64_t n, double* __restrict__ delta, uint8_t* __restrict__ flag)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double dc = coef[i] - coef_prev[i];
    delta[i] = dc;
    flag[i] = dc != 0.0 ? 1 : 0;
    coef_prev[i] = coef[i];
}
__global__ void k_add_f64(double* __restrict__ a, const double* __restrict__ b, int64_t n)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] += b[i];
}

// block-level counts of flagged rows, then scatter with host-scanned offsets
__global__ void k_count_flags(const uint8_t* __restrict__ flag, int64_t n, int32_t* __restrict__ cnt)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int v = (i < n && flag[i]) ? 1 : 0;
    int c = __syncthreads_count(v);
    if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

__global__ void k_scatter_flags(const uint8_t* __restrict__ flag, int64_t n,
                                const int64_t* __restrict__ offs, int64_t* __restrict__ out_idx)
{
    __shared__ int warp_cnt[32];
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int v = (i < n && flag[i]) ? 1 : 0;
    unsigned b = __ballot_sync(0xffffffffu, v);
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) warp_cnt[w] = __popc(b);
    __syncthreads();
    int base = 0;
    for (int k = 0; k < w; ++k) base += warp_cnt[k];
    if (v) out_idx[offs[blockIdx.x] + base + __popc(b & ((1u << lane) - 1))] = i;
}

// SV gather: SV^T [d][nsv_pad] from X^T, norms, and coef[p][nsv_pad] from per-row coefs
__global__ void k_gather_sv(const float* __restrict__ XT, int64_t n_pad, int64_t d,
                            const float* __restrict__ xnorm, const int64_t* __restrict__ sv_idx,
                            int64_t nsv, int64_t nsv_pad, float* __restrict__ SVT,
                            float* __restrict__ svnorm)
{
    // grid.y splits the features (a handful of SVs must still fill the machine)
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsv_pad) return;
    int64_t i = s < nsv ? sv_idx[s] : -1;
    for (int64_t k = blockIdx.y; k < d; k += gridDim.y) SVT[k * nsv_pad + s] = i >= 0 ? XT[k * n_pad + i] : 0.0f;
    if (blockIdx.y == 0) svnorm[s] = i >= 0 ? xnorm[i] : 0.0f;
}

// CSR rows -> dense feature-major columns [d][ld] starting at column 0 (zero-filled first)
__global__ void k_csr_to_XT(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                            const float* __restrict__ vals, const int64_t* __restrict__ rows,
                            int64_t nrows, int64_t row_base, float* __restrict__ XT, int64_t ld)
{
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nrows) return;
    int64_t i = rows ? rows[s] : row_base + s;
    for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) XT[(int64_t)idx[p] * ld + s] = vals[p];
}

__global__ void k_gather_coef(const double* __restrict__ coef_rows, const int64_t* __restrict__ sv_idx,
                              int64_t nsv, int64_t nsv_pad, double* __restrict__ coef_sv)
{
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsv_pad) return;
    coef_sv[s] = s < nsv ? coef_rows[sv_idx[s]] : 0.0;
}

// ---- cross-rank helpers for the sharded path (peer memory over NVLink) ------------------------
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// All-gather of K <= XCH_K doubles per rank: every rank writes its values into every rank's
// buffer (parity-double-buffered by tag), raises its flag there, then waits for all flags.
__global__ void k_xchg(const double* __restrict__ vals, int K, int rank, int world, XchgPeers P,
                       uint32_t tag, double* __restrict__ out, uint64_t timeout_ns, int* err)
{
    const int t = threadIdx.x;
    const int par = tag & 1;
    if (t < K)
        for (int r = 0; r < world; ++r) P.buf[r][((size_t)par * world + rank) * XCH_K + t] = vals[t];
    __threadfence_system();
    __syncthreads();
    if (t == 0)
        for (int r = 0; r < world; ++r) st_rel_sys(P.flags[r] + rank, tag);
    __shared__ int bad;
    if (t == 0) bad = 0;
    __syncthreads();
    if (t < world) {
        uint64_t t0, now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while ((int32_t)(ld_acq_sys(P.flags[rank] + t) - tag) < 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (now - t0 > timeout_ns) { bad = 1; break; }
        }
    }
    __syncthreads();
    if (bad) { if (t == 0) *err = 1; return; }
    for (int i = t; i < world * K; i += blockDim.x) {
        int r = i / K, k = i - r * K;
        out[i] = __ldcg(P.buf[rank] + ((size_t)par * world + r) * XCH_K + k);
    }
}

// Gather the global support-vector set: SV s (global order = rank-major, then local index order)
// is row svidx_r[s - off_r] of rank r; its features come from that rank's X over NVLink.
__global__ void k_gather_global_sv(SvPeers P, int64_t nsv, int64_t nsv_pad, int64_t d, int nprob,
                                   float* __restrict__ SVT, float* __restrict__ svn,
                                   double* __restrict__ coef, int64_t* __restrict__ grow)
{
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsv_pad) return;
    if (s >= nsv) {
        svn[s] = 0.0f;
        for (int p = 0; p < nprob; ++p) coef[(int64_t)p * nsv_pad + s] = 0.0;
        return;
    }
    int r = 0;
    while (r + 1 < P.world && s >= P.off[r + 1]) ++r;
    int64_t li = P.svidx[r][s - P.off[r]];
    if (P.XR[r]) {
        const float* row = P.XR[r] + li * d;
        for (int64_t k = 0; k < d; ++k) SVT[k * nsv_pad + s] = row[k];
    } else {
        for (int64_t p = P.indptr[r][li]; p < P.indptr[r][li + 1]; ++p)
            SVT[(int64_t)P.indices[r][p] * nsv_pad + s] = P.vals[r][p];
    }
    svn[s] = P.norms[r][li];
    for (int p = 0; p < nprob; ++p)
        coef[(int64_t)p * nsv_pad + s] = P.coefx[r][(int64_t)p * P.n_local[r] + li];
    if (grow) grow[s] = P.row0[r] + li;
}

// ---- CSR in slices of 32 rows for the persistent pass (SmoArgs::sell_*) ---------
// Slice s = g * spc + c holds the rows g R + 32 c + l (l < 32) of CTA g that exist (32 c + l < R
// and row < n).  Its length is the longest of those rows in groups of 4 nonzeros.
__global__ void k_sell_len(const int64_t* __restrict__ indptr, int64_t n, int64_t R, int spc,
                           int64_t ns, int64_t* __restrict__ len)
{
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const int64_t g = s / spc, c = s - g * spc;
    const int64_t r0 = g * R + 32 * c;
    const int64_t r1 = min(min(r0 + 32, g * R + R), n);
    int64_t m = 0;
    for (int64_t r = r0; r < r1; ++r) m = max(m, indptr[r + 1] - indptr[r]);
    len[s] = (m + 3) / 4;
}

// One warp per slice: lane l writes the nonzeros of its row, 4 per group, at
// [(gptr[s] + j) * 32 + l] (column indices as u16; past the row's end index d and value 0).
__global__ void k_sell_fill(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                            const float* __restrict__ vals, int64_t n, int64_t d, int64_t R, int spc,
                            int64_t ns, const int64_t* __restrict__ gptr, uint2* __restrict__ sidx,
                            float4* __restrict__ sval)
{
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int64_t g = s / spc, c = s - g * spc;
    const int64_t row = g * R + 32 * c + lane;
    const bool on = 32 * c + lane < R && row < n;
    const int64_t b = on ? indptr[row] : 0, e = on ? indptr[row + 1] : 0;
    const int64_t g0 = gptr[s], ng = gptr[s + 1] - g0;
    for (int64_t j = 0; j < ng; ++j) {
        uint32_t k[4];
        float v[4];
        for (int u = 0; u < 4; ++u) {
            const int64_t p = b + 4 * j + u;
            k[u] = p < e ? (uint32_t)idx[p] : (uint32_t)d;   // padding: feature d (mask 0)
            v[u] = p < e ? vals[p] : 0.0f;
        }
        sidx[(g0 + j) * 32 + lane] = make_uint2(k[0] | (k[1] << 16), k[2] | (k[3] << 16));
        sval[(g0 + j) * 32 + lane] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

inline unsigned nblocks(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

// ---- host launchers --------------------------------------------------------------------------
cudaError_t lay_check_finite(const float* p, int64_t n, int* d_bad, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
    svm_note_launches(1);
    k_check_finite<<<g, 256, 0, st>>>(p, n, d_bad);
    return cudaGetLastError();
}
cudaError_t lay_check_csr(const int64_t* indptr, const int32_t* idx, int64_t n, int64_t d,
                          int64_t nnz, int* d_bad, cudaStream_t st)
{
    svm_note_launches(1);
    k_check_csr<<<nblocks(n, 256), 256, 0, st>>>(indptr, idx, n, d, nnz, d_bad);
    return cudaGetLastError();
}
cudaError_t lay_sell_len(const int64_t* indptr, int64_t n, int64_t R, int spc, int64_t ns,
                         int64_t* len, cudaStream_t st)
{
    if (ns <= 0) return cudaSuccess;
    svm_note_launches(1);
    k_sell_len<<<nblocks(ns, 256), 256, 0, st>>>(indptr, n, R, spc, ns, len);
    return cudaGetLastError();
}
cudaError_t lay_sell_fill(const int64_t* indptr, const int32_t* idx, const float* vals, int64_t n,
                          int64_t d, int64_t R, int spc, int64_t ns, const int64_t* gptr, uint2* sidx,
                          float4* sval, cudaStream_t st)
{
    if (ns <= 0) return cudaSuccess;
    svm_note_launches(1);
    k_sell_fill<<<nblocks(ns * 32, 256), 256, 0, st>>>(indptr, idx, vals, n, d, R, spc, ns, gptr, sidx, sval);
    return cudaGetLastError();
}
cudaError_t lay_rowmajor_to_XT(const float* X, int64_t n, int64_t d, float* XT, int64_t n_pad,
                               cudaStream_t st)
{
    dim3 grid(nblocks(n_pad, 32), nblocks(d, 32));
    svm_note_launches(1);
    k_rowmajor_to_XT<<<grid, dim3(32, 8), 0, st>>>(X, n, d, XT, n_pad);
    return cudaGetLastError();
}
cudaError_t lay_colmajor_to_XT(const float* X, int64_t n, int64_t d, float* XT, int64_t n_pad,
                               cudaStream_t st)
{
    unsigned g = (unsigned)std::min<int64_t>((d * n_pad + 255) / 256, 65535);
    svm_note_launches(1);
    k_colmajor_to_XT<<<g, 256, 0, st>>>(X, n, d, XT, n_pad);
    return cudaGetLastError();
}
cudaError_t lay_XT_to_rowmajor(const float* XT, int64_t n, int64_t d, int64_t n_pad, float* X,
                               cudaStream_t st)
{
    dim3 grid(nblocks(n, 32), nblocks(d, 32));
    svm_note_launches(1);
    k_XT_to_rowmajor<<<grid, dim3(32, 8), 0, st>>>(XT, n, d, n_pad, X);
    return cudaGetLastError();
}
cudaError_t lay_norms_XT(const float* XT, int64_t n, int64_t d, int64_t n_pad, float* xnorm,
                         cudaStream_t st)
{
    svm_note_launches(1);
    k_norms_XT<<<nblocks(n_pad, 256), 256, 0, st>>>(XT, n, d, n_pad, xnorm);
    return cudaGetLastError();
}
cudaError_t lay_norms_csr(const int64_t* indptr, const float* vals, int64_t n, int64_t n_pad,
                          float* xnorm, cudaStream_t st)
{
    svm_note_launches(1);
    k_norms_csr<<<nblocks(n_pad, 256), 256, 0, st>>>(indptr, vals, n, n_pad, xnorm);
    return cudaGetLastError();
}
cudaError_t lay_init_state(const float* yv, int64_t n, int64_t n_pad, int ncopy, double eps,
                           double C, double* alpha, float* G, uint8_t* status, cudaStream_t st)
{
    svm_note_launches(1);
    k_init_state<<<nblocks(n_pad, 256), 256, 0, st>>>(yv, n, n_pad, ncopy, eps, C, alpha, G, status);
    return cudaGetLastError();
}
cudaError_t lay_status_from_alpha(const double* alpha, int64_t n, int64_t n_pad, int ncopy,
                                  double C, uint8_t* status, cudaStream_t st)
{
    svm_note_launches(1);
    k_status_from_alpha<<<nblocks(n, 256), 256, 0, st>>>(alpha, n, n_pad, ncopy, C, status);
    return cudaGetLastError();
}
cudaError_t lay_exclude_fold(const int32_t* fold, int32_t held, int64_t n, int64_t n_pad,
                             int ncopy, uint8_t* status, cudaStream_t st)
{
    svm_note_launches(1);
    k_exclude_fold<<<nblocks(n, 256), 256, 0, st>>>(fold, held, n, n_pad, ncopy, status);
    return cudaGetLastError();
}
cudaError_t lay_pack_state(const double* alpha, const float* G, int64_t n, int64_t n_pad,
                           int ncopy, double* a_out, float* g_out, cudaStream_t st)
{
    svm_note_launches(1);
    k_pack_state<<<nblocks(n * ncopy, 256), 256, 0, st>>>(alpha, G, n, n_pad, ncopy, a_out, g_out);
    return cudaGetLastError();
}
cudaError_t lay_unpack_state(const double* a_in, const float* g_in, int64_t n, int64_t n_pad,
                             int ncopy, double* alpha, float* G, cudaStream_t st)
{
    svm_note_launches(1);
    k_unpack_state<<<nblocks(n * ncopy, 256), 256, 0, st>>>(a_in, g_in, n, n_pad, ncopy, alpha, G);
    return cudaGetLastError();
}
cudaError_t lay_reduce_state(const double* alpha, const float* G, const uint8_t* status,
                             const float* yv, int64_t n, int64_t n_pad, int ncopy, double eps,
                             double C, double* d_out5, cudaStream_t st)
{
    svm_note_launches(1);
    k_init_reduce<<<1, 1, 0, st>>>(d_out5);
    unsigned g = (unsigned)std::min<int64_t>((n * ncopy + 255) / 256, 1184);
    svm_note_launches(1);
    k_reduce_state<<<g, 256, 0, st>>>(alpha, G, status, yv, n, n_pad, ncopy, eps, C, d_out5);
    return cudaGetLastError();
}
cudaError_t lay_coef(const double* alpha, const uint8_t* status, int64_t n, int64_t n_pad,
                     int ncopy, double C, double* coef, uint8_t* svflag, cudaStream_t st)
{
    svm_note_launches(1);
    k_coef<<<nblocks(n, 256), 256, 0, st>>>(alpha, status, n, n_pad, ncopy, C, coef, 0, svflag);
    return cudaGetLastError();
}
cudaError_t lay_coef_delta(const double* coef, double* coef_prev, int64_t n, double* delta,
                           uint8_t* flag, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    svm_note_launches(1);
    k_coef_delta<<<nblocks(n, 256), 256, 0, st>>>(coef, coef_prev, n, delta, flag);
    return cudaGetLastError();
}
cudaError_t lay_add_f64(double* a, const double* b, int64_t n, cudaStream_t st)
{
    if (n <= 0) return cudaSuccess;
    svm_note_launches(1);
    k_add_f64<<<nblocks(n, 256), 256, 0, st>>>(a, b, n);
    return cudaGetLastError();
}
cudaError_t lay_count_flags(const uint8_t* flag, int64_t n, int32_t* cnt, int* nblk_out,
                            cudaStream_t st)
{
    *nblk_out = (int)nblocks(n, 1024);
    svm_note_launches(1);
    k_count_flags<<<*nblk_out, 1024, 0, st>>>(flag, n, cnt);
    return cudaGetLastError();
}
cudaError_t lay_scatter_flags(const uint8_t* flag, int64_t n, const int64_t* offs, int64_t* out,
                              cudaStream_t st)
{
    svm_note_launches(1);
    k_scatter_flags<<<nblocks(n, 1024), 1024, 0, st>>>(flag, n, offs, out);
    return cudaGetLastError();
}
cudaError_t lay_gather_sv(const float* XT, int64_t n_pad, int64_t d, const float* xnorm,
                          const int64_t* sv_idx, int64_t nsv, int64_t nsv_pad, float* SVT,
                          float* svnorm, cudaStream_t st)
{
    svm_note_launches(1);
    const unsigned gx = (unsigned)nblocks(nsv_pad, 256);
    const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(d, (4 * 148 + gx - 1) / gx));
    k_gather_sv<<<dim3(gx, gy), 256, 0, st>>>(XT, n_pad, d, xnorm, sv_idx, nsv, nsv_pad, SVT, svnorm);
    return cudaGetLastError();
}
cudaError_t lay_csr_to_XT(const int64_t* indptr, const int32_t* idx, const float* vals,
                          const int64_t* rows, int64_t nrows, int64_t row_base, float* XT,
                          int64_t ld, cudaStream_t st)
{
    if (nrows <= 0) return cudaSuccess;
    svm_note_launches(1);
    k_csr_to_XT<<<nblocks(nrows, 256), 256, 0, st>>>(indptr, idx, vals, rows, nrows, row_base, XT, ld);
    return cudaGetLastError();
}
cudaError_t lay_gather_coef(const double* coef_rows, const int64_t* sv_idx, int64_t nsv,
                            int64_t nsv_pad, double* coef_sv, cudaStream_t st)
{
    svm_note_launches(1);
    k_gather_coef<<<nblocks(nsv_pad, 256), 256, 0, st>>>(coef_rows, sv_idx, nsv, nsv_pad, coef_sv);
    return cudaGetLastError();
}

cudaError_t lay_xchg(const double* vals, int K, int rank, int world, const XchgPeers& P,
                     uint32_t tag, double* out, uint64_t timeout_ns, int* err, cudaStream_t st)
{
    svm_note_launches(1);
    k_xchg<<<1, 64, 0, st>>>(vals, K, rank, world, P, tag, out, timeout_ns, err);
    return cudaGetLastError();
}
cudaError_t lay_gather_global_sv(const SvPeers& P, int64_t nsv, int64_t nsv_pad, int64_t d,
                                 int nprob, float* SVT, float* svn, double* coef, int64_t* grow,
                                 cudaStream_t st)
{
    svm_note_launches(1);
    k_gather_global_sv<<<nblocks(nsv_pad, 128), 128, 0, st>>>(P, nsv, nsv_pad, d, nprob, SVT, svn,
                                                              coef, grow);
    return cudaGetLastError();
}
