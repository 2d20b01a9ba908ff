// predict.cu -- batched decision values f(x_q) = sum_s coef_s K(sv_s, x_q) + b (the
// "classification" half of Fig. 1's "training and predicting" times), and the same
// contraction over the training rows for the certification pass G = Q a + p (a4).
//
// One fused SIMT kernel: a 128-query x 64-SV tile of dot products is register-blocked (8 x 4 per
// thread) from feature-major operands staged in shared memory, turned into kernel values in
// registers, written once to shared memory and contracted with the coefficient tile into fp64
// per-query accumulators.  The n_q x n_SV kernel matrix never leaves the SM.  SV tiles are split
// across CTAs deterministically (per-split partial sums reduced in a fixed order), so results are
// bit-reproducible.  DESIGN.md gives the roofline (FP32-FMA + MUFU bound, not HBM bound).
#include "layout.cuh"

#include <math.h>

namespace {

constexpr int BQ = 128, BS = 64, BK = 16, PT = 256;

template <int NOUT>
__global__ void __launch_bounds__(PT, 2)
    k_decision(const float* __restrict__ XqT, const float* __restrict__ qnorm, int64_t nq,
               int64_t nq_pad, const float* __restrict__ SVT, const float* __restrict__ svnorm,
               int64_t nsv_pad, int64_t d, const double* __restrict__ coef, int n_out, KParams kp,
               int tiles_per_split, double* __restrict__ Fpart)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto sQ = reinterpret_cast<float (*)[BK][BQ]>(smem_raw);                         // [2][BK][BQ]
    auto sS = reinterpret_cast<float (*)[BK][BS]>(smem_raw + 2 * BK * BQ * 4);       // [2][BK][BS]
    auto sK = reinterpret_cast<float (*)[BS + 1]>(smem_raw + 2 * BK * (BQ + BS) * 4); // [BQ][BS+1]
    auto sCoef = reinterpret_cast<float (*)[BS]>(smem_raw + 2 * BK * (BQ + BS) * 4 + BQ * (BS + 1) * 4);
    float* sQn = reinterpret_cast<float*>(smem_raw + 2 * BK * (BQ + BS) * 4 + BQ * (BS + 1) * 4 + NOUT * BS * 4);
    float* sSn = sQn + BQ;

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;  // dots: SVs tx*4..+3, queries ty*8..+7
    const int64_t q0 = (int64_t)blockIdx.x * BQ;
    const int64_t n_sv_tiles = nsv_pad / BS;
    const int64_t t_begin = (int64_t)blockIdx.y * tiles_per_split;
    const int64_t t_end = min(t_begin + tiles_per_split, n_sv_tiles);
    const int h = tid >> 7, qa = tid & 127;  // accumulation: query qa, SV half h

    if (tid < BQ) sQn[tid] = qnorm[q0 + tid];
    double facc[NOUT];
#pragma unroll
    for (int p = 0; p < NOUT; ++p) facc[p] = 0.0;

    const int nk = (int)((d + BK - 1) / BK);
    for (int64_t t = t_begin; t < t_end; ++t) {
        const int64_t s0 = t * BS;
        __syncthreads();
        if (tid < BS) sSn[tid] = svnorm[s0 + tid];
        for (int i = tid; i < n_out * BS; i += PT) {
            int p = i / BS, s = i - p * BS;
            sCoef[p][s] = (float)coef[(int64_t)p * nsv_pad + s0 + s];
        }
        float acc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

        // staged loads: 2 float4 of the query tile + 1 float4 of the SV tile per thread
        float4 rq[2], rs;
        auto load = [&](int kc) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                int e = tid + u * PT;            // 0..511 float4 of a 16 x 128 tile
                int kk = e >> 5, qq = (e & 31) * 4;
                int64_t k = (int64_t)kc * BK + kk;
                rq[u] = k < d ? *reinterpret_cast<const float4*>(XqT + k * nq_pad + q0 + qq)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            {
                int kk = tid >> 4, ss = (tid & 15) * 4;
                int64_t k = (int64_t)kc * BK + kk;
                rs = k < d ? *reinterpret_cast<const float4*>(SVT + k * nsv_pad + s0 + ss)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        auto store = [&](int buf) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                int e = tid + u * PT;
                *reinterpret_cast<float4*>(&sQ[buf][e >> 5][(e & 31) * 4]) = rq[u];
            }
            *reinterpret_cast<float4*>(&sS[buf][tid >> 4][(tid & 15) * 4]) = rs;
        };
        load(0);
        store(0);
        __syncthreads();
        for (int kc = 0; kc < nk; ++kc) {
            const int buf = kc & 1;
            if (kc + 1 < nk) load(kc + 1);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float4 a0 = *reinterpret_cast<const float4*>(&sQ[buf][kk][ty * 8]);
                float4 a1 = *reinterpret_cast<const float4*>(&sQ[buf][kk][ty * 8 + 4]);
                float4 b = *reinterpret_cast<const float4*>(&sS[buf][kk][tx * 4]);
                float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            if (kc + 1 < nk) store(buf ^ 1);
            __syncthreads();
        }
        // kernel values -> shared tile
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                sK[ty * 8 + i][tx * 4 + j] =
                    kernel_from_dot(kp, acc[i][j], sQn[ty * 8 + i], sSn[tx * 4 + j]);
        __syncthreads();
        // contraction with the coefficient tile (fp32 over 32 SVs, fp64 across tiles)
#pragma unroll
        for (int p = 0; p < NOUT; ++p) {
            if (p < n_out) {
                float part = 0.0f;
#pragma unroll 8
                for (int s = 0; s < 32; ++s) part = fmaf(sCoef[p][h * 32 + s], sK[qa][h * 32 + s], part);
                facc[p] += (double)part;
            }
        }
    }
    // combine the two SV halves and write this split's partial sums
    __syncthreads();
    double* red = reinterpret_cast<double*>(&sK[0][0]);  // reuse: [NOUT][BQ] doubles
    if (h == 1)
        for (int p = 0; p < n_out; ++p) red[p * BQ + qa] = facc[p];
    __syncthreads();
    if (h == 0 && q0 + qa < nq) {
        for (int p = 0; p < n_out; ++p)
            Fpart[((int64_t)blockIdx.y * nq + q0 + qa) * n_out + p] = facc[p] + red[p * BQ + qa];
    }
}

__global__ void k_reduce_splits(const double* __restrict__ Fpart, int splits, int64_t count,
                                double* __restrict__ F)
{
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    double s = 0.0;
    for (int k = 0; k < splits; ++k) s += Fpart[(int64_t)k * count + t];
    F[t] = s;
}

__global__ void k_refresh_G(const double* __restrict__ F, const float* __restrict__ yv,
                            const uint8_t* __restrict__ status, int64_t n, int64_t n_pad, int ncopy,
                            double eps, float* __restrict__ G)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int c = 0; c < ncopy; ++c) {
        int64_t idx = (int64_t)c * n_pad + i;
        double y = (status[idx] & ST_YPOS) ? 1.0 : -1.0;
        double p = ncopy == 1 ? -1.0 : (c == 0 ? eps - (double)yv[i] : eps + (double)yv[i]);
        G[idx] = (float)(p + y * F[i]);
    }
}

// mode 0: regression value; 1: binary sign (labels[0] for f > 0, labels[1] for f < 0,
// first_label for f == 0); 2: one-vs-rest argmax, ties to the lowest class.
__global__ void k_finalize(const double* __restrict__ F, int64_t nq, int n_out,
                           const double* __restrict__ b, int mode, const double* __restrict__ labels,
                           double first_label, float* __restrict__ decision, float* __restrict__ out)
{
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    double best = -INFINITY;
    int arg = 0;
    for (int p = 0; p < n_out; ++p) {
        double f = F[q * n_out + p] + b[p];
        if (decision) decision[q * n_out + p] = (float)f;
        if (p == 0 || f > best) { best = f; arg = p; }
    }
    if (!out) return;
    if (mode == 0) out[q] = (float)best;
    else if (mode == 1) out[q] = (float)(best > 0.0 ? labels[0] : (best < 0.0 ? labels[1] : first_label));
    else out[q] = (float)labels[arg];
}

constexpr int decision_smem(int nout)
{
    return 2 * BK * (BQ + BS) * 4 + BQ * (BS + 1) * 4 + nout * BS * 4 + (BQ + BS) * 4;
}

}  // namespace

static double* g_fpart = nullptr;
static size_t g_fpart_bytes = 0;

cudaError_t pred_decision(const float* XqT, const float* qnorm, int64_t nq, int64_t nq_pad,
                          const float* SVT, const float* svnorm, int64_t nsv, int64_t nsv_pad,
                          int64_t d, const double* coef, int n_out, const KParams& kp, double* F,
                          cudaStream_t st)
{
    (void)nsv;
    if (nq <= 0) return cudaSuccess;
    int64_t q_tiles = nq_pad / BQ, s_tiles = nsv_pad / BS;
    if (s_tiles == 0) return cudaMemsetAsync(F, 0, sizeof(double) * nq * n_out, st);
    int64_t want = std::max<int64_t>(1, (4 * 148 + q_tiles - 1) / q_tiles);
    int splits = (int)std::min<int64_t>(want, s_tiles);
    int tps = (int)((s_tiles + splits - 1) / splits);
    splits = (int)((s_tiles + tps - 1) / tps);
    size_t need = sizeof(double) * (size_t)splits * nq * n_out;
    double* part = F;
    if (splits > 1) {
        if (need > g_fpart_bytes) {
            if (g_fpart) cudaFreeAsync(g_fpart, st);
            g_fpart = nullptr;
            g_fpart_bytes = 0;
            cudaError_t e = cudaMallocAsync(&g_fpart, need, st);
            if (e != cudaSuccess) return e;
            g_fpart_bytes = need;
        }
        part = g_fpart;
    }
    dim3 grid((unsigned)q_tiles, (unsigned)splits);
    const int smem1 = decision_smem(1), smem16 = decision_smem(16);
    cudaFuncSetAttribute(k_decision<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
    cudaFuncSetAttribute(k_decision<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem16);
    svm_note_launches(1);
    if (n_out == 1)
        k_decision<1><<<grid, PT, smem1, st>>>(XqT, qnorm, nq, nq_pad, SVT, svnorm, nsv_pad, d, coef,
                                           n_out, kp, tps, part);
    else
        k_decision<16><<<grid, PT, smem16, st>>>(XqT, qnorm, nq, nq_pad, SVT, svnorm, nsv_pad, d, coef,
                                            n_out, kp, tps, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || splits == 1) return e;
    int64_t count = nq * n_out;
    svm_note_launches(1);
    k_reduce_splits<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(part, splits, count, F);
    return cudaGetLastError();
}

cudaError_t pred_refresh_G(const double* F, const float* yv, const uint8_t* status, int64_t n,
                           int64_t n_pad, int ncopy, double eps, float* G, cudaStream_t st)
{
    svm_note_launches(1);
    k_refresh_G<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(F, yv, status, n, n_pad, ncopy, eps, G);
    return cudaGetLastError();
}

cudaError_t pred_finalize(const double* F, int64_t nq, int n_out, const double* b, int mode,
                          const double* labels, double first_label, float* decision, float* out,
                          cudaStream_t st)
{
    if (nq <= 0) return cudaSuccess;
    svm_note_launches(1);
    k_finalize<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(F, nq, n_out, b, mode, labels,
                                                            first_label, decision, out);
    return cudaGetLastError();
}
