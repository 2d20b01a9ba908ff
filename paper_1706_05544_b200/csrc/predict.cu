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
#ifdef TC_PROFILE
#include <cstdio>
#endif
#include <cstdlib>
#include <cstring>
#include <algorithm>

namespace {

constexpr int BQ = 128, BS = 64, BK = 16, PT = 256;

// RBF epilogue of the tcgen05 decision kernels: K = exp(-g (|q|^2 + |s|^2 - 2 q.s)) evaluated as
// 2^min(a dot + (ng |s|^2 + bq), 0) with ng = -g log2(e), bq = ng |q|^2 (per query) and a = -2 ng
// times the operand scale: two FFMA, one FMNMX and one MUFU.EX2 per pair (kernel_from_dot's
// generic switch, __expf range handling and separate scalings cost ~4x the issue slots).  The
// min(., 0) is the d2 >= 0 clamp of kernel_from_dot.
struct RbfEpi {
    float a, ng, bq;
};
__device__ __forceinline__ RbfEpi rbf_epi(const KParams& kp, float dot_scale, float qn)
{
    const float ng = -kp.gamma * 1.4426950408889634f;
    return {-2.0f * ng * dot_scale, ng, ng * qn};
}
__device__ __forceinline__ float rbf_k(const RbfEpi& r, float dot, float sn)
{
    float t = fminf(fmaf(r.a, dot, fmaf(r.ng, sn, r.bq)), 0.0f), y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t));
    return y;
}

template <int NOUT>
__global__ void __launch_bounds__(PT, 2)
    k_decision(const float* __restrict__ XqT, const float* __restrict__ qnorm, int64_t nq,
               int64_t nq_pad, const float* __restrict__ SVT, const float* __restrict__ svnorm,
               int64_t nsv_pad, int64_t d, const double* __restrict__ coef, int n_out, KParams kp,
               int tiles_per_split, double* __restrict__ Fpart)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
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

// ---- tcgen05 3xTF32 variant (d <= 128): D[128 queries x 64 SVs] in TMEM ----------------------
// Operands K-major in shared memory, SWIZZLE_NONE canonical layout: core matrix = 8 rows x 4
// consecutive k (16 B per row, 128 B), at ((row / 8) * KC + k / 4) * 128 B with KC = dp / 4; the
// descriptor's LBO (next k chunk) = 128 B, SBO (next 8-row group) = KC * 128 B.  kind::tf32 reads
// the top 19 bits of each fp32 operand (truncation, measured with scripts/tc_probe.cu), so each
// operand is split x = hi + lo with hi = rna_tf32(x), lo = x - hi (exact, |lo| <= 2^-11 |x|) and
// x.w = lo.lo + lo.hi + hi.lo + hi.hi: four MMAs per k-step, fp32 accumulation in TMEM (the
// truncation of lo costs ~2^-21 relative per product).  One query per thread = one TMEM lane, so the
// epilogue (kernel value, coefficient contraction) needs no cross-thread reduction.
constexpr int TQ = 128, TS = 64;

template <int NOUT>
__global__ void __launch_bounds__(TQ, 1)
    k_decision_tc(const float* __restrict__ XqT, const float* __restrict__ qnorm, int64_t nq,
                  int64_t nq_pad, const float* __restrict__ SVT, const float* __restrict__ svnorm,
                  int64_t nsv_pad, int d, int dp, const double* __restrict__ coef, int n_out,
                  KParams kp, int tiles_per_split, double* __restrict__ Fpart)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* Ah = reinterpret_cast<float*>(smem_raw);
    float* Al = Ah + TQ * dp;
    float* Bh = Al + TQ * dp;
    float* Bl = Bh + TS * dp;
    float* sSn = Bl + TS * dp;
    float* sCoef = sSn + TS;                                   // [NOUT][TS]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sCoef + NOUT * TS);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(mbar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int KC = dp >> 2;
    const int64_t q0 = (int64_t)blockIdx.x * TQ;
    const int64_t n_tiles = nsv_pad / TS;
    const int64_t t_begin = (int64_t)blockIdx.y * tiles_per_split;
    const int64_t t_end = min(t_begin + tiles_per_split, n_tiles);

    // the CTA's 128 queries, resident for all SV tiles (hi and lo parts)
    for (int e = tid; e < dp * TQ; e += TQ) {
        const int k = e / TQ, r = e - k * TQ;
        const float x = k < d ? XqT[(int64_t)k * nq_pad + q0 + r] : 0.0f;
        float hi, lo;
        tf32_split(x, hi, lo);
        Ah[kmaj_off(r, k, KC)] = hi;
        Al[kmaj_off(r, k, KC)] = lo;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)), "r"(TS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(mbar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TS >> 3) << 17) |
                           ((uint32_t)(TQ >> 4) << 24);   // F32 accum, TF32 A/B, K-major, M128 N64
    const float qn = qnorm[q0 + tid];
    double facc[NOUT];
#pragma unroll
    for (int p = 0; p < NOUT; ++p) facc[p] = 0.0;
    uint32_t phase = 0;
    for (int64_t t = t_begin; t < t_end; ++t) {
        const int64_t s0 = t * TS;
        for (int e = tid; e < dp * TS; e += TQ) {
            const int k = e / TS, r = e - k * TS;
            const float x = k < d ? SVT[(int64_t)k * nsv_pad + s0 + r] : 0.0f;
            float hi, lo;
            tf32_split(x, hi, lo);
            Bh[kmaj_off(r, k, KC)] = hi;
            Bl[kmaj_off(r, k, KC)] = lo;
        }
        if (tid < TS) sSn[tid] = svnorm[s0 + tid];
        for (int i = tid; i < n_out * TS; i += TQ) {
            const int p = i / TS, sI = i - p * TS;
            sCoef[p * TS + sI] = (float)coef[(int64_t)p * nsv_pad + s0 + sI];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (tid == 0) {
            const uint32_t sbo = (uint32_t)KC * 128u;
            const uint32_t ah = su32(Ah), al = su32(Al), bh = su32(Bh), bl = su32(Bl);
            for (int ks = 0; ks < (dp >> 3); ++ks)
#pragma unroll
                for (int ps = 0; ps < 4; ++ps) {   // lo.lo, lo.hi, hi.lo, then hi.hi
                    const uint64_t da = umma_desc_kmajor((ps <= 1 ? al : ah) + ks * 256, sbo);
                    const uint64_t db = umma_desc_kmajor((ps == 0 || ps == 2 ? bl : bh) + ks * 256, sbo);
                    const uint32_t acc = (ks > 0 || ps > 0) ? 1u : 0u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mbar)) : "memory");
        }
        {
            uint32_t ok = 0, spins = 0;
            uint64_t t0 = 0;
            for (;;) {
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(su32(mbar)), "r"(phase) : "memory");
                if (ok) break;
                if (++spins == 1024) {   // watchdog: a lost commit must fail the launch, not hang the GPU
                    spins = 0;
                    uint64_t now;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                    if (t0 == 0) t0 = now;
                    else if (now - t0 > 5000000000ull) __trap();
                }
            }
            phase ^= 1u;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t v[TS];
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
#define TC_LD16(o) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
    : "=r"(v[o+0]), "=r"(v[o+1]), "=r"(v[o+2]), "=r"(v[o+3]), "=r"(v[o+4]), "=r"(v[o+5]), "=r"(v[o+6]), "=r"(v[o+7]), \
      "=r"(v[o+8]), "=r"(v[o+9]), "=r"(v[o+10]), "=r"(v[o+11]), "=r"(v[o+12]), "=r"(v[o+13]), "=r"(v[o+14]), "=r"(v[o+15]) : "r"(ta + o))
        TC_LD16(0); TC_LD16(16); TC_LD16(32); TC_LD16(48);
#undef TC_LD16
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int p = 0; p < NOUT; ++p) {
            if (p < n_out) {
                float part = 0.0f;
#pragma unroll
                for (int sI = 0; sI < TS; ++sI)
                    part = fmaf(sCoef[p * TS + sI], kernel_from_dot(kp, __uint_as_float(v[sI]), qn, sSn[sI]), part);
                facc[p] += (double)part;
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();   // B, the norms / coefficients and D are reused by the next tile
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (q0 + tid < nq)
        for (int p = 0; p < n_out; ++p) Fpart[((int64_t)blockIdx.y * nq + q0 + tid) * n_out + p] = facc[p];
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TS));
}

// ---- pipelined tcgen05 variant: SV tiles pre-laid-out in global memory (K-major core layout,
// [tile][hi | lo][TS * dp]), one cp.async.bulk per tile into a 2-slot ring; warp 8 lane 0 is the
// producer and MMA issuer, accumulators double-buffered in TMEM (2 x 64 columns) so tile j's MMAs
// overlap tile j-1's epilogue; 8 epilogue warps (warp w: TMEM lanes 32 (w % 4) .., columns
// 32 (w / 4) ..) ---------------------------------------------------------------------------------
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0, spins = 0;
    uint64_t t0 = 0;
    for (;;) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (ok) return;
        if (++spins == 1024) {   // watchdog: a lost stage must fail the launch, not hang the GPU
            spins = 0;
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (t0 == 0) t0 = now;
            else if (now - t0 > 5000000000ull) __trap();
        }
    }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

constexpr int TP_EPI = 16;                 // epilogue warps: TMEM lanes 32 (w % 4), columns 16 (w / 4)
constexpr int TP_THREADS = (TP_EPI + 1) * 32;
template <int NOUT>
__global__ void __launch_bounds__(TP_THREADS, 1)
    k_decision_tcp(const float* __restrict__ XqT, const float* __restrict__ qnorm, int64_t nq,
                   int64_t nq_pad, const float* __restrict__ SVtc, const float* __restrict__ svnorm,
                   int64_t nsv_pad, int d, int dp, const double* __restrict__ coef, int n_out,
                   KParams kp, int tiles_per_split, double* __restrict__ Fpart)
{
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* Ah = reinterpret_cast<float*>(smem_raw);
    float* Al = Ah + TQ * dp;
    float* Bs = Al + TQ * dp;                                   // [2 slots][hi | lo][TS * dp]
    float* sSn = Bs + 2 * 2 * TS * dp;                          // [4][TS] SV norms (ring j & 3)
    float* sCf = sSn + 4 * TS;                                  // [4][NOUT][TS] fp32 coefficients
    uint64_t* bars = reinterpret_cast<uint64_t*>(sCf + 4 * NOUT * TS);   // bfull[2] accfull[2] accfree[2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 6);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KC = dp >> 2;
    const int64_t q0 = (int64_t)blockIdx.x * TQ;
    const int64_t n_tiles = nsv_pad / TS;
    const int64_t t_begin = (int64_t)blockIdx.y * tiles_per_split;
    const int64_t t_end = min(t_begin + tiles_per_split, n_tiles);
    const int nt = (int)(t_end - t_begin);
    const uint32_t tile_bytes = (uint32_t)(2 * TS * dp * 4);
    const float* coef32 = SVtc + (size_t)n_tiles * 2 * TS * dp;   // [n_out][nsv_pad] after the tiles
    (void)coef;
    const uint32_t b_bfull = su32(bars), b_accfull = su32(bars + 2), b_accfree = su32(bars + 4);

    for (int e = tid; e < dp * TQ; e += TP_THREADS) {   // resident query tile (hi, lo)
        const int k = e / TQ, r = e - k * TQ;
        const float x = k < d ? XqT[(int64_t)k * nq_pad + q0 + r] : 0.0f;
        float hi, lo;
        tf32_split(x, hi, lo);
        Ah[kmaj_off(r, k, KC)] = hi;
        Al[kmaj_off(r, k, KC)] = lo;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)), "r"(2 * TS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_bfull + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_accfull + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_accfree + 8 * i), "r"(TP_EPI));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // query tile -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;

    if (warp == TP_EPI) {
        if (lane == 0 && nt > 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TS >> 3) << 17) |
                                   ((uint32_t)(TQ >> 4) << 24);
            const uint32_t sbo = (uint32_t)KC * 128u;
            // tile j -> B slot j & 1 and norm / coefficient slot j & 3.  Safe to overwrite: B slot
            // j & 1 once tile j - 2's MMAs completed (waited below), small slot j & 3 once tile
            // j - 4's epilogue finished (implied by the wait for tile j - 3's TMEM release)
            auto issue = [&](int j) {
                const int sl = j & 1, ss = j & 3;
                const int64_t t = t_begin + j, s0 = t * TS;
                const uint32_t bar = b_bfull + 8 * sl;
                const uint32_t bytes = tile_bytes + TS * 4 + (uint32_t)(n_out * TS * 4);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
                bulk_g2s(su32(Bs + (size_t)sl * 2 * TS * dp), SVtc + (size_t)t * 2 * TS * dp, tile_bytes, bar);
                bulk_g2s(su32(sSn + ss * TS), svnorm + s0, TS * 4, bar);
                for (int p = 0; p < n_out; ++p)
                    bulk_g2s(su32(sCf + ((size_t)ss * NOUT + p) * TS), coef32 + (int64_t)p * nsv_pad + s0, TS * 4, bar);
            };
            issue(0);
            if (nt > 1) issue(1);
#ifdef TC_PROFILE
            long long pc[4] = {0, 0, 0, 0}, pt = clock64();
#define PMARK(i) { long long _n = clock64(); pc[i] += _n - pt; pt = _n; }
#else
#define PMARK(i)
#endif
            for (int j = 0; j < nt; ++j) {
                const int sl = j & 1;
                mb_wait(b_bfull + 8 * sl, (uint32_t)((j >> 1) & 1));
                PMARK(0)
                if (j >= 2) mb_wait(b_accfree + 8 * sl, (uint32_t)(((j - 2) >> 1) & 1));   // TMEM slot drained
                PMARK(1)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t bh = su32(Bs + (size_t)sl * 2 * TS * dp), bl = bh + TS * dp * 4;
                const uint32_t ah = su32(Ah), al = su32(Al);
                const uint32_t dcol = tmem + (uint32_t)(sl * TS);
                for (int ks = 0; ks < (dp >> 3); ++ks)
#pragma unroll
                    for (int ps = 1; ps < 4; ++ps) {   // lo.hi, hi.lo, then hi.hi (lo.lo <= 2^-22: dropped)
                        const uint64_t da = umma_desc_kmajor((ps <= 1 ? al : ah) + ks * 256, sbo);
                        const uint64_t db = umma_desc_kmajor((ps == 0 || ps == 2 ? bl : bh) + ks * 256, sbo);
                        const uint32_t acc = (ks > 0 || ps > 1) ? 1u : 0u;
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(dcol), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b_accfull + 8 * sl) : "memory");
                PMARK(2)
                // the other B slot (tile j - 1) is refilled with tile j + 1 as soon as tile j - 1's
                // MMAs have completed, so the copy overlaps tile j's MMAs and tile j - 1's epilogue
                if (j >= 1 && j + 1 < nt) {
                    mb_wait(b_accfull + 8 * (sl ^ 1), (uint32_t)(((j - 1) >> 1) & 1));
                    issue(j + 1);
                }
                PMARK(3)
            }
#ifdef TC_PROFILE
            if (blockIdx.x == 0 && blockIdx.y == 0)
                printf("[tcp] producer per tile (%d tiles): wait B %.0f, wait TMEM free %.0f, issue MMAs %.0f, refill %.0f cycles\n",
                       nt, (double)pc[0] / nt, (double)pc[1] / nt, (double)pc[2] / nt, (double)pc[3] / nt);
#endif
        }
    } else {
        const int quad = warp & 3, half = warp >> 2;   // half = column quarter (16 columns)
        const float qn = qnorm[q0 + quad * 32 + lane];
        double facc[NOUT];
#pragma unroll
        for (int p = 0; p < NOUT; ++p) facc[p] = 0.0;
#ifdef TC_PROFILE
        long long ec[3] = {0, 0, 0}, et = clock64();
#define EMARK(i) { long long _n = clock64(); ec[i] += _n - et; et = _n; }
#else
#define EMARK(i)
#endif
        for (int j = 0; j < nt; ++j) {
            const int sl = j & 1;
            const int ss = j & 3;
            mb_wait(b_accfull + 8 * sl, (uint32_t)((j >> 1) & 1));
            EMARK(0)
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t v[16];
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(sl * TS + half * 16);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            EMARK(1)
            const float* sn = sSn + ss * TS + half * 16;
            if (kp.kernel == 2) {
                // RBF: kernel values once (two FFMA + FMNMX + EX2 each), then the contractions
                const RbfEpi r = rbf_epi(kp, 1.0f, qn);
                const float4* sn4 = reinterpret_cast<const float4*>(sn);
                float kv[16];
#pragma unroll
                for (int c4 = 0; c4 < 4; ++c4) {
                    const float4 s = sn4[c4];
                    kv[4 * c4 + 0] = rbf_k(r, __uint_as_float(v[4 * c4 + 0]), s.x);
                    kv[4 * c4 + 1] = rbf_k(r, __uint_as_float(v[4 * c4 + 1]), s.y);
                    kv[4 * c4 + 2] = rbf_k(r, __uint_as_float(v[4 * c4 + 2]), s.z);
                    kv[4 * c4 + 3] = rbf_k(r, __uint_as_float(v[4 * c4 + 3]), s.w);
                }
#pragma unroll
                for (int p = 0; p < NOUT; ++p) {
                    if (p < n_out) {
                        const float4* cf4 = reinterpret_cast<const float4*>(sCf + ((size_t)ss * NOUT + p) * TS + half * 16);
                        float part = 0.0f;
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) {
                            const float4 w = cf4[c4];
                            part = fmaf(w.x, kv[4 * c4 + 0], part);
                            part = fmaf(w.y, kv[4 * c4 + 1], part);
                            part = fmaf(w.z, kv[4 * c4 + 2], part);
                            part = fmaf(w.w, kv[4 * c4 + 3], part);
                        }
                        facc[p] += (double)part;
                    }
                }
            } else {
#pragma unroll
            for (int p = 0; p < NOUT; ++p) {
                if (p < n_out) {
                    const float* cf = sCf + ((size_t)ss * NOUT + p) * TS + half * 16;
                    float part = 0.0f;
#pragma unroll
                    for (int sI = 0; sI < 16; ++sI)
                        part = fmaf(cf[sI], kernel_from_dot(kp, __uint_as_float(v[sI]), qn, sn[sI]), part);
                    facc[p] += (double)part;
                }
            }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b_accfree + 8 * sl) : "memory");
            EMARK(2)
        }
#ifdef TC_PROFILE
        if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0)
            printf("[tcp] epilogue warp 0 per tile: wait acc %.0f, tmem ld %.0f, compute %.0f cycles (facc %g)\n",
                   (double)ec[0] / nt, (double)ec[1] / nt, (double)ec[2] / nt, facc[0]);
#endif
        // the four column quarters of a query are combined in a fixed order (0 + 1 + 2 + 3)
        double* red = reinterpret_cast<double*>(Bs);   // B slots are free once every tile is done
        __syncthreads();
        if (half > 0)
            for (int p = 0; p < n_out; ++p) red[((half - 1) * TQ + quad * 32 + lane) * NOUT + p] = facc[p];
        __syncthreads();
        if (half == 0 && q0 + quad * 32 + lane < nq)
            for (int p = 0; p < n_out; ++p) {
                double f = facc[p];
                for (int h = 0; h < 3; ++h) f += red[(h * TQ + quad * 32 + lane) * NOUT + p];
                Fpart[((int64_t)blockIdx.y * nq + q0 + quad * 32 + lane) * n_out + p] = f;
            }
    }
    if (warp == TP_EPI) { __syncthreads(); __syncthreads(); }   // match the epilogue warps' barriers
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TS));
}

// ---- d > 128: both operands streamed in K-chunks (fp16-split tensor-core operands, see
// svm_internal.cuh).  Query tiles of 128 rows and SV blocks of 256 (MMA N) are pre-split once per
// call into [tile][kc][hi | lo][rows x 32]; a persistent CTA walks work items (query tile, SV
// split), each a run of SV blocks.  Warp 0 lane 0 streams stages (query chunk 16 KB + SV chunk
// 32 KB) through an mbarrier ring, warp 2 lane 0 issues three kind::f16 MMAs per 16 features into
// one of two TMEM accumulators (128 x 256 fp32 each), 16 epilogue warps (TMEM lanes 32 (w % 4),
// columns 64 (w / 4 % 4)) turn the dots into kernel values and contract them with the block's
// coefficients (fp32 per block, fp64 across blocks); the four column quarters are written as
// separate partials and summed in a fixed order by k_reduce_splits (bit-reproducible).
constexpr int DF_KCH = 32, DF_SVB = 256, DF_EPI = 16;
constexpr int DF_THREADS = (3 + DF_EPI) * 32;
constexpr int DF_ATILE = 2 * 128 * DF_KCH, DF_BTILE = 2 * DF_SVB * DF_KCH;   // fp16 elements

// [tile][kc][hi | lo][R x 32] from a feature-major fp32 matrix XT[d][ld] (rows >= nrows, k >= d -> 0)
__global__ void k_split_tiles(const float* __restrict__ XT, int64_t ld, int64_t nrows, int64_t d, int R,
                              int ntiles, int nkc, float sigma, uint16_t* __restrict__ out)
{
    const int RG = R / 8;
    const int64_t total = (int64_t)ntiles * nkc * RG * (DF_KCH / 8) * 8;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int r7 = (int)(t & 7), kq = (int)((t >> 3) % (DF_KCH / 8));
        const int64_t rest = (t >> 3) / (DF_KCH / 8);
        const int rg = (int)(rest % RG);
        const int64_t tk = rest / RG;                 // tile * nkc + kc
        const int kc = (int)(tk % nkc);
        const int64_t tile = tk / nkc;
        const int r = rg * 8 + r7;
        const int64_t row = tile * R + r;
        const int64_t f0 = (int64_t)kc * DF_KCH + kq * 8;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            uint16_t h0, l0, h1, l1;
            const float x0 = (row < nrows && f0 + j < d) ? XT[(f0 + j) * ld + row] : 0.0f;
            const float x1 = (row < nrows && f0 + j + 1 < d) ? XT[(f0 + j + 1) * ld + row] : 0.0f;
            f16_split(x0, sigma, h0, l0);
            f16_split(x1, sigma, h1, l1);
            hw[j >> 1] = h0 | ((uint32_t)h1 << 16);
            lw[j >> 1] = l0 | ((uint32_t)l1 << 16);
        }
        uint16_t* base = out + (size_t)tk * 2 * R * DF_KCH;
        const int off = kmaj16_off_kc(r, kq * 8, DF_KCH / 8);
        *reinterpret_cast<uint4*>(base + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(base + R * DF_KCH + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// max |X[k][c]| over k < d, c < ncols of a feature-major [d][ld] matrix (padding columns excluded:
// they may hold stale values), as float bits into *out
__global__ void k_absmax2d(const float* __restrict__ XT, int64_t ld, int64_t ncols, int64_t d, unsigned int* out)
{
    float m = 0.0f;   // blocks stride over the feature rows, threads over the columns (no division)
    for (int64_t k = blockIdx.x; k < d; k += gridDim.x)
        for (int64_t c = threadIdx.x; c < ncols; c += blockDim.x) m = fmaxf(m, fabsf(XT[k * ld + c]));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

__device__ __forceinline__ void df_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void df_epi_bar()
{
    asm volatile("bar.sync 1, %0;" ::"n"(DF_EPI * 32) : "memory");
}
__device__ __forceinline__ void df_wait_sleep(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (ok) return;
        __nanosleep(32);
        if ((spins & 1023) == 1023) {
            uint64_t now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (t0 == 0) t0 = now;
            else if (now - t0 > 5000000000ull) __trap();
        }
    }
}

template <int NOUT>
__global__ void __launch_bounds__(DF_THREADS, 1)
    k_decision_f16(const uint16_t* __restrict__ QH, const float* __restrict__ qnorm, int64_t nq, int nqt,
                   const uint16_t* __restrict__ SH, const float* __restrict__ svnorm,
                   const float* __restrict__ coef32, int64_t nsv_ld, int nsb, int nkc, int n_out, KParams kp,
                   float isg, int nsplit, int bps, int nstage, double* __restrict__ Fpart)
{
    extern __shared__ __align__(1024) unsigned char df_smem[];
    uint16_t* As = reinterpret_cast<uint16_t*>(df_smem);                    // [NS][hi | lo][128 x 32]
    uint16_t* Bs = As + (size_t)nstage * DF_ATILE;                           // [NS][hi | lo][256 x 32]
    float* sCf = reinterpret_cast<float*>(Bs + (size_t)nstage * DF_BTILE);   // [2][NOUT][256]
    float* sSn = sCf + 2 * NOUT * DF_SVB;                                    // [2][256]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sSn + 2 * DF_SVB);          // full[8] empty[8] accf[2] acce[2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 20);
    const uint32_t b_full = su32(bars), b_empty = b_full + 64, b_accf = b_full + 128, b_acce = b_full + 144;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nitems = nqt * nsplit;
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < nstage; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_full + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_empty + 8 * i), "r"(1));
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_accf + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_acce + 8 * i), "r"(DF_EPI));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        // ---------------- producer: stage = (query chunk, SV chunk) ------------------------------
        if (lane == 0) {
            const uint32_t abytes = DF_ATILE * 2, bbytes = DF_BTILE * 2;
            int s = 0, c = 0;
            uint32_t pe = 1;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const int qt = it / nsplit, sp = it - qt * nsplit;
                const int b0 = sp * bps, b1 = min(nsb, b0 + bps);
                for (int sb = b0; sb < b1; ++sb)
                    for (int kc = 0; kc < nkc; ++kc, ++c) {
                        if (c >= nstage) mb_wait(b_empty + 8 * s, pe);
                        const uint32_t bar = b_full + 8 * s;
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(abytes + bbytes) : "memory");
                        bulk_g2s(su32(As + (size_t)s * DF_ATILE), QH + ((size_t)qt * nkc + kc) * DF_ATILE, abytes, bar);
                        bulk_g2s(su32(Bs + (size_t)s * DF_BTILE), SH + ((size_t)sb * nkc + kc) * DF_BTILE, bbytes, bar);
                        if (++s == nstage) { s = 0; pe ^= 1u; }
                    }
            }
        }
    } else if (warp == 2) {
        // ---------------- MMA issuer (lean loop: precomputed descriptors, counter slots) --------
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(DF_SVB >> 3) << 17) | (8u << 24);
            const uint32_t sbo = (DF_KCH / 8) * 128u;
            const uint64_t a0 = umma_desc_kmajor(su32(As), sbo), bd0 = umma_desc_kmajor(su32(Bs), sbo);
            const uint64_t astep = DF_ATILE * 2 / 16, bstep = DF_BTILE * 2 / 16;
            const uint64_t alo = 128 * DF_KCH * 2 / 16, blo = DF_SVB * DF_KCH * 2 / 16;
            int s = 0, j = 0;
            uint32_t pf = 0;
            for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                const int qt = it / nsplit, sp = it - qt * nsplit;
                const int b0 = sp * bps, b1 = min(nsb, b0 + bps);
                (void)qt;
                for (int sb = b0; sb < b1; ++sb, ++j) {
                    const int ab = j & 1;
                    if (j >= 2) mb_wait(b_acce + 8 * ab, (uint32_t)(((j >> 1) - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t dcol = tmem + (uint32_t)(ab * DF_SVB);
                    for (int kc = 0; kc < nkc; ++kc) {
                        mb_wait(b_full + 8 * s, pf);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint64_t ah = a0 + (uint64_t)s * astep, bh = bd0 + (uint64_t)s * bstep;
                        const uint32_t acc0 = kc > 0 ? 1u : 0u;
#pragma unroll
                        for (int ks = 0; ks < DF_KCH / 16; ++ks) {
                            const uint64_t k16 = (uint64_t)(ks * 16);
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                         ::"r"(dcol), "l"(ah + k16), "l"(bh + k16), "r"(idesc), "r"(ks > 0 ? 1u : acc0));
                            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                                         ::"r"(dcol), "l"(ah + k16), "l"(bh + blo + k16), "r"(idesc));
                            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                                         ::"r"(dcol), "l"(ah + alo + k16), "l"(bh + k16), "r"(idesc));
                        }
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b_empty + 8 * s) : "memory");
                        if (++s == nstage) { s = 0; pf ^= 1u; }
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b_accf + 8 * ab) : "memory");
                }
            }
        }
    } else if (warp >= 3) {
        // ---------------- epilogue -------------------------------------------------------------
        const int e = warp - 3, et = tid - 96;   // 0 .. 15, 0 .. 511
        const int q = warp & 3, cq = (e >> 2) & 3;   // TMEM lane quadrant, column quarter
        int j = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int qt = it / nsplit, sp = it - qt * nsplit;
            const int b0 = sp * bps, b1 = min(nsb, b0 + bps);
            const int64_t qi = (int64_t)qt * 128 + q * 32 + lane;
            const float qn = qi < nq ? qnorm[qi] : 0.0f;
            double facc[NOUT];
#pragma unroll
            for (int p = 0; p < NOUT; ++p) facc[p] = 0.0;
            // the coefficients and norms of SV block sb + 1 are loaded into registers while block
            // sb is computed (their L2 latency used to stall every block before its barrier)
            constexpr int PF = (NOUT * DF_SVB + DF_EPI * 32 - 1) / (DF_EPI * 32);
            float rcf[PF], rsn = 0.0f;
            auto load_block = [&](int sb) {
#pragma unroll
                for (int u = 0; u < PF; ++u) {
                    const int x = et + u * DF_EPI * 32, p = x / DF_SVB, c = x - p * DF_SVB;
                    rcf[u] = x < n_out * DF_SVB ? coef32[(int64_t)p * nsv_ld + (int64_t)sb * DF_SVB + c] : 0.0f;
                }
                if (et < DF_SVB) rsn = svnorm[(int64_t)sb * DF_SVB + et];
            };
            if (b0 < b1) load_block(b0);
            for (int sb = b0; sb < b1; ++sb, ++j) {
                const int ab = j & 1;
                float* cf = sCf + (size_t)ab * NOUT * DF_SVB;
                float* sn = sSn + ab * DF_SVB;
                // (slot ab was last read in block j - 2: every epilogue thread has passed the
                // barrier of block j - 1 since)
#pragma unroll
                for (int u = 0; u < PF; ++u) {
                    const int x = et + u * DF_EPI * 32;
                    if (x < n_out * DF_SVB) cf[x] = rcf[u];   // [p][DF_SVB] = x
                }
                if (et < DF_SVB) sn[et] = rsn;
                df_epi_bar();
                if (sb + 1 < b1) load_block(sb + 1);
                df_wait_sleep(b_accf + 8 * ab, (uint32_t)((j >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint32_t v[4][16];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * DF_SVB + cq * 64 + h * 16);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                                 : "=r"(v[h][0]), "=r"(v[h][1]), "=r"(v[h][2]), "=r"(v[h][3]), "=r"(v[h][4]), "=r"(v[h][5]), "=r"(v[h][6]), "=r"(v[h][7]),
                                   "=r"(v[h][8]), "=r"(v[h][9]), "=r"(v[h][10]), "=r"(v[h][11]), "=r"(v[h][12]), "=r"(v[h][13]), "=r"(v[h][14]), "=r"(v[h][15])
                                 : "r"(ta));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) df_arrive(b_acce + 8 * ab);
                if (NOUT == 1 && kp.kernel == 2) {
                    // RBF, one output: four partial sums (one per TMEM load), 16-byte smem reads
                    const RbfEpi r = rbf_epi(kp, isg, qn);
                    float ph[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float4* sn4 = reinterpret_cast<const float4*>(sn + cq * 64 + h * 16);
                        const float4* cf4 = reinterpret_cast<const float4*>(cf + cq * 64 + h * 16);
                        float acc = 0.0f;
#pragma unroll
                        for (int c4 = 0; c4 < 4; ++c4) {
                            const float4 s = sn4[c4], w = cf4[c4];
                            acc = fmaf(w.x, rbf_k(r, __uint_as_float(v[h][4 * c4 + 0]), s.x), acc);
                            acc = fmaf(w.y, rbf_k(r, __uint_as_float(v[h][4 * c4 + 1]), s.y), acc);
                            acc = fmaf(w.z, rbf_k(r, __uint_as_float(v[h][4 * c4 + 2]), s.z), acc);
                            acc = fmaf(w.w, rbf_k(r, __uint_as_float(v[h][4 * c4 + 3]), s.w), acc);
                        }
                        ph[h] = acc;
                    }
                    facc[0] += (double)((ph[0] + ph[1]) + (ph[2] + ph[3]));
                } else {
                float part[NOUT];
#pragma unroll
                for (int p = 0; p < NOUT; ++p) part[p] = 0.0f;
                auto contract = [&](auto kfun) {
#pragma unroll
                    for (int h = 0; h < 4; ++h)
#pragma unroll
                        for (int c = 0; c < 16; ++c) {
                            const int col = cq * 64 + h * 16 + c;
                            const float kv = kfun(__uint_as_float(v[h][c]), sn[col]);
#pragma unroll
                            for (int p = 0; p < NOUT; ++p)
                                if (p < n_out) part[p] = fmaf(cf[p * DF_SVB + col], kv, part[p]);
                        }
                };
                if (kp.kernel == 2) {
                    const RbfEpi r = rbf_epi(kp, isg, qn);
                    contract([&](float dot, float s) { return rbf_k(r, dot, s); });
                } else {
                    contract([&](float dot, float s) { return kernel_from_dot(kp, dot * isg, qn, s); });
                }
#pragma unroll
                for (int p = 0; p < NOUT; ++p) facc[p] += (double)part[p];
                }
            }
            if (qi < nq) {
                const int64_t count = nq * n_out;
                double* dst = Fpart + (int64_t)(sp * 4 + cq) * count + qi * n_out;
                for (int p = 0; p < n_out; ++p) dst[p] = facc[p];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// SV tiles for k_decision_tcp: [tile][hi | lo][TS * dp] in the K-major core layout
__global__ void k_coef32(const double* __restrict__ coef, int64_t count, float* __restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)coef[i];
}
__global__ void k_sv_tiles(const float* __restrict__ SVT, int64_t nsv_pad, int d, int dp, float* __restrict__ out)
{
    const int64_t total = nsv_pad * dp;
    const int KC = dp >> 2;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / nsv_pad, s = e - k * nsv_pad;
        const float x = k < d ? SVT[k * nsv_pad + s] : 0.0f;
        float hi, lo;
        tf32_split(x, hi, lo);
        const int64_t t = s / TS;
        const int r = (int)(s - t * TS);
        float* base = out + (size_t)t * 2 * TS * dp;
        base[kmaj_off(r, (int)k, KC)] = hi;
        base[TS * dp + kmaj_off(r, (int)k, KC)] = lo;
    }
}

constexpr int decision_smem(int nout)
{
    return 2 * BK * (BQ + BS) * 4 + BQ * (BS + 1) * 4 + nout * BS * 4 + (BQ + BS) * 4;
}

}  // namespace

static cudaError_t pred_decision_f16(const float* XqT, const float* qnorm, int64_t nq, int64_t nq_pad,
                                     const float* SVT, const float* svnorm, int64_t nsv, int64_t nsv_pad, int64_t d,
                                     const double* coef, int n_out, const KParams& kp, double* F, cudaStream_t st,
                                     bool any_d);

cudaError_t pred_decision(const float* XqT, const float* qnorm, int64_t nq, int64_t nq_pad,
                          const float* SVT, const float* svnorm, int64_t nsv, int64_t nsv_pad,
                          int64_t d, const double* coef, int n_out, const KParams& kp, double* F,
                          cudaStream_t st, const float* SVtc, bool f16_any_d)
{
    (void)nsv;
    if (nq <= 0) return cudaSuccess;
    if ((d > 128 || f16_any_d || getenv("SVMB200_F16_ALL")) && nsv_pad > 0) {
        const cudaError_t e = pred_decision_f16(XqT, qnorm, nq, nq_pad, SVT, svnorm, nsv, nsv_pad, d, coef, n_out, kp, F, st,
                                                f16_any_d);
        if (e != cudaErrorNotSupported) return e;
    }
    // tcgen05 3xTF32 path for d <= 128 (query tile resident in shared memory)
    const bool tc = d <= 128 && n_out <= 16 && !getenv("SVMB200_NO_TC") && nq_pad % TQ == 0 && nsv_pad % TS == 0;
    int64_t q_tiles = nq_pad / (tc ? TQ : BQ), s_tiles = nsv_pad / (tc ? TS : BS);
    if (s_tiles == 0) return cudaMemsetAsync(F, 0, sizeof(double) * nq * n_out, st);
    int64_t want = std::max<int64_t>(1, (4 * 148 + q_tiles - 1) / q_tiles);
    int splits = (int)std::min<int64_t>(want, s_tiles);
    int tps = (int)((s_tiles + splits - 1) / splits);
    splits = (int)((s_tiles + tps - 1) / tps);
    size_t need = sizeof(double) * (size_t)splits * nq * n_out;
    double* part = F;
    double* fpart = nullptr;   // per-call scratch on the caller's stream (private pool)
    if (splits > 1) {
        cudaError_t e = svm_scratch_alloc(reinterpret_cast<void**>(&fpart), need, st);
        if (e != cudaSuccess) return e;
        part = fpart;
    }
    struct StreamFree {   // the partials go back to the pool after the reduction, on `st`
        void* p;
        cudaStream_t st;
        ~StreamFree() { if (p) cudaFreeAsync(p, st); }
    } free_part{fpart, st};
    dim3 grid((unsigned)q_tiles, (unsigned)splits);
    if (tc && SVtc) {   // pipelined variant (pre-laid-out SV tiles), when its shared memory fits
        const int dp = (int)pred_tc_dp(d);
        auto tcp_smem = [&](int nout) {
            return (int)((2 * TQ * dp + 4 * TS * dp + 4 * TS) * 4 + 4 * nout * TS * 4 + 6 * 8 + 16);
        };
        const int nout_t = n_out == 1 ? 1 : 16;
        // (the final reduction reuses the B slots: 3 x 128 x nout doubles must fit 4 x 64 x dp floats)
        if (tcp_smem(nout_t) <= 227 * 1024 && 3 * TQ * nout_t * 8 <= 4 * TS * dp * 4 && !getenv("SVMB200_NO_TCP")) {
            svm_note_launches(1);
            if (n_out == 1) {
                cudaFuncSetAttribute(k_decision_tcp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tcp_smem(1));
                k_decision_tcp<1><<<grid, TP_THREADS, tcp_smem(1), st>>>(XqT, qnorm, nq, nq_pad, SVtc, svnorm, nsv_pad,
                                                                        (int)d, dp, coef, n_out, kp, tps, part);
            } else {
                cudaFuncSetAttribute(k_decision_tcp<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, tcp_smem(16));
                k_decision_tcp<16><<<grid, TP_THREADS, tcp_smem(16), st>>>(XqT, qnorm, nq, nq_pad, SVtc, svnorm, nsv_pad,
                                                                          (int)d, dp, coef, n_out, kp, tps, part);
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess || splits == 1) return e;
            int64_t count = nq * n_out;
            svm_note_launches(1);
            k_reduce_splits<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(part, splits, count, F);
            return cudaGetLastError();
        }
    }
    if (tc) {
        const int dp = (int)((d + 7) / 8 * 8);
        auto tc_smem = [&](int nout) { return (int)((2 * TQ * dp + 2 * TS * dp + TS + nout * TS) * 4 + 16); };
        cudaError_t e;
        svm_note_launches(1);
        if (n_out == 1) {
            cudaFuncSetAttribute(k_decision_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(1));
            k_decision_tc<1><<<grid, TQ, tc_smem(1), st>>>(XqT, qnorm, nq, nq_pad, SVT, svnorm, nsv_pad, (int)d, dp,
                                                        coef, n_out, kp, tps, part);
        } else {
            cudaFuncSetAttribute(k_decision_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem(16));
            k_decision_tc<16><<<grid, TQ, tc_smem(16), st>>>(XqT, qnorm, nq, nq_pad, SVT, svnorm, nsv_pad, (int)d, dp,
                                                          coef, n_out, kp, tps, part);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess || splits == 1) return e;
        int64_t count = nq * n_out;
        svm_note_launches(1);
        k_reduce_splits<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(part, splits, count, F);
        return cudaGetLastError();
    }
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

// d > 128 on tcgen05 (fp16-split operands): pre-split query / SV tiles, persistent kernel,
// partials per (split, column quarter) reduced in a fixed order.  Returns cudaErrorNotSupported when
// the configuration is not covered (the caller falls back to the SIMT kernel).
static cudaError_t pred_decision_f16(const float* XqT, const float* qnorm, int64_t nq, int64_t nq_pad,
                                     const float* SVT, const float* svnorm, int64_t nsv, int64_t nsv_pad, int64_t d,
                                     const double* coef, int n_out, const KParams& kp, double* F, cudaStream_t st,
                                     bool any_d)
{
    // d <= 128: the resident-query 3xTF32 kernel (k_decision_tcp) unless SVMB200_F16_ALL is set
    if ((d <= 128 && !any_d && !getenv("SVMB200_F16_ALL")) || n_out > 16 || getenv("SVMB200_NO_TC") || getenv("SVMB200_NO_F16"))
        return cudaErrorNotSupported;
    const int nsm = svm_device_sms();
    const int nkc = (int)((d + DF_KCH - 1) / DF_KCH);
    const int nqt = (int)((nq + 127) / 128);
    const int nsb = (int)((std::max<int64_t>(nsv, 1) + DF_SVB - 1) / DF_SVB);   // blocks of the real SVs
    const int64_t nsv_ld = (int64_t)nsb * DF_SVB;
    // SV splits: items (query tile, split) go round-robin to the nsm CTAs, so the makespan is
    // ceil(items / nsm) * bps blocks; take the split count with the best balance (c2: 3 splits,
    // 98% against 88% for the old "items >= 4 nsm" rule)
    int nsplit = 1;
    {
        double best = -1;
        for (int ns = 1; ns <= std::min(nsb, n_out > 1 ? 4 : 16); ++ns) {   // (16 outputs: partials 8 x 16 B per query per split)
            const int b = (nsb + ns - 1) / ns, nse = (nsb + b - 1) / b;
            const int64_t items = (int64_t)nqt * nse, waves = (items + nsm - 1) / nsm;
            const double eff = (double)nqt * nsb / ((double)waves * nsm * b);
            if (eff > best + 0.01) { best = eff; nsplit = nse; }
        }
    }
    const int bps = (nsb + nsplit - 1) / nsplit;
    nsplit = (nsb + bps - 1) / bps;
    const size_t qh_b = (size_t)nqt * nkc * DF_ATILE * 2, sh_b = (size_t)nsb * nkc * DF_BTILE * 2;
    const size_t cf_b = (size_t)n_out * nsv_ld * 4, sn_b = (size_t)nsv_ld * 4;
    const size_t part_b = (size_t)nsplit * 4 * nq * n_out * 8;
    // per-call scratch on the caller's stream from the library's private pool (its release
    // threshold keeps the memory mapped between calls: no OS round trip per certification)
    const size_t total = qh_b + sh_b + cf_b + sn_b + part_b + 256;
    char* buf = nullptr;
    cudaError_t e = svm_scratch_alloc(reinterpret_cast<void**>(&buf), total, st);
    if (e != cudaSuccess) return e;
    uint16_t* QH = reinterpret_cast<uint16_t*>(buf);
    uint16_t* SH = reinterpret_cast<uint16_t*>(buf + qh_b);
    float* cf = reinterpret_cast<float*>(buf + qh_b + sh_b);
    float* sn = reinterpret_cast<float*>(buf + qh_b + sh_b + cf_b);
    double* part = reinterpret_cast<double*>(buf + qh_b + sh_b + cf_b + sn_b);
    unsigned int* mx = reinterpret_cast<unsigned int*>(buf + qh_b + sh_b + cf_b + sn_b + part_b);
    // sigma from max |x| over queries and SVs (one scale for both operands)
    if ((e = cudaMemsetAsync(mx, 0, sizeof(unsigned int), st)) != cudaSuccess) goto out;
    svm_note_launches(2);
    k_absmax2d<<<4 * nsm, 256, 0, st>>>(XqT, nq_pad, nq, d, mx);
    k_absmax2d<<<4 * nsm, 256, 0, st>>>(SVT, nsv_pad, nsv, d, mx);
    if ((e = cudaGetLastError()) != cudaSuccess) goto out;
    {
        unsigned int mb = 0;
        if ((e = cudaMemcpyAsync(&mb, mx, sizeof mb, cudaMemcpyDeviceToHost, st)) != cudaSuccess) goto out;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) goto out;
        float m = 0, sigma = 1, isg = 1;
        memcpy(&m, &mb, sizeof m);
        f16_sigma(m, &sigma, &isg);
        svm_note_launches(2);
        k_split_tiles<<<8 * nsm, 256, 0, st>>>(XqT, nq_pad, nq, d, 128, nqt, nkc, sigma, QH);
        k_split_tiles<<<8 * nsm, 256, 0, st>>>(SVT, nsv_pad, nsv, d, DF_SVB, nsb, nkc, sigma, SH);
        // coefficients and norms of the nsv real SVs; the padding is 0 (not the model's padding)
        if ((e = cudaMemsetAsync(cf, 0, cf_b + sn_b, st)) != cudaSuccess) goto out;
        if (nsv > 0) {
            for (int p = 0; p < n_out; ++p) {
                k_coef32<<<(unsigned)std::min<int64_t>((nsv + 255) / 256, 148 * 16), 256, 0, st>>>(
                    coef + (int64_t)p * nsv_pad, nsv, cf + (int64_t)p * nsv_ld);
            }
            svm_note_launches(n_out - 1);
            if ((e = cudaMemcpyAsync(sn, svnorm, sizeof(float) * nsv, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) goto out;
        }
        const int nout_t = n_out == 1 ? 1 : 16;
        auto smem_for = [&](int ns) { return ns * (DF_ATILE + DF_BTILE) * 2 + (2 * nout_t * DF_SVB + 2 * DF_SVB) * 4 + 20 * 8 + 16; };
        int nstage = 2;
        while (nstage < 8 && smem_for(nstage + 1) <= 225 * 1024) ++nstage;
        const int smem = smem_for(nstage);
        const int grid = std::min(nsm, nqt * nsplit);
        svm_note_launches(1);
        if (n_out == 1) {
            cudaFuncSetAttribute(k_decision_f16<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_decision_f16<1><<<grid, DF_THREADS, smem, st>>>(QH, qnorm, nq, nqt, SH, sn, cf, nsv_ld, nsb, nkc, n_out, kp,
                                                              isg, nsplit, bps, nstage, part);
        } else {
            cudaFuncSetAttribute(k_decision_f16<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_decision_f16<16><<<grid, DF_THREADS, smem, st>>>(QH, qnorm, nq, nqt, SH, sn, cf, nsv_ld, nsb, nkc, n_out, kp,
                                                               isg, nsplit, bps, nstage, part);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) goto out;
        const int64_t count = nq * n_out;
        svm_note_launches(1);
        k_reduce_splits<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(part, nsplit * 4, count, F);
        e = cudaGetLastError();
    }
out:
    cudaFreeAsync(buf, st);
    return e;
}

int64_t pred_tc_dp(int64_t d)
{
    if (d > 128 || getenv("SVMB200_NO_TC")) return 0;
    return (d + 7) / 8 * 8;
}

int64_t pred_sv_tiles_floats(int64_t nsv_pad, int64_t d, int n_out)
{
    return 2 * nsv_pad * pred_tc_dp(d) + (int64_t)n_out * nsv_pad;
}

cudaError_t pred_sv_tiles(const float* SVT, int64_t nsv_pad, int64_t d, const double* coef, int n_out,
                          float* out, cudaStream_t st)
{
    const int64_t dp = pred_tc_dp(d);
    if (dp == 0 || nsv_pad % TS != 0) return cudaErrorInvalidValue;
    const int64_t total = nsv_pad * dp;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
    svm_note_launches(1);
    k_sv_tiles<<<blocks, 256, 0, st>>>(SVT, nsv_pad, (int)d, (int)dp, out);
    const int64_t cc = (int64_t)n_out * nsv_pad;
    svm_note_launches(1);
    k_coef32<<<(unsigned)std::min<int64_t>((cc + 255) / 256, 148 * 16), 256, 0, st>>>(coef, cc, out + 2 * total);
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
