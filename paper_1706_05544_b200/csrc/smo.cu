// smo.cu -- the persistent working-set kernel: the hot loop of Rgtsvm's optimizer.
//
// One cooperative launch runs the whole loop of P:53 ("iteratively optimizing 16 heuristically
// selected dual space coefficients ... until convergence").  Every CTA owns a contiguous slice of
// training rows and, per iteration:
//   a1  merges the 8+8 candidates every CTA (of every rank) published into the working set W
//       ("picking 16 dual space coefficients based on which partial derivatives ... are the
//       largest, subject to dual space constraints") -- redundantly and identically
//       in every CTA, so no CTA ever waits on a single solver CTA;
//   a2  solves the |W|-variable subproblem in fp64 on warp 0 ("optimized based on the local
//       gradient"; P:69 for eps-SVR) WHILE the other 15 warps already form the kernel-row
//       dot products x_i . X_W for their rows;
//   a3  finishes the fused pass G_i += y_i sum_r c_r K(x_i, x_r) ("calculating the gradient for
//       all dual space coefficients"; "the responses terms are updated"), writing the
//       new up/low scores to shared memory -- the n x |W| kernel block is never stored;
//   and writes its CTA top-8 up / top-8 low candidates as self-tagged 8-byte words into every
//   rank's receive buffer (the one-shot all-gather of SURVEY 8(e), fused into the pass; no fence,
//   no flag: readers poll the words' tags).
// Measured B200 latencies that shaped this (scripts/ubench.cu): REDUX 22 cycles, SHFL 30, LDS 54,
// L2 load ~290, __threadfence ~800-1100, __threadfence_system ~1700-3100, flag round trip ~3000.
// DESIGN.md has the layout, the roofline and what differs from the paper's GTSVM design.
#include "svm_internal.cuh"

#include <cuda_fp16.h>

#include <float.h>
#include <math.h>

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SOLVER_WARP = SMO_WARPS - 1;
// X_W^T row stride in floats: dense reads broadcast one feature per warp (16 is fine); CSR reads
// 32 random features per warp, so the stride is padded to 20 floats (80 B = 5 x 16 B, coprime
// with the 8 16-byte bank groups) -- with 16 all lanes fell into two bank groups (16-way conflict).
constexpr int WSTR_CSR = 20;
// CSR: the 16-bit group mask of X_W^T row k lives in one of the row's 4 padding words, chosen so
// that 32 random rows hit 32 different banks (20 k mod 32 alone takes only 8 values)
__device__ __forceinline__ int csr_mask_slot(int k) { return k * WSTR_CSR + 16 + ((k >> 3) & 3); }

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p, bool sys)
{
    uint64_t v;
    if (sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v, bool sys)
{
    if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 64-bit warp max from two 32-bit REDUX reductions (all lanes participate).
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k)
{
    uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    uint32_t mh = __reduce_max_sync(FULL, hi);
    uint32_t ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    return ((uint64_t)mh << 32) | ml;
}

__device__ __forceinline__ float exp2f_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Order-preserving map of fp64 to u64 (exact, so argmax over keys == argmax over values).
__device__ __forceinline__ uint64_t mono64(double x)
{
    uint64_t u = (uint64_t)__double_as_longlong(x + 0.0);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unmono64(uint64_t u)
{
    return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}

template <int RPT>
__device__ __forceinline__ void zero_acc(float (&acc)[RPT][SVM_WS])
{
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
        for (int r = 0; r < SVM_WS; ++r) acc[j][r] = 0.0f;
}

// Dense kernel-row dot products acc[j][r] = x_{li+j} . x_{W_r} for RPT consecutive rows.  X^T is
// feature-major with row stride `ld` (global [d][n_pad], or the CTA's slice staged in shared
// memory); X_W^T is [d][16] in shared memory, read with 4 broadcast LDS.128 per feature.
// acc[0..15] += x * w[0..15] as eight packed FFMA2 (sm_100): each lane of the pair rounds exactly
// like fmaf, so the result is bit-identical to sixteen scalar FMAs at half the issue slots.
__device__ __forceinline__ void fma_row16_scalar(float x, const float4 (&wv)[4], float* acc)
{
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        acc[4 * q + 0] = fmaf(x, wv[q].x, acc[4 * q + 0]);
        acc[4 * q + 1] = fmaf(x, wv[q].y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(x, wv[q].z, acc[4 * q + 2]);
        acc[4 * q + 3] = fmaf(x, wv[q].w, acc[4 * q + 3]);
    }
}
__device__ __forceinline__ void fma_row16(float x, const float4 (&wv)[4], float* acc)
{
    const float2 xx = make_float2(x, x);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 lo = __ffma2_rn(xx, make_float2(wv[q].x, wv[q].y), make_float2(acc[4 * q], acc[4 * q + 1]));
        const float2 hi = __ffma2_rn(xx, make_float2(wv[q].z, wv[q].w), make_float2(acc[4 * q + 2], acc[4 * q + 3]));
        acc[4 * q] = lo.x;
        acc[4 * q + 1] = lo.y;
        acc[4 * q + 2] = hi.x;
        acc[4 * q + 3] = hi.y;
    }
}

// CSR: acc[0..15] += x * X_W^T[k][0..15] reading only the 4-row groups of X_W with a nonzero at
// feature k (16-bit mask m in the row's padding word, set while X_W is staged).  X_W rows are as
// sparse as X (c5: ~1.6 of 16 nonzero), so most groups are skipped; a skipped group would add
// x * 0, which leaves acc unchanged, so the result equals the dense update.
__device__ __forceinline__ void fma_row16_masked(float x, const float4* w4k, uint32_t m, float* acc)
{
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (m & (0xFu << (4 * q))) {
            const float4 w = w4k[q];
            const float2 xx = make_float2(x, x);
            const float2 lo = __ffma2_rn(xx, make_float2(w.x, w.y), make_float2(acc[4 * q], acc[4 * q + 1]));
            const float2 hi = __ffma2_rn(xx, make_float2(w.z, w.w), make_float2(acc[4 * q + 2], acc[4 * q + 3]));
            acc[4 * q] = lo.x;
            acc[4 * q + 1] = lo.y;
            acc[4 * q + 2] = hi.x;
            acc[4 * q + 3] = hi.y;
        }
    }
}

// Four rows at once with packed FFMA2, W loaded one float4 (4 columns) at a time so that only 4 W
// registers are live: acc[j][c] += x_j * w_c for j < 4, c < 16.  Per lane each FFMA2 half rounds
// exactly like fmaf, so the sums are bit-identical to fma_row16_scalar / fma_row16.
__device__ __forceinline__ void fma_rows4_x16(const float (&x)[4], const float4* w4k, float (&acc)[4][SVM_WS])
{
    float2 xx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xx[j] = make_float2(x[j], x[j]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 w = w4k[q];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 lo = __ffma2_rn(xx[j], make_float2(w.x, w.y), make_float2(acc[j][4 * q], acc[j][4 * q + 1]));
            const float2 hi = __ffma2_rn(xx[j], make_float2(w.z, w.w), make_float2(acc[j][4 * q + 2], acc[j][4 * q + 3]));
            acc[j][4 * q] = lo.x;
            acc[j][4 * q + 1] = lo.y;
            acc[j][4 * q + 2] = hi.x;
            acc[j][4 * q + 3] = hi.y;
        }
    }
}

template <int RPT>
__device__ __forceinline__ void dots_dense(const float* __restrict__ xcol, int64_t ld, int d,
                                           bool active, const float* sXW,
                                           float (&acc)[RPT][SVM_WS])
{
    zero_acc<RPT>(acc);
    if (!active) return;
    const float* p = xcol;
    const float4* w4 = reinterpret_cast<const float4*>(sXW);
#pragma unroll 8
    for (int k = 0; k < d; ++k) {
        float x[RPT];
        if constexpr (RPT == 4) {
            float4 v = *reinterpret_cast<const float4*>(p);
            x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
        } else if constexpr (RPT == 2) {
            float2 v = *reinterpret_cast<const float2*>(p);
            x[0] = v.x; x[1] = v.y;
        } else {
            x[0] = *p;
        }
        p += ld;
        float4 wv[4] = {w4[4 * k], w4[4 * k + 1], w4[4 * k + 2], w4[4 * k + 3]};
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            if constexpr (RPT == 4) fma_row16_scalar(x[j], wv, acc[j]);   // pairs would spill
            else fma_row16(x[j], wv, acc[j]);
        }
    }
}

#ifndef SMO_PF4
#define SMO_PF4 8    // features in flight per lane at 4 rows per thread (64 B each; 16 measured slower)
#endif
// Streamed X (global): each lane keeps a private ring of PF_X feature slots in shared memory,
// filled by cp.async (one commit group per feature), so PF_X features of its rows are in flight
// without holding registers -- with 64 accumulators per thread ptxas keeps only ~2 plain loads
// in flight, which left the streamed pass latency-bound.
template <int RPT>
__host__ __device__ constexpr int pf_x() { return RPT == 1 ? 16 : (RPT == 4 ? SMO_PF4 : 8); }  // X in flight per warp: 2-8 KB
template <int RPT>
__device__ __forceinline__ void cp_async_x(uint32_t dst, const float* src)
{
#ifdef SMO_EXP_NOX   // diagnostic build (bound experiments): no X loads, FMAs on stale ring data
    return;
#endif
    if constexpr (RPT == 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    else if constexpr (RPT == 2)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int RPT>
__device__ __forceinline__ void x_fma_slot(uint32_t sa, const float4* w4k, float (&acc)[RPT][SVM_WS])
{
    float x[RPT];
    if constexpr (RPT == 4) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(sa) : "memory");
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else if constexpr (RPT == 2) {
        float2 v;
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(sa) : "memory");
        x[0] = v.x; x[1] = v.y;
    } else {
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[0]) : "r"(sa) : "memory");
    }
    if constexpr (RPT == 4) {
#ifdef SMO_EXP_NOFMA   // diagnostic build (bound experiments): stream X, no dot FMAs
        for (int j = 0; j < 4; ++j) acc[j][0] += x[j];
#else
        fma_rows4_x16(x, w4k, acc);
#endif
    } else {
        float4 wv[4] = {w4k[0], w4k[1], w4k[2], w4k[3]};
#pragma unroll
        for (int j = 0; j < RPT; ++j) fma_row16(x[j], wv, acc[j]);
    }
}

// Streamed X: feature k of the lane's rows sits in ring slot k mod PF_X (one cp.async commit group
// per feature, PF_X features in flight).  Features [0, d - PF_X) refill their slot with feature
// k + PF_X; the main part runs in blocks of PF_X with compile-time slot offsets and the source
// pointer advanced by ld (no index arithmetic on the FMA path).
template <int RPT>
__device__ __forceinline__ void dots_dense_async(const float* __restrict__ xcol, int64_t ld, int d,
                                                 bool active, const float* sXW, uint32_t ring,
                                                 float (&acc)[RPT][SVM_WS])
{
    zero_acc<RPT>(acc);
    if (!active) return;
    constexpr uint32_t SLOT = 32u * 4u * RPT;  // bytes per slot across the warp
    constexpr int PF_X = pf_x<RPT>();
    const float4* w4 = reinterpret_cast<const float4*>(sXW);
    const float* src = xcol;
#pragma unroll
    for (int f = 0; f < PF_X; ++f) {
        if (f < d) cp_async_x<RPT>(ring + f * SLOT, src);
        src += ld;
        cp_async_commit();
    }
    int k = 0;
    for (; k + 2 * PF_X <= d; k += PF_X) {   // every feature of the block refills its slot
#pragma unroll
        for (int u = 0; u < PF_X; ++u) {
            cp_async_wait<PF_X - 1>();
            x_fma_slot<RPT>(ring + u * SLOT, w4 + 4 * (k + u), acc);
            cp_async_x<RPT>(ring + u * SLOT, src);
            src += ld;
            cp_async_commit();
        }
    }
#pragma unroll 2
    for (; k < d; ++k) {   // the last < 2 PF_X features: refill while features remain
        cp_async_wait<PF_X - 1>();
        const uint32_t sa = ring + (uint32_t)(k & (PF_X - 1)) * SLOT;
        x_fma_slot<RPT>(sa, w4 + 4 * k, acc);
        if (k + PF_X < d) {
            cp_async_x<RPT>(sa, src);
            src += ld;
        }
        cp_async_commit();
    }
    cp_async_wait<0>();
}

// Dense kernel-row dot products from a TMA-staged chunk tile [d][CH] (CH = 32 RPT rows, lane l
// owns rows RPT l .. RPT l + RPT - 1): one conflict-free LDS per feature for the lane's rows plus
// the 4 broadcast LDS.128 of X_W, then 16 RPT FMAs (the same order as dots_dense: bit-identical).
template <int RPT>
__device__ __forceinline__ void dots_tile(const float* tile, int d, int lane, const float* sXW,
                                          float (&acc)[RPT][SVM_WS])
{
    zero_acc<RPT>(acc);
    constexpr int CH = 32 * RPT;
    const float* p = tile + lane * RPT;
    const float4* w4 = reinterpret_cast<const float4*>(sXW);
#pragma unroll 4
    for (int k = 0; k < d; ++k) {
        float x[RPT];
        if constexpr (RPT == 4) {
            const float4 v = *reinterpret_cast<const float4*>(p + k * CH);
            x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
        } else if constexpr (RPT == 2) {
            const float2 v = *reinterpret_cast<const float2*>(p + k * CH);
            x[0] = v.x; x[1] = v.y;
        } else {
            x[0] = p[k * CH];
        }
        float4 wv[4] = {w4[4 * k], w4[4 * k + 1], w4[4 * k + 2], w4[4 * k + 3]};
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            if constexpr (RPT == 4) fma_row16_scalar(x[j], wv, acc[j]);
            else fma_row16(x[j], wv, acc[j]);
        }
    }
}

// CSR kernel-row dot products for one row: sum over its nnz of v * X_W^T[col][r].
__device__ __forceinline__ void dots_csr(const int64_t* __restrict__ indptr,
                                         const int32_t* __restrict__ indices,
                                         const float* __restrict__ vals, int64_t li, bool active,
                                         const float* sXW, float (&acc)[1][SVM_WS])
{
    zero_acc<1>(acc);
    if (!active) return;
    const float4* w4 = reinterpret_cast<const float4*>(sXW);
    int64_t b = __ldg(indptr + li), e = __ldg(indptr + li + 1);
    for (int64_t p = b; p < e; ++p) {
        int k = __ldg(indices + p);
        float v = __ldg(vals + p);
        const uint32_t m = __float_as_uint(sXW[csr_mask_slot(k)]);
        fma_row16_masked(v, w4 + 5 * k, m, acc[0]);
    }
}

// CSR pass with per-warp staging: the 32 rows of a chunk own one contiguous nonzero range
// [indptr[r0], indptr[r0 + 32]); the warp loads it coalesced into shared memory, then every
// lane walks its own row from there (no dependent global loads on the FMA chain).  Ranges
// larger than the buffer fall back to direct loads.
constexpr int CSR_CAP = 1472;  // nonzeros per warp stage (c5: 32 rows x 40 +- 6 nnz: 1280 +- 34; beyond -> direct loads)
__device__ __forceinline__ void dots_csr_staged(const int64_t* __restrict__ indptr,
                                                const int32_t* __restrict__ indices,
                                                const float* __restrict__ vals, int64_t li0_warp,
                                                int64_t row_end, int lane, uint16_t* st_idx,
                                                float* st_val, const float* sXW,
                                                float (&acc)[1][SVM_WS])
{
    zero_acc<1>(acc);
    const int64_t li = li0_warp + lane;
    const int64_t rlast = min(li0_warp + 32, row_end);
    if (li0_warp >= row_end) return;
    const int64_t z0 = __ldg(indptr + li0_warp), z1 = __ldg(indptr + rlast);
    const bool active = li < row_end;
    int64_t b = 0, e = 0;
    if (active) { b = __ldg(indptr + li); e = __ldg(indptr + li + 1); }
    if (z1 - z0 > CSR_CAP) {  // rare: direct path
        dots_csr(indptr, indices, vals, li, active, sXW, acc);
        return;
    }
    // 16 (index, value) loads in flight per lane before the shared-memory stores: the stage is a
    // few memory round trips, not one per 32 nonzeros
    const int cnt = (int)(z1 - z0);
    for (int base = 0; base < cnt; base += 32 * 16) {
        int32_t ii[16];
        float vv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int q = base + u * 32 + lane;
            ii[u] = q < cnt ? __ldg(indices + z0 + q) : 0;
            vv[u] = q < cnt ? __ldg(vals + z0 + q) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int q = base + u * 32 + lane;
            if (q < cnt) { st_idx[q] = (uint16_t)ii[u]; st_val[q] = vv[u]; }
        }
    }
    __syncwarp();
    if (active) {
        const float4* w4 = reinterpret_cast<const float4*>(sXW);
        for (int64_t p = b; p < e; ++p) {
            const int k = st_idx[p - z0];
            const float v = st_val[p - z0];
            const uint32_t m = __float_as_uint(sXW[csr_mask_slot(k)]);
            fma_row16_masked(v, w4 + 5 * k, m, acc[0]);
        }
    }
    __syncwarp();
}

// CSR pass from the slice copy (SmoArgs::sell_*, built once per training by layout.cu
// k_sell_fill): lane l walks the nonzeros of its row 4 at a time from [(g0 + j) * 32 + l] --
// coalesced 256-B index and 512-B value loads straight into registers, SELL_PF groups in flight
// per lane, no shared-memory staging and no bank conflicts on the stage -- with the same per-row
// order and masked X_W updates as dots_csr, so the sums are bit-identical to the staged path.
constexpr int SELL_PF = 4;
__device__ __forceinline__ uint32_t lds_u32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void dots_sell(const uint2* __restrict__ gi, const float4* __restrict__ gv,
                                          int ng, const float* sXW, const uint32_t* sMask,
                                          float (&acc)[1][SVM_WS])
{
    zero_acc<1>(acc);
    uint32_t wsm = (uint32_t)__cvta_generic_to_shared(sXW);   // X_W^T [d][WSTR_CSR] fp32
    uint32_t msm = (uint32_t)__cvta_generic_to_shared(sMask); // 4-bit group masks [d + 1] (d: padding, 0)
    asm volatile("" : "+r"(wsm), "+r"(msm));   // keep the bases in registers (no S2R rematerialisation)
    uint2 ri[SELL_PF];
    float4 rv[SELL_PF];
#pragma unroll
    for (int p = 0; p < SELL_PF; ++p) {
        ri[p] = make_uint2(0u, 0u);
        rv[p] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < ng) { ri[p] = __ldcs(gi + p * 32); rv[p] = __ldcs(gv + p * 32); }
    }
    for (int j0 = 0; j0 < ng; j0 += SELL_PF) {
#pragma unroll
        for (int p = 0; p < SELL_PF; ++p) {
            const int j = j0 + p;
            if (j < ng) {
                const uint2 ci = ri[p];
                const float4 cv = rv[p];
                if (j + SELL_PF < ng) {
                    ri[p] = __ldcs(gi + (j + SELL_PF) * 32);
                    rv[p] = __ldcs(gv + (j + SELL_PF) * 32);
                }
                const int kk[4] = {(int)(ci.x & 0xffffu), (int)(ci.x >> 16), (int)(ci.y & 0xffffu), (int)(ci.y >> 16)};
                const float vv[4] = {cv.x, cv.y, cv.z, cv.w};
                // the 4 group masks first (no branch between them: the loads issue together);
                // padding past a row's end has feature index d, whose mask is 0: no update
                uint32_t m[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) m[u] = lds_u32(msm + 4u * (uint32_t)kk[u]);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t wk = wsm + 4u * WSTR_CSR * (uint32_t)kk[u];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (m[u] & (1u << q)) {   // group q of X_W has a nonzero (as fma_row16_masked)
                            const float4 w = lds_f4(wk + 16u * q);
                            const float2 xx = make_float2(vv[u], vv[u]);
                            const float2 lo = __ffma2_rn(xx, make_float2(w.x, w.y), make_float2(acc[0][4 * q], acc[0][4 * q + 1]));
                            const float2 hi = __ffma2_rn(xx, make_float2(w.z, w.w), make_float2(acc[0][4 * q + 2], acc[0][4 * q + 3]));
                            acc[0][4 * q] = lo.x;
                            acc[0][4 * q + 1] = lo.y;
                            acc[0][4 * q + 2] = hi.x;
                            acc[0][4 * q + 3] = hi.y;
                        }
                    }
                }
            }
        }
    }
}

// Shared state of one persistent CTA (static part; X_W, the staged keys, the score arrays and
// the optional X slice are dynamic).
struct SmoShared {
    uint64_t warp_up[SMO_WARPS][8], warp_low[SMO_WARPS][8];
    uint64_t cta_up[8], cta_low[8];
    uint64_t win_up[8], win_low[8];      // merged global winners (keys)
    int32_t win_up_src[8], win_low_src[8];
    uint64_t gm_key[2][8][8];            // two-level merge: [side][part] sorted top-8 of part's lists
    int32_t gm_src[2][8][8];
    int64_t w_gidx[SVM_WS];              // working set, ascending dual index
    int32_t w_src[SVM_WS];               // exchange word index (slot * 64 + candidate) per position
    int32_t w_slot[SVM_WS];              // distinct-row slot of each position
    int64_t r_row[SVM_WS];               // distinct rows (global)
    double kr[SVM_WS * SVM_WS];          // K between distinct rows, fp64
    double kpos[SVM_WS * SVM_WS];        // K between working-set positions, fp64
    double inv_eta[SVM_WS * SVM_WS];     // 1 / max(K_aa + K_bb - 2 K_ab, tau)
    double qpart[136 * 4];               // k-split partial sums of the row-pair reductions
    double w_alpha[SVM_WS], w_G[SVM_WS], w_dalpha[SVM_WS], w_anew[SVM_WS];
    int32_t w_y[SVM_WS];
    float c[SVM_WS];                     // c_r = sum_{a: row r} y_a dalpha_a
    float xn[SVM_WS];                    // |x_r|^2 of the distinct rows
    uint64_t rk_key[2][SVM_MAX_RANKS * 8];   // rank level: [side][rank * 8 + position]
    int32_t rk_src[2][SVM_MAX_RANKS * 8];
    int32_t nw, nr, stop, timeout, next_chunk, next_chunk2, inner_steps, sub_done;
    int32_t c_slot[SVM_WS], c_ins[SVM_WS], c_mode;   // kernel-column cache (8(f) #3): per W row
    int32_t c_off, c_wh, c_rh, c_rl;     // cache switched off; cache passes, row hits and lookups
                                         // in the current window
    alignas(8) uint64_t mb_full[8], mb_empty[8];   // wide-mode / TMA-ring pipeline barriers
    uint64_t tma_seq[8];                 // TMA ring: chunk sequence number last issued into each slot
    double m_up, M_low;
};

// The rows one CTA's rank owns, as seen by that CTA.  A real rank (one GPU) sees its own arrays;
// a virtual rank (SmoArgs::virt, all ranks in one launch) sees its row range of the full arrays
// through offset pointers (the copy stride n_pad stays the full one).
struct RankView {
    const float* XT;
    const int64_t* indptr;
    const float* xnorm;
    double* alpha;
    float* G;
    uint8_t* status;
    int64_t n_local, row0;
    int rank, cta, nblk;
};
__device__ __forceinline__ RankView rank_view(const SmoArgs& a)
{
    RankView v;
    if (a.virt) {
        v.rank = (int)blockIdx.x / a.nblk;
        v.cta = (int)blockIdx.x - v.rank * a.nblk;
        v.row0 = a.rank_row0[v.rank];
        v.n_local = a.rank_row0[v.rank + 1] - v.row0;
    } else {
        v.rank = a.rank;
        v.cta = (int)blockIdx.x;
        v.row0 = a.row0;
        v.n_local = a.n_local;
    }
    v.nblk = a.nblk;
    const int64_t off = a.virt ? v.row0 : 0;
    v.XT = a.XT ? a.XT + off : nullptr;
    v.indptr = a.indptr ? a.indptr + off : nullptr;
    v.xnorm = a.xnorm + off;
    v.alpha = a.alpha + off;
    v.G = a.G + off;
    v.status = a.status + off;
    return v;
}

// Per-row epilogue shared by the scan (do_update = false) and the pass: kernel values from the
// dot products, G update, and each dual's 64-bit up / low candidate keys (score << 32 | ~index;
// 0 = not a candidate) kept in registers: ku[2 j + c], kl[2 j + c] for row j, copy c.
template <int RPT, bool RBFK>
__device__ __forceinline__ void row_epilogue(const SmoArgs& a, const RankView& v, const SmoShared& sh, int64_t li0,
                                             int64_t cta_end, bool do_update,
                                             const float (&acc)[RPT][SVM_WS],
                                             uint64_t (&ku)[2 * RPT], uint64_t (&kl)[2 * RPT],
                                             int kmode = 0, float* kc = nullptr)
{
    // kmode (kernel-column cache): 0 = K from the dot products; 1 = the same, and
    // the columns of the W rows newly cached this iteration (sh.c_ins[r] >= 0) are stored into
    // kc[slot][row]; 2 = every W row is cached: K read from kc[sh.c_slot[r]][row] (no X, no dots);
    // 3 = acc already holds those cached K values (copied to shared memory during phase A).
    // The stored values are exactly the ones the computing path uses, and S sums over r in the
    // same order either way, so all three modes give bit-identical G.
    if constexpr (RPT == 4) {
        // A lane's 4 rows are consecutive and li0 is a multiple of 4 (rows_per_cta and n_pad are):
        // the norms, G and status of all 4 rows (both copies) are loaded up front as one 16-byte /
        // one 4-byte load per array, before any store.  (Row by row, the uint8_t status load of
        // row j + 1 may alias the G store of row j, so the compiler kept 4 dependent global round
        // trips per call.)  Identical arithmetic; rows >= cta_end are never written.
#pragma unroll
        for (int q = 0; q < 2 * RPT; ++q) ku[q] = kl[q] = 0ull;
        if (li0 >= cta_end) return;
        float4 g4[2];
        uint32_t st4[2] = {0u, 0u};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            g4[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < a.ncopy) {
                const int64_t idx = (int64_t)c * a.n_pad + li0;
                st4[c] = *reinterpret_cast<const uint32_t*>(v.status + idx);
                g4[c] = *reinterpret_cast<const float4*>(v.G + idx);
            }
        }
        float S[4] = {0.f, 0.f, 0.f, 0.f};
        const bool full = li0 + 4 <= cta_end;
        if (do_update && kmode == 3) {   // acc holds the cached K values (phase A copy)
#pragma unroll
            for (int r = 0; r < SVM_WS; ++r)
#pragma unroll
                for (int j = 0; j < 4; ++j) S[j] = fmaf(sh.c[r], acc[j][r], S[j]);
        } else if (do_update && kmode == 2) {
#pragma unroll
            for (int r = 0; r < SVM_WS; ++r) {
                const int sl = sh.c_slot[r];
                const float4 K = sl >= 0 ? *reinterpret_cast<const float4*>(kc + (int64_t)sl * a.n_pad + li0)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                S[0] = fmaf(sh.c[r], K.x, S[0]);
                S[1] = fmaf(sh.c[r], K.y, S[1]);
                S[2] = fmaf(sh.c[r], K.z, S[2]);
                S[3] = fmaf(sh.c[r], K.w, S[3]);
            }
        } else if (do_update) {
            const float4 xn4 = __ldg(reinterpret_cast<const float4*>(v.xnorm + li0));
            const float xn[4] = {xn4.x, xn4.y, xn4.z, xn4.w};
            const float ng = -a.kp.gamma * 1.4426950408889634f;
#pragma unroll
            for (int r = 0; r < SVM_WS; ++r) {
                float K[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if constexpr (RBFK) {
                        const float d2 = fmaxf(fmaf(-2.0f, acc[j][r], xn[j] + sh.xn[r]), 0.0f);
                        K[j] = exp2f_approx(ng * d2);
                    } else {
                        K[j] = kernel_from_dot(a.kp, acc[j][r], xn[j], sh.xn[r]);
                    }
                    S[j] = fmaf(sh.c[r], K[j], S[j]);
                }
                if (kmode == 1) {
                    const int ins = sh.c_ins[r];
                    if (ins >= 0) {
                        float* dst = kc + (int64_t)ins * a.n_pad + li0;
                        if (full) *reinterpret_cast<float4*>(dst) = make_float4(K[0], K[1], K[2], K[3]);
                        else
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (li0 + j < cta_end) dst[j] = K[j];
                    }
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (c >= a.ncopy) break;
            float g[4] = {g4[c].x, g4[c].y, g4[c].z, g4[c].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t st = (st4[c] >> (8 * j)) & 0xffu;
                const float yv = (st & ST_YPOS) ? 1.0f : -1.0f;
                if (do_update) g[j] = fmaf(yv, S[j], g[j]);
                const float sc = -yv * g[j];
                const uint64_t gi = (uint64_t)c * (uint64_t)a.n_global + (uint64_t)(v.row0 + li0 + j);
                const uint64_t lo = (uint64_t)(0xffffffffu - (uint32_t)gi);
                const bool in = li0 + j < cta_end;
                if (in && st_in_up(st)) ku[2 * j + c] = ((uint64_t)ord_f32(sc) << 32) | lo;
                if (in && st_in_low(st)) kl[2 * j + c] = ((uint64_t)ord_f32(-sc) << 32) | lo;
            }
            if (do_update) {
                const int64_t idx = (int64_t)c * a.n_pad + li0;
                if (full) {
                    *reinterpret_cast<float4*>(v.G + idx) = make_float4(g[0], g[1], g[2], g[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (li0 + j < cta_end) v.G[idx + j] = g[j];
                }
            }
        }
        return;
    } else {
    // RPT 1 / 2: every row's status, G and norm loaded before the first G store (as above)
    uint32_t stv[RPT][2];
    float gv[RPT][2], xnv[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        const int64_t li = li0 + j;
        xnv[j] = (do_update && li < cta_end) ? __ldg(v.xnorm + li) : 0.0f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            stv[j][c] = 0u;
            gv[j][c] = 0.0f;
            if (li < cta_end && c < a.ncopy) {
                const int64_t idx = (int64_t)c * a.n_pad + li;
                stv[j][c] = v.status[idx];
                gv[j][c] = v.G[idx];
            }
        }
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        const int64_t li = li0 + j;
        ku[2 * j] = ku[2 * j + 1] = kl[2 * j] = kl[2 * j + 1] = 0ull;
        if (li >= cta_end) continue;
        float S = 0.0f;
        if (do_update && kmode == 3) {
#pragma unroll
            for (int r = 0; r < SVM_WS; ++r) S = fmaf(sh.c[r], acc[j][r], S);
        } else if (do_update && kmode == 2) {
#pragma unroll
            for (int r = 0; r < SVM_WS; ++r) {
                const int sl = sh.c_slot[r];
                S = fmaf(sh.c[r], sl >= 0 ? kc[(int64_t)sl * a.n_pad + li] : 0.0f, S);
            }
        } else if (do_update) {
            const float xn = xnv[j];
            const float ng = -a.kp.gamma * 1.4426950408889634f;  // exp(z) = 2^(z log2 e)
            auto kval = [&](int r) -> float {
                if constexpr (RBFK) {  // exp(-gamma |x_i - x_r|^2) with the distance from the norms
                    const float d2 = fmaxf(fmaf(-2.0f, acc[j][r], xn + sh.xn[r]), 0.0f);
                    return exp2f_approx(ng * d2);
                } else {
                    return kernel_from_dot(a.kp, acc[j][r], xn, sh.xn[r]);
                }
            };
            if (kmode == 1) {   // cache inserts of the new W columns (same S order as below)
#pragma unroll
                for (int r = 0; r < SVM_WS; ++r) {
                    const float K = kval(r);
                    S = fmaf(sh.c[r], K, S);
                    if (sh.c_ins[r] >= 0) kc[(int64_t)sh.c_ins[r] * a.n_pad + li] = K;
                }
            } else {
#pragma unroll
                for (int r = 0; r < SVM_WS; ++r) S = fmaf(sh.c[r], kval(r), S);
            }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (c >= a.ncopy) break;
            const int64_t idx = (int64_t)c * a.n_pad + li;
            const uint32_t st = stv[j][c];
            const float yv = (st & ST_YPOS) ? 1.0f : -1.0f;
            float g = gv[j][c];
            if (do_update) {
                g = fmaf(yv, S, g);
                v.G[idx] = g;
            }
            const float sc = -yv * g;
            const uint64_t gi = (uint64_t)c * (uint64_t)a.n_global + (uint64_t)(v.row0 + li);
            const uint64_t lo = (uint64_t)(0xffffffffu - (uint32_t)gi);
            if (st_in_up(st)) ku[2 * j + c] = ((uint64_t)ord_f32(sc) << 32) | lo;
            if (st_in_low(st)) kl[2 * j + c] = ((uint64_t)ord_f32(-sc) << 32) | lo;
        }
    }
}   // RPT 1 / 2
}

// Descending sort of a lane's NK keys (odd-even transposition network, fully unrolled).
template <int NK>
__device__ __forceinline__ void sort_desc(uint64_t (&k)[NK])
{
#pragma unroll
    for (int i = 0; i < NK; ++i) {
#pragma unroll
        for (int j = (i & 1); j + 1 < NK; j += 2) {
            const uint64_t x = k[j], y = k[j + 1];
            const bool sw = y > x;
            k[j] = sw ? y : x;
            k[j + 1] = sw ? x : y;
        }
    }
}

// Merge one chunk's candidate keys (NK per lane) into the warp's running top-8 lists (lane l < 8
// holds the l-th best, descending; 0 = empty), up and low together.  Only keys above the current
// 8th can enter: their warp-wide count (capped at 8) bounds the rounds.  Each lane sorts its keys
// once; a round takes the 64-bit warp max of the lanes' heads and inserts it into the list at
// rank popc(ballot(list > key)) (entries below shift down one lane); the winning lane pops its
// head.  Keys are unique, so the result is exact.
template <int NK>
__device__ __forceinline__ void merge_chunk(uint64_t (&ku)[NK], uint64_t (&kl)[NK], uint64_t& wlu,
                                            uint64_t& wll, int lane)
{
    const uint64_t thu = __shfl_sync(FULL, wlu, 7), thl = __shfl_sync(FULL, wll, 7);
    uint32_t cu = 0, cl = 0;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        cu += ku[k] > thu ? 1u : 0u;
        cl += kl[k] > thl ? 1u : 0u;
    }
    int ru = (int)min(__reduce_add_sync(FULL, cu), 8u);
    int rl = (int)min(__reduce_add_sync(FULL, cl), 8u);
    if (ru == 0 && rl == 0) return;
    if (ru) sort_desc<NK>(ku);
    if (rl) sort_desc<NK>(kl);
    const int rounds = ru > rl ? ru : rl;
#pragma unroll 1
    for (int r = 0; r < rounds; ++r) {
        const bool du = r < ru, dl = r < rl;   // warp-uniform
        const uint64_t hu = du ? ku[0] : 0ull, hl = dl ? kl[0] : 0ull;
        const uint64_t bu = warp_max_u64(hu);
        const uint64_t bl = warp_max_u64(hl);
        const uint64_t pu = __shfl_up_sync(FULL, wlu, 1), pl = __shfl_up_sync(FULL, wll, 1);
        const int posu = __popc(__ballot_sync(FULL, lane < 8 && wlu > bu));
        const int posl = __popc(__ballot_sync(FULL, lane < 8 && wll > bl));
        if (du && bu != 0ull && posu < 8) {
            if (lane == posu) wlu = bu;
            else if (lane > posu && lane < 8) wlu = pu;
            if (hu == bu) {
#pragma unroll
                for (int q = 0; q + 1 < NK; ++q) ku[q] = ku[q + 1];
                ku[NK - 1] = 0ull;
            }
        } else ru = 0;      // nothing left above the 8th on this side
        if (dl && bl != 0ull && posl < 8) {
            if (lane == posl) wll = bl;
            else if (lane > posl && lane < 8) wll = pl;
            if (hl == bl) {
#pragma unroll
                for (int q = 0; q + 1 < NK; ++q) kl[q] = kl[q + 1];
                kl[NK - 1] = 0ull;
            }
        } else rl = 0;
    }
}

// One copy per row (C-SVC): only the even key slots are used, so merge RPT keys per lane.
template <int RPT>
__device__ __forceinline__ void merge_chunk_rows(uint64_t (&ku)[2 * RPT], uint64_t (&kl)[2 * RPT],
                                                 uint64_t& wlu, uint64_t& wll, int lane, int ncopy)
{
    if (ncopy == 1) {
        uint64_t cu[RPT], cl[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) { cu[j] = ku[2 * j]; cl[j] = kl[2 * j]; }
        merge_chunk<RPT>(cu, cl, wlu, wll, lane);
    } else {
        merge_chunk<2 * RPT>(ku, kl, wlu, wll, lane);
    }
}

// Explicit shared-memory 64-bit load for the list merges.  With plain indexed loads
// (keys[l * 8 + hd + 1]) nvcc 12.9 / sm_100a returned the element one past the intended one for
// some shared-memory carve-outs (found by a partition-invariance test: L = 40 lists, the merge
// skipped one list entry); the explicit ld.shared reads exactly the addressed word.
__device__ __forceinline__ uint64_t lds_u64(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

// Merge SMO_WARPS sorted warp lists into the CTA top-8 (one warp).
__device__ __forceinline__ void cta_merge(const uint64_t (*lists)[8], uint64_t* out, int lane)
{
    int idx = 0;
    uint64_t head = lane < SMO_WARPS ? lds_u64(&lists[lane][0]) : 0;
    uint64_t next = lane < SMO_WARPS ? lds_u64(&lists[lane][1]) : 0;
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
        uint64_t best = warp_max_u64(head);
        if (lane == 0) out[r] = best;
        if (best == 0) {
            if (lane > r && lane < 8) out[lane] = 0;
            break;
        }
        if (head == best && lane < SMO_WARPS) {
            ++idx;
            head = next;
            next = idx + 1 < 8 ? lds_u64(&lists[lane][idx + 1]) : 0;
        }
    }
}

// One warp, one sorted 8-list per lane (heads in registers, the next key prefetched): the top-8
// of the union in 8 rounds of a 64-bit warp max.  key(l, j) / src(l, j) read list l's j-th entry.
template <class KeyF, class SrcF>
__device__ __forceinline__ void lane_list_merge(int nl, KeyF key, SrcF srcf, uint64_t* out,
                                                int32_t* src, int lane)
{
    int hd = 0;
    uint64_t cur = lane < nl ? key(lane, 0) : 0ull;
    uint64_t nxt = lane < nl ? key(lane, 1) : 0ull;
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
        const uint64_t best = warp_max_u64(cur);
        if (best == 0ull) {
            if (lane < 8 && lane >= r) { out[lane] = 0ull; src[lane] = -1; }
            break;
        }
        if (cur == best) {   // unique owner (keys are unique)
            out[r] = best;
            src[r] = srcf(lane, hd);
            ++hd;
            cur = nxt;
            nxt = hd + 1 < 8 ? key(lane, hd + 1) : 0ull;
        }
    }
}

__device__ __forceinline__ int owner_rank(const SmoArgs& a, int64_t row)
{
    int r = 0;
    while (r + 1 < a.world && row >= a.rank_row0[r + 1]) ++r;
    return r;
}

__device__ __forceinline__ double lds_f64(uint32_t addr)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// The |W|-variable subproblem (a2) on one warp, lane a = position a: max-violating-pair steps in
// fp64 ("optimized based on the local gradient").  argmax_{I_up} s and
// argmin_{I_low} s are exact 64-bit REDUX reductions of order-preserving keys, ties to the lowest
// lane = lowest position.  The step in score form (s_a = -y_a G_a):
//   t = (s_i - s_j) / eta_ij clipped to the box;  s_a += t (K_aj - K_ai)
// which is the oracle's G_W += Q_Wi y_i t - Q_Wj y_j t, since Q_ab = y_a y_b K_ab.
__device__ __forceinline__ int solve_subproblem(SmoShared& sh, int nw, double C, double inner_tol,
                                                int inner_max, int lane)
{
    const int pa = lane & 15;
    const bool valid = lane < nw;
    const int y = valid ? sh.w_y[lane] : 1;
    const double al0 = valid ? sh.w_alpha[lane] : 0.0;
    double s = valid ? -(double)y * sh.w_G[lane] : 0.0;
    // shared-window addresses computed once (keeps S2R/LEA off the per-step chain)
    const uint32_t a_ie = (uint32_t)__cvta_generic_to_shared(sh.inv_eta);
    const uint32_t a_krow = (uint32_t)__cvta_generic_to_shared(sh.kpos + pa * SVM_WS);
    // room to move y_a alpha_a up (> 0 <=> a in I_up) and down (> 0 <=> a in I_low)
    double up_room = valid ? (y > 0 ? C - al0 : al0) : 0.0;
    double dn_room = valid ? (y > 0 ? al0 : C - al0) : 0.0;
    int step = 0;
    for (; step < inner_max; ++step) {
        const uint64_t ku = up_room > 0.0 ? mono64(s) : 0ull;
        const uint64_t kl = dn_room > 0.0 ? mono64(-s) : 0ull;
        const uint32_t hu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32));
        const uint32_t hl = __reduce_max_sync(FULL, (uint32_t)(kl >> 32));
        const uint32_t lu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32) == hu ? (uint32_t)ku : 0u);
        const uint32_t ll = __reduce_max_sync(FULL, (uint32_t)(kl >> 32) == hl ? (uint32_t)kl : 0u);
        const uint64_t mu = ((uint64_t)hu << 32) | lu, ml = ((uint64_t)hl << 32) | ll;
        const int i = (__ffs(__ballot_sync(FULL, ku == mu)) - 1) & 15;
        const int j = (__ffs(__ballot_sync(FULL, kl == ml)) - 1) & 15;
        // the step's operands are loaded before the stop test (in bounds for any i, j < 16), so
        // the shared-memory latency overlaps the test instead of following it
        const double ie = lds_f64(a_ie + 8u * (uint32_t)(i * SVM_WS + j));
        const double kai = lds_f64(a_krow + 8u * (uint32_t)i);
        const double kaj = lds_f64(a_krow + 8u * (uint32_t)j);
        // lim_i = room of i to move up, lim_j = room of j to move down
        const double lim_i = __shfl_sync(FULL, up_room, i), lim_j = __shfl_sync(FULL, dn_room, j);
        const double si = unmono64(mu), sj = -unmono64(ml);
        if (mu == 0 || ml == 0 || si - sj <= inner_tol) break;
        double t = (si - sj) * ie;
        const bool ci = t >= lim_i;
        t = ci ? lim_i : t;
        const bool cj = t >= lim_j;
        t = cj ? lim_j : t;
        const bool clip_i = ci && (!cj || lim_i == lim_j);
        if (lane == i) {  // y_i alpha_i += t; clipped -> exactly at its bound
            up_room = clip_i ? 0.0 : up_room - t;
            dn_room = clip_i ? C : dn_room + t;
        }
        if (lane == j) {  // y_j alpha_j -= t
            dn_room = cj ? 0.0 : dn_room - t;
            up_room = cj ? C : up_room + t;
        }
        s = fma(t, kaj - kai, s);
    }
    if (lane < SVM_WS) sh.w_anew[lane] = valid ? (y > 0 ? C - up_room : up_room) : 0.0;
    return step;
}

// ---- wide-mode pipeline primitives (mbarrier + bulk async copy, sm_90+ PTX) -----------------
constexpr int WIDE_STAGES = 8;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t gtimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity)
{
    uint32_t ok = 0;
    uint32_t spins = 0;
    uint64_t t0 = 0;
    for (;;) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
        if (ok) return;
        if (++spins == 1024) {   // watchdog: a lost stage must fail the launch, not hang the GPU
            spins = 0;
            const uint64_t now = gtimer_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 5000000000ull) __trap();
        }
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// 2D tensor copy (TMA) of one box of the map into shared memory, completing on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
                   "r"(smem_u32(bar)) : "memory");
}

template <bool CSR, int RPT, bool XS, bool RBFK>
__global__ void __launch_bounds__(SMO_THREADS, 1) smo_persistent(const __grid_constant__ SmoArgs a)
{
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    __shared__ SmoShared sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const RankView v = rank_view(a);
    const int L = a.nblk;      // this rank's CTA lists (local level of the exchange)
    const int P = a.world;     // ranks (rank level of the exchange when > 1)
    const int d = (int)a.d;
    const int dp = (d + 3) & ~3;
    const int R = (int)a.rows_per_cta;
    float* sXW = reinterpret_cast<float*>(dyn_smem);                        // [d][16] fp32
    constexpr int WS = CSR ? WSTR_CSR : SVM_WS;                               // sXW row stride
    uint64_t* sKU = reinterpret_cast<uint64_t*>(sXW + (size_t)((d * WS + 3) & ~3));  // [L][8]
    uint64_t* sKL = sKU + (size_t)L * 8;                                     // [L][8]
    float* sX = reinterpret_cast<float*>(sKL + (size_t)L * 8);               // [d][R] (XS)
    // dot-product buffer: [16][dbuf_rows] fp32, column r holds x_i . x_{W_r} for the CTA's first
    // dbuf_rows rows (filled while the subproblem runs, read by the epilogue afterwards)
    const bool sell = CSR && a.sell_idx != nullptr;   // CSR from the slice copy (no staging)
    int32_t* sGp = reinterpret_cast<int32_t*>(sX);     // SELL: [spc + 1] group offsets of this CTA
    uint32_t* sMask = reinterpret_cast<uint32_t*>(sX) + ((a.sell_spc + 4) & ~3);   // SELL: [d + 1] masks
    float* csr_val = sX + (size_t)warp * CSR_CAP;                                   // CSR only
    uint16_t* csr_idx = reinterpret_cast<uint16_t*>(sX + (size_t)SMO_WARPS * CSR_CAP) + (size_t)warp * CSR_CAP;
    // TMA ring (streamed dense X, a.x_tma): tma_ns slots of [d][32 RPT] fp32, 128-byte aligned
    constexpr bool TMA_OK = !CSR && !XS;
    const bool tma = TMA_OK && a.x_tma != 0;
    const int NS = tma ? a.tma_ns : 1;
    constexpr int CH = 32 * RPT;
    float* tring = reinterpret_cast<float*>(dyn_smem + ((smem_u32(sX) + 127u) & ~127u) - smem_u32(dyn_smem));
    const uint32_t stage_floats = (uint32_t)d * CH;
    float* sDot = tma ? tring + (size_t)NS * stage_floats
                      : sX + (XS ? (size_t)d * R : (CSR ? (sell ? (size_t)((a.sell_spc + 4) & ~3) + (size_t)((d + 4) & ~3) : (size_t)SMO_WARPS * CSR_CAP * 6 / 4)
                                                        : (size_t)SMO_THREADS * pf_x<RPT>() * RPT));
    const int dbuf_rows = a.dbuf_rows;

    const int64_t cta_begin = (int64_t)v.cta * a.rows_per_cta;
    const int64_t cta_end = min(cta_begin + a.rows_per_cta, v.n_local);
    const int nvalid = cta_end > cta_begin ? (int)(cta_end - cta_begin) : 0;
    // rows per chunk (work item of one warp): 32 RPT, or fewer (a.chunk_rows, a multiple of 4)
    // so that the chunk count is a multiple of the warp count and every warp gets the same
    // number of chunks; lanes beyond the chunk's rows idle (lane_on)
    const int rows_per_chunk = (a.chunk_rows > 0 && a.chunk_rows < 32 * RPT) ? a.chunk_rows : 32 * RPT;
    const int nchunks = (nvalid + rows_per_chunk - 1) / rows_per_chunk;
    const bool lane_on = lane * RPT < rows_per_chunk;
    const int slot = v.cta;
    const bool sys = a.world > 1 && !a.virt;   // peers across NVLink: system scope
    const bool reporter = blockIdx.x == 0;  // CTA 0 of every rank reports for its rank
    uint64_t* rxr = a.peer_xw[v.rank];      // this rank's exchange buffer: rank level ...
    uint64_t* rxw = rxr + XW_RANK_WORDS;    // ... and local level (its own CTAs' lists)

#ifdef SMO_POISON
    {
        uint32_t dsz;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsz));
        for (uint32_t i = tid; i < dsz / 4; i += SMO_THREADS) reinterpret_cast<uint32_t*>(dyn_smem)[i] = SMO_POISON;
        __syncthreads();
    }
#endif
    // stage this CTA's X^T slice into shared memory once (resident across iterations)
    if constexpr (XS) {
        for (int k = warp; k < d; k += SMO_WARPS)
            for (int r = lane; r < R; r += 32)
                sX[(size_t)k * R + r] = v.XT[(int64_t)k * a.n_pad + cta_begin + r];
    }
    // SELL CSR: this CTA's slice offsets, relative to its first group (constant for the training)
    int64_t sell_g0 = 0;
    if (sell) {
        const int64_t* gp = a.sell_gptr + ((a.virt ? (int64_t)v.rank * a.nblk : 0) + v.cta) * a.sell_spc;
        sell_g0 = gp[0];
        for (int c = tid; c <= a.sell_spc; c += SMO_THREADS) sGp[c] = (int32_t)(gp[c] - sell_g0);
        __syncthreads();
    }
    auto csr_dots = [&](int ch, int64_t li0, float (&acc)[1][SVM_WS]) {
        if (sell) {
            const int64_t g0 = sell_g0 + sGp[ch];
            dots_sell(a.sell_idx + g0 * 32 + lane, a.sell_val + g0 * 32 + lane, sGp[ch + 1] - sGp[ch],
                      sXW, sMask, acc);
        } else {
            dots_csr_staged(v.indptr, a.indices, a.vals, li0 - lane, cta_end, lane, csr_idx, csr_val, sXW, acc);
        }
    };
    const float* xbase = XS ? sX : v.XT + cta_begin;
    const int64_t xld = XS ? R : a.n_pad;
    // per-lane cp.async ring for streamed X (in the place of the resident slice)
    const uint32_t xring = (uint32_t)__cvta_generic_to_shared(sX) +
                           (uint32_t)(warp * pf_x<RPT>() * 32 * 4 * RPT + lane * 4 * RPT);

    // ---- wide mode (streamed dense rows, large d): CTA-wide bulk-copy pipeline --------------
    // Stage T of the run holds features [kc (T % nst), +kc) of the CTA's R rows ([kc][R] fp32,
    // one contiguous R * 4 B copy per feature) in slot T % 8; the producer (lane 0 of warp ncw)
    // runs 8 stages ahead of the consumer warps, across iteration boundaries (X does not depend
    // on W), so the next iteration's first stages load during this one's epilogue and exchange.
    constexpr bool WIDE_OK = !CSR && !XS && RPT == 1;   // compiled out elsewhere (registers)
    const bool wide = WIDE_OK && a.wide != 0;
    const int wkc = a.wide_kc > 0 ? a.wide_kc : 8;
    const int nst = (d + wkc - 1) / wkc;
    const int ncw = (R + 31) / 32;                        // consumer warps, 32 rows each
    const int Rs = ncw * 32 + 8;                          // stage row stride: = 8 mod 32 floats
    float* wring = sX;                                    // [8][wkc][Rs]
    auto wide_issue = [&](uint64_t T) {
        const int s = (int)(T % WIDE_STAGES);
        const int k0 = (int)(T % (uint64_t)nst) * wkc, kn = min(wkc, d - k0);
        mbar_arrive_tx(&sh.mb_full[s], (uint32_t)(kn * R * 4));
        float* dst = wring + (size_t)s * wkc * Rs;
        for (int q = 0; q < kn; ++q)
            bulk_g2s(dst + (size_t)q * Rs, v.XT + (int64_t)(k0 + q) * a.n_pad + cta_begin,
                     (uint32_t)(R * 4), &sh.mb_full[s]);
    };
    if (wide) {
        if (tid == 0) {
            for (int s = 0; s < WIDE_STAGES; ++s) {
                mbar_init(&sh.mb_full[s], 1);
                mbar_init(&sh.mb_empty[s], (uint32_t)ncw);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (warp == ncw && lane == 0)
            for (int T = 0; T < WIDE_STAGES; ++T) wide_issue((uint64_t)T);
    }

    // ---- TMA ring for streamed dense X (a.x_tma): chunk sequence T = t * nchunks + j -----------
    // slot T % NS holds chunk j = T % nchunks ([d][CH] rows cta_begin + j CH ..).  The consumer of
    // T refills the slot with T + NS once its warp has read it; a consumer of T first waits until
    // the slot's sequence number says T was issued (so the mbarrier is in T's phase), then on the
    // phase parity (T / NS) & 1.  Chunks are consumed in increasing j within each iteration
    // (phase A hands out 0, 1, ..; phase B the rest), so the ring runs ahead across iterations.
    const uint32_t stage_bytes = stage_floats * 4u;
    const int map_row0 = (int)((a.virt ? v.row0 : 0) + cta_begin);
    auto tma_issue = [&](uint64_t T) {      // one thread
        const int s = (int)(T % (uint64_t)NS);
        const int j = (int)(T % (uint64_t)nchunks);
        mbar_arrive_tx(&sh.mb_full[s], stage_bytes);
        tma_load_2d(tring + (size_t)s * stage_floats, &a.xmap, map_row0 + j * CH, 0, &sh.mb_full[s]);
        *reinterpret_cast<volatile uint64_t*>(&sh.tma_seq[s]) = T;
    };
    auto tma_acquire = [&](uint64_t T) -> const float* {   // whole warp
        const int s = (int)(T % (uint64_t)NS);
        if (lane == 0)
            while (*reinterpret_cast<volatile uint64_t*>(&sh.tma_seq[s]) != T) {}
        __syncwarp();
        mbar_wait(&sh.mb_full[s], (uint32_t)((T / (uint64_t)NS) & 1));
        return tring + (size_t)s * stage_floats;
    };
    auto tma_release = [&](uint64_t T) {   // whole warp, after its reads of T's slot
        __syncwarp();
        if (lane == 0) tma_issue(T + (uint64_t)NS);
    };
    if (tma) {
        if (tid == 0) {
            for (int s = 0; s < NS; ++s) {
                mbar_init(&sh.mb_full[s], 1);
                sh.tma_seq[s] = ~0ull;
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && nchunks > 0)
            for (int T = 0; T < NS; ++T) tma_issue((uint64_t)T);
    }

    if (tid == 0) { sh.c_off = 0; sh.c_wh = 0; sh.c_rh = 0; sh.c_rl = 0; sh.c_mode = 0; }   // (read after the prologue's barriers)

    // ---- end of a pass: warp lists -> CTA top-8 up / low ---------------------------------------
    auto finish_lists = [&](uint64_t wlu, uint64_t wll) {
        if (lane < 8) {
            sh.warp_up[warp][lane] = wlu;
            sh.warp_low[warp][lane] = wll;
        }
        __syncthreads();
        if (warp == 0) cta_merge(sh.warp_up, sh.cta_up, lane);
        else if (warp == 1) cta_merge(sh.warp_low, sh.cta_low, lane);
        __syncthreads();
    };

    // ---- publish: 16 key words + 48 payload words per rank, each carrying the tag ------------
    auto publish = [&](uint32_t tag) {
        const int par = tag & 1;
        const uint64_t tg = tag16_of(tag);
        if (tid < 16) {
            const uint64_t k = tid < 8 ? sh.cta_up[tid] : sh.cta_low[tid - 8];
            uint64_t wkey = tg, w0 = tg, w1 = tg, w2 = tg;
            if (k) {
                const uint64_t g = key_index(k);
                const int c = g >= (uint64_t)a.n_global ? 1 : 0;
                const int64_t li = (int64_t)(g - (uint64_t)c * a.n_global) - v.row0;
                const int64_t idx = (int64_t)c * a.n_pad + li;
                const uint64_t pos = (uint64_t)c * (uint64_t)R + (uint64_t)(li - cta_begin);
                wkey = tg | ((k >> 32) << 16) | pos;
                const uint64_t ab = (uint64_t)__double_as_longlong(v.alpha[idx]);
                w0 = tg | (ab >> 16);
                w1 = tg | ((ab & 0xffffull) << 32) | (uint64_t)__float_as_uint(v.G[idx]);
                w2 = tg | (uint64_t)v.status[idx];
            }
            // the rank's own local level only (payload words are read by other ranks over NVLink)
            uint64_t* dst = rxw + ((size_t)par * L + slot) * XW_PER_SLOT;
            st_relaxed_u64(dst + 16 + 3 * tid, w0, sys);
            st_relaxed_u64(dst + 17 + 3 * tid, w1, sys);
            st_relaxed_u64(dst + 18 + 3 * tid, w2, sys);
            st_relaxed_u64(dst + tid, wkey, sys);
        }
    };

    // ---- exact CTA selection from the stored G / status (prologue, and the rare fallback when a
    // lane's top-3 may have truncated its candidates): per-warp extraction over fixed chunks ---
    auto exact_select = [&]() {
        uint64_t wlu = 0, wll = 0;
        float acc[RPT][SVM_WS];
        zero_acc<RPT>(acc);
        for (int ch = warp; ch < nchunks; ch += SMO_WARPS) {
            const int64_t li0 = lane_on ? cta_begin + (int64_t)ch * rows_per_chunk + lane * RPT : cta_end;
            uint64_t ku[2 * RPT], kl[2 * RPT];
            row_epilogue<RPT, RBFK>(a, v, sh, li0, cta_end, false, acc, ku, kl);
            merge_chunk_rows<RPT>(ku, kl, wlu, wll, lane, a.ncopy);
        }
        finish_lists(wlu, wll);
    };

    // ---- prologue: scan the current (alpha, G) and publish tag0 + 1 ---------------------------
    if (!a.pass_only) {
        exact_select();
        publish(a.tag0 + 1);
    }
    // per-iteration exchange latency (CTA 0, thread 0): its publish -> every rank's slots staged.
    // Includes the wait for the slowest CTA of any rank, i.e. what the collective costs the loop.
    // One 32-bit register across the loop (differences mod 2^32); the sums go out as fire-and-
    // forget reductions into the zeroed info block.
    uint32_t x_pub = (uint32_t)clock();
    if (reporter && tid == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.info->loop_cycles), (unsigned long long)(-clock64()));

#ifdef SMO_PROFILE
    // B200 __syncthreads is BAR.SYNC.DEFER_BLOCKING: the warp only blocks at the next use of
    // barrier-protected state, so each timestamp first consumes a shared-memory load.
    auto fenced_clock = [&]() -> long long {
        int v = *reinterpret_cast<volatile int*>(&sh.nw);
        asm volatile("" ::"r"(v) : "memory");
        return clock64();
    };
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long wprof[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // worker view (warp 0)
    long long wprev = 0;
    auto wmark = [&](int ph) {
        long long now = fenced_clock();
        if (ph >= 0) wprof[ph] += now - wprev;
        wprev = now;
    };
#else
    auto wmark = [](int) {};
#endif
#ifdef SMO_PROFILE
    long long tprev = clock64();
    auto mark = [&](int ph) {
        long long now = fenced_clock();
        prof[ph] += now - tprev;
        tprev = now;
    };
#else
    auto mark = [](int) {};
#endif
    for (int64_t t = 0;; ++t) {
        const uint32_t tag = a.tag0 + 1 + (uint32_t)t;
        const int par = tag & 1;
        const uint64_t tg = tag16_of(tag);
        // no bulk copy may outlive the CTA (wide mode): wait for the stages the producer issued
        auto drain_wide = [&]() {
            if (wide && warp == ncw && lane == 0)
                for (uint64_t T = (uint64_t)t * nst; T < (uint64_t)t * nst + WIDE_STAGES; ++T)
                    mbar_wait(&sh.mb_full[T % WIDE_STAGES], (uint32_t)((T / WIDE_STAGES) & 1));
            if (tma && tid == 0 && nchunks > 0)   // the NS chunks issued ahead for iteration t
                for (uint64_t T = (uint64_t)t * nchunks; T < (uint64_t)t * nchunks + NS; ++T) {
                    const int s = (int)(T % (uint64_t)NS);
                    while (*reinterpret_cast<volatile uint64_t*>(&sh.tma_seq[s]) != T) {}
                    mbar_wait(&sh.mb_full[s], (uint32_t)((T / (uint64_t)NS) & 1));
                }
        };
        if (a.pass_only) {
            // ---- pass-only diagnostic: fixed W (local rows of a single rank), fixed c ----------
            if (t >= a.max_iter) {
                drain_wide();
                if (reporter && tid == 0) {
                    a.info->iterations = t;
                    atomicAdd(reinterpret_cast<unsigned long long*>(&a.info->loop_cycles), (unsigned long long)clock64());
                }
#ifdef SMO_PROFILE
                if (reporter && tid == SOLVER_WARP * 32)
                    for (int ph = 0; ph < 8; ++ph) a.info->phase_cycles[ph] = prof[ph];
                if (reporter && tid == 0)
                    for (int ph = 0; ph < 8; ++ph) a.info->phase_cycles[8 + ph] = wprof[ph];
#endif
                return;
            }
            if (tid == 0) {
                sh.next_chunk = 0;
                sh.next_chunk2 = 0;
                sh.sub_done = 1;   // no subproblem: phase A buffers nothing, phase B streams all
                sh.nr = a.pass_nr;
                sh.nw = a.pass_nr;
            }
            if (t == 0 && tid < SVM_WS) {
                sh.r_row[tid] = tid < a.pass_nr ? a.pass_rows[tid] : 0;
                sh.c[tid] = tid < a.pass_nr ? a.pass_c[tid] : 0.0f;
            }
            __syncthreads();
        } else {
        // ---- a1 (1/3): wait for + stage this rank's CTA lists (16 key words each, decoded) -----
        if (tid == 0) sh.timeout = 0;
        {
            const uint64_t* src = rxw + (size_t)par * L * XW_PER_SLOT;
            constexpr int SW = 8;  // words per thread per batch: all loads in flight at once
            uint64_t t0 = 0;
            for (int base = 0; base < L * 16; base += SMO_THREADS * SW) {
                uint64_t w[SW];
#pragma unroll
                for (int u = 0; u < SW; ++u) {
                    const int i = base + tid + u * SMO_THREADS;
                    w[u] = i < L * 16 ? ld_relaxed_u64(src + (size_t)(i >> 4) * XW_PER_SLOT + (i & 15), sys)
                                      : tg;
                }
#pragma unroll
                for (int u = 0; u < SW; ++u) {
                    const int i = base + tid + u * SMO_THREADS;
                    if (i >= L * 16) continue;
                    const int sl = i >> 4, q = i & 15;
                    const uint64_t* pw = src + (size_t)sl * XW_PER_SLOT + q;
                    int spins = 0;
                    while ((w[u] & 0xffff000000000000ull) != tg) {
                        if (++spins == 256) {
                            spins = 0;
                            const uint64_t now = globaltimer_ns();
                            if (t0 == 0) t0 = now;
                            else if (now - t0 > a.timeout_ns) { sh.timeout = 1; break; }
                        }
                        w[u] = ld_relaxed_u64(pw, sys);
                    }
                    uint64_t key = 0;
                    const uint32_t score = (uint32_t)(w[u] >> 16);
                    if (score) {
                        const uint64_t Rr = (uint64_t)R;
                        const uint64_t pos = w[u] & 0xffffull;
                        const uint64_t c = pos >= Rr ? 1 : 0;
                        const uint64_t row = (uint64_t)v.row0 + (uint64_t)sl * Rr + pos - c * Rr;
                        const uint64_t g = c * (uint64_t)a.n_global + row;
                        key = ((uint64_t)score << 32) | (uint64_t)(0xffffffffu - (uint32_t)g);
                    }
                    (q < 8 ? sKU : sKL)[sl * 8 + (q & 7)] = key;
                }
            }
        }
        __syncthreads();
        auto report_exchange = [&]() {   // a shared load first: the barrier is DEFER_BLOCKING
            if (reporter && tid == 0) {
                const int vv = *reinterpret_cast<volatile int*>(&sh.timeout);
                const uint32_t dt = (uint32_t)clock() - x_pub + (uint32_t)(vv & 0);
                atomicAdd(reinterpret_cast<unsigned long long*>(&a.info->exch_cycles), (unsigned long long)dt);
                atomicAdd(&a.info->exch_hist[exch_bin(dt)], 1u);
            }
        };
        auto timed_out = [&]() {
            if (!sh.timeout) return false;
            if (reporter && tid == 0) a.info->error = 1;
            drain_wide();
            return true;
        };
        if (P == 1) report_exchange();
        mark(0);
        if (timed_out()) return;
        // ---- a1 (2/3): merge of the rank's L <= 256 lists (warp 0: I_up top-8, warp 1: I_low
        // top-8).  Two levels: 8 warps per side merge <= 32 lists each (one per lane), then one
        // warp per side merges the 8 partial top-8 lists.  src = (rank << 24) | (CTA slot << 4) |
        // candidate word (0-7 up, 8-15 low) throughout.
        wmark(-1);
        {
            const int side = warp >> 3, part = warp & 7;
            const uint64_t* keys = side == 0 ? sKU : sKL;
            const int per = (L + 7) >> 3, l0 = part * per;
            const int nl = max(0, min(per, L - l0));
            const int32_t sbase = (v.rank << 24) | (side << 3);
#ifdef SMO_PROFILE
            const long long c0 = clock64();
#endif
            lane_list_merge(nl, [&](int i, int j) { return lds_u64(keys + (l0 + i) * 8 + j); },
                            [&](int i, int j) { return sbase | ((l0 + i) << 4) | j; },
                            sh.gm_key[side][part], sh.gm_src[side][part], lane);
#ifdef SMO_PROFILE
            {   // I-cache probe: the same merge again (warm instructions), into scratch
                uint64_t sk[8]; int32_t ss[8];
                const int v0 = *reinterpret_cast<volatile int*>(&sh.nw);
                const long long c1 = clock64() + (v0 & 0);
                lane_list_merge(nl, [&](int i, int j) { return lds_u64(keys + (l0 + i) * 8 + j); },
                                [&](int i, int j) { return sbase | ((l0 + i) << 4) | j; }, sk, ss, lane);
                const int v1 = *reinterpret_cast<volatile int*>(&sh.nw);
                const long long c2 = clock64() + (v1 & 0) + (long long)(sk[0] & 0);
                if (warp == 0) { wprof[6] += c1 - c0; wprof[7] += c2 - c1; }
            }
#endif
        }
        __syncthreads();
        if (warp < 2) {
            uint64_t* out = warp == 0 ? sh.win_up : sh.win_low;
            int32_t* srcs = warp == 0 ? sh.win_up_src : sh.win_low_src;
            lane_list_merge(8, [&](int i, int j) { return lds_u64(&sh.gm_key[warp][i][j]); },
                            [&](int i, int j) { return sh.gm_src[warp][i][j]; }, out, srcs, lane);
        }
        __syncthreads();
        if (P > 1) {
            // ---- a1 (3/3), world > 1: CTA 0 of every rank publishes the rank's merged 8 + 8 list
            // into every rank's rank level; every CTA stages the P lists and merges them.  The
            // global top-8 is contained in the union of the per-rank top-8s, so this is exact.
            if (v.cta == 0 && tid < 16) {
                const uint64_t k = tid < 8 ? sh.win_up[tid] : sh.win_low[tid - 8];
                const int32_t s = tid < 8 ? sh.win_up_src[tid] : sh.win_low_src[tid - 8];
                uint64_t w0 = tg, w1 = tg;
                if (k) {
                    const uint64_t g = key_index(k);
                    const int c = g >= (uint64_t)a.n_global ? 1 : 0;
                    const int64_t li = (int64_t)(g - (uint64_t)c * a.n_global) - v.row0;
                    const int blk = (s >> 4) & 0xfffff;
                    const uint64_t pos = (uint64_t)c * (uint64_t)R + (uint64_t)(li - (int64_t)blk * R);
                    w0 = tg | ((k >> 32) << 16) | (uint64_t)blk;
                    w1 = tg | ((uint64_t)(s & 15) << 16) | pos;
                }
                const size_t base = ((size_t)par * SVM_MAX_RANKS + v.rank) * XW_RANK_SLOT + 2 * tid;
                for (int r = 0; r < P; ++r) {
                    uint64_t* dst = a.peer_xw[r] + base;
                    st_relaxed_u64(dst + 1, w1, sys);
                    st_relaxed_u64(dst, w0, sys);
                }
            }
            if (tid < P * 16) {
                const int o = tid >> 4, cnd = tid & 15;
                const uint64_t* pw = rxr + ((size_t)par * SVM_MAX_RANKS + o) * XW_RANK_SLOT + 2 * cnd;
                uint64_t w0 = ld_relaxed_u64(pw, sys), w1 = ld_relaxed_u64(pw + 1, sys);
                uint64_t t0 = 0;
                int spins = 0;
                while ((w0 & 0xffff000000000000ull) != tg || (w1 & 0xffff000000000000ull) != tg) {
                    if (++spins == 256) {
                        spins = 0;
                        const uint64_t now = globaltimer_ns();
                        if (t0 == 0) t0 = now;
                        else if (now - t0 > a.timeout_ns) { sh.timeout = 1; break; }
                    }
                    w0 = ld_relaxed_u64(pw, sys);
                    w1 = ld_relaxed_u64(pw + 1, sys);
                }
                uint64_t key = 0;
                int32_t src = -1;
                const uint32_t score = (uint32_t)(w0 >> 16);
                if (score) {
                    const uint64_t blk = w0 & 0xffffull, pos = w1 & 0xffffull, q = (w1 >> 16) & 0xfull;
                    const uint64_t Rr = (uint64_t)a.rank_rpc[o];
                    const uint64_t c = pos >= Rr ? 1 : 0;
                    const uint64_t row = (uint64_t)a.rank_row0[o] + blk * Rr + pos - c * Rr;
                    const uint64_t g = c * (uint64_t)a.n_global + row;
                    key = ((uint64_t)score << 32) | (uint64_t)(0xffffffffu - (uint32_t)g);
                    src = (int32_t)(((uint32_t)o << 24) | ((uint32_t)blk << 4) | (uint32_t)q);
                }
                sh.rk_key[cnd >> 3][o * 8 + (cnd & 7)] = key;
                sh.rk_src[cnd >> 3][o * 8 + (cnd & 7)] = src;
            }
            __syncthreads();
            report_exchange();
            if (timed_out()) return;
            if (warp < 2) {
                uint64_t* out = warp == 0 ? sh.win_up : sh.win_low;
                int32_t* srcs = warp == 0 ? sh.win_up_src : sh.win_low_src;
                lane_list_merge(P, [&](int i, int j) { return lds_u64(&sh.rk_key[warp][i * 8 + j]); },
                                [&](int i, int j) { return sh.rk_src[warp][i * 8 + j]; }, out, srcs, lane);
            }
            __syncthreads();
        }
        if (warp == 0) {
            // W = sorted union of |W|/2 up winners and |W|/2 low winners, deduplicated
            const int half = a.q >> 1;
            uint64_t key = 0;
            int32_t src = -1;
            if (lane < 8 && lane < half) {
                key = sh.win_up[lane];
                if (key) src = sh.win_up_src[lane];
            } else if (lane >= 8 && lane < 16 && lane - 8 < half) {
                key = sh.win_low[lane - 8];
                if (key) src = sh.win_low_src[lane - 8];
            }
            const uint64_t g = key ? key_index(key) : ~0ull;
            bool valid = key != 0;
            uint64_t gj[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) gj[j] = __shfl_sync(FULL, g, j);
            if (lane >= 8 && lane < 16) {
#pragma unroll
                for (int j = 0; j < 8; ++j) valid = valid && gj[j] != g;
            }
            valid = valid && lane < 16;
            const uint32_t vm = __ballot_sync(FULL, valid);
            int rank = 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) rank += (((vm >> j) & 1u) && gj[j] < g) ? 1 : 0;
            const int nw = __popc(vm);
            const int64_t row = valid ? (int64_t)(g >= (uint64_t)a.n_global ? g - a.n_global : g) : -1;
            if (valid) {
                sh.w_gidx[rank] = (int64_t)g;
                sh.w_src[rank] = src;
            }
            // distinct rows in position order (eps-SVR may select both copies of one row)
            int64_t rowp[16];
            int rk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                rowp[j] = __shfl_sync(FULL, row, j);
                rk[j] = __shfl_sync(FULL, rank, j);
            }
            int64_t myrow = -1;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (((vm >> j) & 1u) && rk[j] == lane) myrow = rowp[j];
            int fo = lane;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (((vm >> j) & 1u) && rowp[j] == myrow && rk[j] < fo) fo = rk[j];
            const uint32_t firsts = __ballot_sync(FULL, lane < nw && fo == lane);
            if (lane < nw) {
                const int sl = __popc(firsts & ((1u << fo) - 1u));
                sh.w_slot[lane] = sl;
                if (fo == lane) sh.r_row[sl] = myrow;
            }
            if (lane == 0) {
                sh.nw = nw;
                sh.nr = __popc(firsts);
                const uint64_t ku0 = sh.win_up[0], kl0 = sh.win_low[0];
                sh.m_up = ku0 ? (double)unord_f32((uint32_t)(ku0 >> 32)) : -INFINITY;
                sh.M_low = kl0 ? -(double)unord_f32((uint32_t)(kl0 >> 32)) : INFINITY;
                sh.stop = (sh.m_up - sh.M_low <= a.tol) || (t >= a.max_iter) || nw == 0;
                sh.next_chunk = 0;
                sh.next_chunk2 = 0;
                sh.sub_done = 0;
            }
            if (a.cache_slots > 0 && sh.c_off) {   // switched off: plain passes, no inserts
                if (lane < SVM_WS) { sh.c_slot[lane] = -1; sh.c_ins[lane] = -1; }
                if (lane == 0) sh.c_mode = 0;
            } else if (a.cache_slots > 0) {
                // ---- kernel-column cache: this CTA's 4-way set-associative LRU of
                // K(x_i, x_r) columns over its rows.  Every CTA takes the same decisions from the
                // same W sequence; tags and stamps are per CTA (global, L1-resident).  A hit
                // refreshes the stamp; a miss takes its set's least recently used way that no W row
                // of this iteration uses (not when an earlier missing W row has the same set), and
                // its column is written by this iteration's pass.  All W rows hit -> cache pass.
                __syncwarp();
                const int nrr = __popc(firsts);
                const int nsets = a.cache_slots >> 2;
                int32_t* ctag = a.cache_tag + (size_t)blockIdx.x * a.cache_slots;
                uint32_t* cstamp = a.cache_stamp + (size_t)blockIdx.x * a.cache_slots;
                const uint32_t now = (uint32_t)(t + 1);
                const bool mine = lane < nrr;
                const int64_t crow = mine ? sh.r_row[lane] : 0;
                const int cset = mine ? (int)(crow % nsets) : -1;
                int hitw = -1;
                if (mine) {
                    const int4 tg = *reinterpret_cast<const int4*>(ctag + cset * 4);
                    const int cr = (int)crow;
                    hitw = tg.x == cr ? 0 : tg.y == cr ? 1 : tg.z == cr ? 2 : tg.w == cr ? 3 : -1;
                    if (hitw >= 0) cstamp[cset * 4 + hitw] = now;
                }
                const uint32_t hm = __ballot_sync(FULL, hitw >= 0);
                const uint32_t all = nrr >= 32 ? FULL : ((1u << nrr) - 1u);
                const bool allhit = nrr > 0 && hm == all;
                const uint32_t mm = all & ~hm;
                int sets[SVM_WS];
#pragma unroll
                for (int q = 0; q < SVM_WS; ++q) sets[q] = __shfl_sync(FULL, cset, q);
                __syncwarp();
                int ins = -1;
                if (mine && hitw < 0 && !allhit) {
                    bool first = true;
#pragma unroll
                    for (int q = 0; q < SVM_WS; ++q)
                        if (q < lane && ((mm >> q) & 1u) && sets[q] == cset) first = false;
                    if (first) {
                        const uint4 sp = *reinterpret_cast<const uint4*>(cstamp + cset * 4);
                        const uint32_t s4[4] = {sp.x, sp.y, sp.z, sp.w};
                        int best = -1;
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            if (s4[w] != now && (best < 0 || s4[w] < s4[best])) best = w;
                        if (best >= 0) {
                            ctag[cset * 4 + best] = (int32_t)crow;
                            cstamp[cset * 4 + best] = now;
                            ins = cset * 4 + best;
                        }
                    }
                }
                if (lane < SVM_WS) {
                    sh.c_slot[lane] = hitw >= 0 ? cset * 4 + hitw : -1;
                    sh.c_ins[lane] = ins;
                }
                if (lane == 0) {
                    sh.c_mode = allhit ? 2 : 1;
                    // the cache switches itself off when it cannot pay: from iteration 8192 on,
                    // a 2048-iteration window with a row hit rate below 5% (c5: a 940k-SV active
                    // set, 1,600 affordable columns, 0.5% row hits; c4: > 20% already while the
                    // cache fills, 72% overall -- its cache passes only start once the active set
                    // shrinks, so their rate is no early criterion) -- the same decision in every
                    // CTA (the same W history)
                    sh.c_wh += allhit ? 1 : 0;
                    sh.c_rh += __popc(hm);
                    sh.c_rl += nrr;
                    if (((t + 1) & 2047) == 0) {
                        if (t + 1 >= 8192 && sh.c_rh * 20 < sh.c_rl) sh.c_off = 1;
                        sh.c_wh = sh.c_rh = sh.c_rl = 0;
                    }
                    if (reporter) {
                        a.info->cache_lookups += nrr;
                        a.info->cache_hits += __popc(hm);
                        a.info->cache_allhit += allhit ? 1 : 0;
                    }
                }
            }
        }
        __syncthreads();
        mark(1);
        if (sh.stop) {
            drain_wide();
            if (reporter && tid == 0) {
                a.info->iterations = t;
                a.info->m_up = sh.m_up;
                a.info->M_low = sh.M_low;
                a.info->converged = (sh.m_up - sh.M_low <= a.tol) ? 1 : 0;
                atomicAdd(reinterpret_cast<unsigned long long*>(&a.info->loop_cycles), (unsigned long long)clock64());
            }
#ifdef SMO_PROFILE
            if (reporter && tid == SOLVER_WARP * 32)
                for (int ph = 0; ph < 8; ++ph) a.info->phase_cycles[ph] = prof[ph];
            if (reporter && tid == 0)
                for (int ph = 0; ph < 8; ++ph) a.info->phase_cycles[8 + ph] = wprof[ph];
#endif
            return;
        }
        }   // !pass_only
        // ---- a2 setup: X_W rows (fp32 [d][16], for the pass and for K_WW), their
        // norms and the W payloads; one warp per row, no integer division -------------------
        const int nw = sh.nw, nr = sh.nr;
        if (!a.pass_only || t == 0) {
        if constexpr (CSR) {
            for (int i = tid; i < d * WS; i += SMO_THREADS) sXW[i] = 0.0f;
            if (sell)
                for (int i = tid; i <= d; i += SMO_THREADS) sMask[i] = 0u;
        } else {
            for (int i = tid; i < d * SVM_WS; i += SMO_THREADS)
                if ((i & 15) >= nr) sXW[i] = 0.0f;
        }
        if constexpr (CSR) __syncthreads();
        if (!a.pass_only && warp == SMO_WARPS - 1 && lane < nw) {  // payloads of W (tagged words,
            // in the owner rank's local level: src = (rank << 24) | (CTA slot << 4) | candidate)
            const int p = lane;
            const int32_t s = sh.w_src[p];
            const int o = s >> 24, blk = (s >> 4) & 0xfffff, q = s & 15;
            const uint64_t* pl = a.peer_xw[o] + XW_RANK_WORDS +
                                 ((size_t)par * a.rank_nblk[o] + blk) * XW_PER_SLOT + 16 + 3 * q;
            uint64_t w0 = ld_relaxed_u64(pl, sys), w1 = ld_relaxed_u64(pl + 1, sys),
                     w2 = ld_relaxed_u64(pl + 2, sys);
            while ((w0 & 0xffff000000000000ull) != tg) w0 = ld_relaxed_u64(pl, sys);
            while ((w1 & 0xffff000000000000ull) != tg) w1 = ld_relaxed_u64(pl + 1, sys);
            while ((w2 & 0xffff000000000000ull) != tg) w2 = ld_relaxed_u64(pl + 2, sys);
            const uint64_t ab = ((w0 & 0xffffffffffffull) << 16) | ((w1 >> 32) & 0xffffull);
            sh.w_alpha[p] = __longlong_as_double((long long)ab);
            sh.w_G[p] = (double)__uint_as_float((uint32_t)w1);
            sh.w_y[p] = ((uint32_t)w2 & ST_YPOS) ? 1 : -1;
        }
        if (warp < nr) {  // one warp per distinct W row (coalesced along the row)
            const int r = warp;
            const int64_t row = sh.r_row[r];
            const int o = owner_rank(a, row);
            const int64_t lr = row - a.rank_row0[o];
            if constexpr (!CSR) {
                const float* src = a.peer_XR[o] + lr * a.d;
                for (int k0 = 0; k0 < d; k0 += 8 * 32) {  // 8 loads in flight per lane
                    float xv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int k = k0 + u * 32 + lane;
                        xv[u] = k < d ? __ldg(src + k) : 0.0f;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int k = k0 + u * 32 + lane;
                        if (k < d) sXW[k * SVM_WS + r] = xv[u];
                    }
                }
            } else {
                const int64_t b = a.peer_indptr[o][lr], e = a.peer_indptr[o][lr + 1];
                for (int64_t p = b + lane; p < e; p += 32) {
                    const int k = a.peer_indices[o][p];
                    const float xv = a.peer_vals[o][p];
                    sXW[k * WS + r] = xv;
                    if (xv != 0.0f)   // group mask
                        atomicOr(sell ? sMask + k : reinterpret_cast<unsigned int*>(sXW + csr_mask_slot(k)),
                                 sell ? 1u << (r >> 2) : 1u << r);   // SELL: 4-row group bits
                }
            }
            if (lane == 0) sh.xn[r] = a.peer_xnorm[o][lr];
        }
        if (tid >= nr && tid < SVM_WS) sh.xn[tid] = 0.0f;
        __syncthreads();
        }   // X_W staged (once in pass-only mode)
        mark(2);
        wmark(-1);
        // ---- K between the distinct W rows in fp64 ---------------------------------------------
        if (!CSR && !a.pass_only && a.qww_mma) {
            // Gram X_W X_W^T on the fp64 tensor cores (mma.sync m8n8k4, as the batched solve):
            // warps 0-5 = 3 8x8 tiles x 2 k-parts, operands promoted exactly from the fp32 tile,
            // parts summed in a fixed order; RBF distance G_aa + G_bb - 2 G_ab clamped at 0
            // (exactly 0 on the diagonal)
            double* gpart = sh.qpart;                 // [2 parts][3 tiles][64]
            double* gram = sh.kpos;                   // [16][16] (kpos is rebuilt from kr below)
            const int dp4 = (d + 3) & ~3, nsteps = dp4 >> 2;
            if (warp < 6) {
                const int tl = warp >> 1, part = warp & 1;
                const int I = tl == 2 ? 1 : 0, J = tl == 0 ? 0 : 1;
                const int ra = I * 8 + (lane >> 2), rb = J * 8 + (lane >> 2), kk = lane & 3;
                double c0 = 0.0, c1 = 0.0;
                for (int st = part; st < nsteps; st += 2) {
                    const int k = 4 * st + kk;
                    const double a0 = k < d ? (double)sXW[k * SVM_WS + ra] : 0.0;
                    const double b0 = k < d ? (double)sXW[k * SVM_WS + rb] : 0.0;
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(c0), "+d"(c1) : "d"(a0), "d"(b0));
                }
                gpart[(part * 3 + tl) * 64 + (lane >> 2) * 8 + (lane & 3) * 2] = c0;
                gpart[(part * 3 + tl) * 64 + (lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1;
            }
            __syncthreads();
            if (tid < SVM_WS * SVM_WS) {
                const int ra = tid >> 4, rb = tid & 15;
                const bool sw = (ra >> 3) > (rb >> 3);
                const int I = sw ? rb >> 3 : ra >> 3, J = sw ? ra >> 3 : rb >> 3;
                const int tl = I == 0 ? (J == 0 ? 0 : 1) : 2;
                const int e = sw ? (rb & 7) * 8 + (ra & 7) : (ra & 7) * 8 + (rb & 7);
                gram[tid] = gpart[tl * 64 + e] + gpart[(3 + tl) * 64 + e];
            }
            __syncthreads();
            wmark(6);
            if (tid < SVM_WS * SVM_WS) {
                const int ra = tid >> 4, rb = tid & 15;
                if (ra < nr && rb < nr) {
                    double dv = gram[tid];
                    if (a.kp.kernel == 2) {
                        dv = ra == rb ? 0.0 : gram[ra * 17] + gram[rb * 17] - 2.0 * gram[tid];
                        dv = dv > 0.0 ? dv : 0.0;
                    }
                    sh.kr[tid] = kernel_fp64_from(dv, a.kp);
                }
            }
            __syncthreads();
            wmark(7);
            if (tid < SVM_WS * SVM_WS) {
                const int pa = tid >> 4, pb = tid & 15;
                double kab = 0.0, ie = 0.0;
                if (pa < nw && pb < nw) {
                    const int sa = sh.w_slot[pa], sb = sh.w_slot[pb];
                    kab = sh.kr[sa * SVM_WS + sb];
                    const double eta = sh.kr[sa * SVM_WS + sa] + sh.kr[sb * SVM_WS + sb] - 2.0 * kab;
                    ie = 1.0 / (eta < 1e-12 ? 1e-12 : eta);
                }
                sh.kpos[tid] = kab;
                sh.inv_eta[tid] = ie;
            }
            __syncthreads();
        } else if (!a.pass_only) {
            // k-split pair sums from the fp32 tile (all threads, up to 4 parts per pair)
            const int npairs = nr * (nr + 1) / 2;
            const int kp = max(1, min(4, SMO_THREADS / max(npairs, 1)));
            const int klen = ((d + kp - 1) / kp + 3) & ~3;
            if (tid < npairs * kp) {
                // part-major: the lanes of a warp share one k range and walk consecutive pairs
                // (same row r, columns s = r..15): broadcast / distinct-bank loads instead of the
                // 3-way conflicts of pair-major parts (k offsets 36 x 16 floats apart hit one
                // bank); each pair's per-part sums are unchanged (bit-identical)
                const int part = tid / npairs, p = tid - part * npairs;
                int r = 0, rem = p;
                while (rem >= nr - r) { rem -= nr - r; ++r; }
                const int sidx = r + rem;
                double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
                // from the fp32 [d][WS] tile (the fp32 inputs promoted exactly): four interleaved
                // fp64 accumulators over k, features >= d contribute exact zeros
                if (sidx != r || a.kp.kernel != 2) {
                    const int k0 = part * klen, k1 = min(k0 + klen, dp);
                    const float* xr = sXW + r;
                    const float* xs = sXW + sidx;
                    auto ld = [&](const float* x, int k) { return k < d ? (double)x[k * WS] : 0.0; };
                    if (a.kp.kernel == 2) {
#pragma unroll 2
                        for (int k = k0; k < k1; k += 4) {
                            const double t0 = ld(xr, k) - ld(xs, k), t1 = ld(xr, k + 1) - ld(xs, k + 1);
                            const double t2 = ld(xr, k + 2) - ld(xs, k + 2), t3 = ld(xr, k + 3) - ld(xs, k + 3);
                            acc0 = fma(t0, t0, acc0);
                            acc1 = fma(t1, t1, acc1);
                            acc2 = fma(t2, t2, acc2);
                            acc3 = fma(t3, t3, acc3);
                        }
                    } else {
#pragma unroll 2
                        for (int k = k0; k < k1; k += 4) {
                            acc0 = fma(ld(xr, k), ld(xs, k), acc0);
                            acc1 = fma(ld(xr, k + 1), ld(xs, k + 1), acc1);
                            acc2 = fma(ld(xr, k + 2), ld(xs, k + 2), acc2);
                            acc3 = fma(ld(xr, k + 3), ld(xs, k + 3), acc3);
                        }
                    }
                }
                sh.qpart[p * 4 + part] = (acc0 + acc1) + (acc2 + acc3);
            }
            __syncthreads();
            wmark(6);
            if (tid < npairs) {
                int r = 0, rem = tid;
                while (rem >= nr - r) { rem -= nr - r; ++r; }
                const int sidx = r + rem;
                double dsum = 0.0;
                for (int part = 0; part < kp; ++part) dsum += sh.qpart[tid * 4 + part];
                const double kv = kernel_fp64_from(dsum, a.kp);
                sh.kr[r * SVM_WS + sidx] = kv;
                sh.kr[sidx * SVM_WS + r] = kv;
            }
            __syncthreads();
            wmark(7);
            if (tid < SVM_WS * SVM_WS) {
                const int pa = tid >> 4, pb = tid & 15;
                double kab = 0.0, ie = 0.0;
                if (pa < nw && pb < nw) {
                    const int sa = sh.w_slot[pa], sb = sh.w_slot[pb];
                    kab = sh.kr[sa * SVM_WS + sb];
                    const double eta = sh.kr[sa * SVM_WS + sa] + sh.kr[sb * SVM_WS + sb] - 2.0 * kab;
                    ie = 1.0 / (eta < 1e-12 ? 1e-12 : eta);
                }
                sh.kpos[tid] = kab;
                sh.inv_eta[tid] = ie;
            }
            __syncthreads();
        }
        mark(3);

        uint64_t wlu = 0, wll = 0;  // this warp's running top-8 lists (exact, per chunk)
        const int nbuf = dbuf_rows / rows_per_chunk < nchunks ? dbuf_rows / rows_per_chunk : nchunks;
        // feature slicing (wide d, streamed X): every (chunk, slice) item is buffered in phase A
        const int nsl = a.nslice > 1 ? a.nslice : 1;
        const int ks = nsl > 1 ? (d + nsl - 1) / nsl : d;
        const int kmode = a.cache_slots > 0 ? sh.c_mode : 0;   // kernel-column cache mode
        float* kcache = a.cache_data ? a.cache_data + (a.virt ? v.row0 : 0) : nullptr;
        // cache pass: phase A copies the buffered chunks' cached K values into the dot buffer
        // while the subproblem runs (HBM is otherwise idle then); no dots anywhere
        const int nitems = kmode == 2 ? (nsl > 1 ? 0 : nbuf) : (nsl > 1 ? nchunks * nsl : nbuf);
        // ---- phase A: dot products x_i . X_W of the buffered chunks into shared memory --------
        auto phase_a = [&]() {
            for (;;) {
                // chunks are buffered only while the subproblem runs: once it is solved the rest
                // are cheaper fused with their epilogue in phase B (no tail of buffered work)
                int it = nitems;
                if (lane == 0 && (nsl > 1 || !*reinterpret_cast<volatile int32_t*>(&sh.sub_done)))
                    it = atomicAdd(&sh.next_chunk, 1);
                it = __shfl_sync(FULL, it, 0);
                if (it >= nitems) break;
                const int ch = nsl > 1 ? it / nsl : it, sl = nsl > 1 ? it - ch * nsl : 0;
                const int k0 = sl * ks, kn = min(d, k0 + ks) - k0;
                const int64_t lrow = cta_begin + (int64_t)ch * rows_per_chunk + lane * RPT;
                const int64_t li0 = lane_on ? lrow : cta_end;   // idle lanes: past the CTA's rows
                float acc[RPT][SVM_WS];
                if (kmode == 2) {   // the cached K columns of the W rows (K values, not dots)
#pragma unroll
                    for (int r = 0; r < SVM_WS; ++r) {
                        const int csl = sh.c_slot[r];
                        const float* src = kcache + (int64_t)(csl >= 0 ? csl : 0) * a.n_pad + li0;
                        const bool ok = csl >= 0 && li0 < cta_end;
                        if constexpr (RPT == 4) {
                            const float4 kv = ok ? *reinterpret_cast<const float4*>(src) : make_float4(0.f, 0.f, 0.f, 0.f);
                            acc[0][r] = kv.x; acc[1][r] = kv.y; acc[2][r] = kv.z; acc[3][r] = kv.w;
                        } else if constexpr (RPT == 2) {
                            const float2 kv = ok ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
                            acc[0][r] = kv.x; acc[1][r] = kv.y;
                        } else {
                            acc[0][r] = ok ? *src : 0.0f;
                        }
                    }
                }
                else if constexpr (CSR) csr_dots(ch, li0, acc);
                else if (tma) {
                    const uint64_t T = (uint64_t)t * nchunks + ch;
                    dots_tile<RPT>(tma_acquire(T), d, lane, sXW, acc);
                    tma_release(T);
                }
                else if (XS || !a.x_ring) dots_dense<RPT>(xbase + (li0 - cta_begin) + (int64_t)k0 * xld, xld, kn, li0 < cta_end, sXW + k0 * SVM_WS, acc);
                else dots_dense_async<RPT>(xbase + (li0 - cta_begin) + (int64_t)k0 * xld, xld, kn, li0 < cta_end, sXW + k0 * SVM_WS, xring, acc);
                const int lr = (int)(lrow - cta_begin);
#pragma unroll
                for (int r = 0; r < SVM_WS; ++r) {
                    if (!lane_on) break;
                    float* dst = sDot + (size_t)(sl * SVM_WS + r) * dbuf_rows + lr;
                    if constexpr (RPT == 4) *reinterpret_cast<float4*>(dst) = make_float4(acc[0][r], acc[1][r], acc[2][r], acc[3][r]);
                    else if constexpr (RPT == 2) *reinterpret_cast<float2*>(dst) = make_float2(acc[0][r], acc[1][r]);
                    else *dst = acc[0][r];
                }
            }
        };
        if (warp == SOLVER_WARP && !a.pass_only) {
            // ---- a2: the subproblem on the solver warp (the highest warp id: the SM's warp
            // arbiter favours high ids), overlapped with phase A on the other warps ------------
            const int steps = solve_subproblem(sh, nw, a.C, a.inner_tol, a.inner_max, lane);
            if (lane == 0) *reinterpret_cast<volatile int32_t*>(&sh.sub_done) = 1;
            __syncwarp();
            if (lane < nw) sh.w_dalpha[lane] = sh.w_anew[lane] - sh.w_alpha[lane];
            __syncwarp();
            if (lane < SVM_WS) {
                double cr = 0.0;
                for (int b = 0; b < nw; ++b)
                    if (sh.w_slot[b] == lane) cr += (double)sh.w_y[b] * sh.w_dalpha[b];
                sh.c[lane] = lane < nr ? (float)cr : 0.0f;
            }
            // the owner writes alpha and status of its W entries (before the pass reads status)
            if (lane < nw) {
                const int64_t g = sh.w_gidx[lane];
                const int c = g >= a.n_global ? 1 : 0;
                const int64_t li = g - (int64_t)c * a.n_global - v.row0;
                if (li >= cta_begin && li < cta_end) {
                    const int64_t idx = (int64_t)c * a.n_pad + li;
                    v.alpha[idx] = sh.w_anew[lane];
                    v.status[idx] = make_status(sh.w_y[lane], sh.w_anew[lane], a.C);
                }
            }
            if (reporter) {
                if (lane < nw) {
                    a.info->last_w[lane] = sh.w_gidx[lane];
                    a.info->last_dalpha[lane] = sh.w_dalpha[lane];
                }
                if (lane == 0) {
                    a.info->last_nw = nw;
                    a.info->last_inner = steps;
                    a.info->inner_total += steps;
                }
            }
            mark(4);
        }
        if (wide) {
            // ---- a3 in wide mode: consumer warps stream every feature stage through registers,
            // then (after the subproblem) the epilogue of their own rows -------------------------
            float acc[RPT][SVM_WS];
            const int lr = warp * 32 + lane;   // this lane's local row
            if (warp < ncw) {
                zero_acc<RPT>(acc);
                const uint64_t Tb = (uint64_t)t * nst;
                wmark(-1);
                for (int j = 0; j < nst; ++j) {
                    const uint64_t T = Tb + j;
                    const int s = (int)(T % WIDE_STAGES);
                    mbar_wait(&sh.mb_full[s], (uint32_t)((T / WIDE_STAGES) & 1));
                    wmark(0);
                    const float* st = wring + (size_t)s * wkc * Rs + lr;
                    const int k0 = j * wkc, kn = min(wkc, d - k0);
                    const float4* w4 = reinterpret_cast<const float4*>(sXW + k0 * SVM_WS);
#pragma unroll 4
                    for (int q = 0; q < kn; ++q) {
                        const float4 wv[4] = {w4[4 * q], w4[4 * q + 1], w4[4 * q + 2], w4[4 * q + 3]};
                        fma_row16(st[(size_t)q * Rs], wv, acc[0]);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sh.mb_empty[s]);
                    wmark(1);
                }
            } else if (warp == ncw && lane == 0) {
                const uint64_t Tb = (uint64_t)t * nst + WIDE_STAGES;
                for (int j = 0; j < nst; ++j) {
                    const uint64_t T = Tb + j;
                    mbar_wait(&sh.mb_empty[T % WIDE_STAGES], (uint32_t)(((T / WIDE_STAGES) - 1) & 1));
                    wide_issue(T);
                }
            }
            __syncthreads();
            mark(5);
            wmark(-1);
            if (warp < ncw) {
                uint64_t ku[2 * RPT], kl[2 * RPT];
                row_epilogue<RPT, RBFK>(a, v, sh, cta_begin + lr, cta_end, true, acc, ku, kl);
                merge_chunk_rows<RPT>(ku, kl, wlu, wll, lane, a.ncopy);
            }
        } else {
        // overlap == 2 (default): the warps sharing the solver's SM sub-partition (warp % 4 == 3) leave
        // its issue slots to the subproblem and join phase A when it is solved
        if (a.overlap == 2 && (warp & 3) == (SOLVER_WARP & 3)) named_bar_sync(1, 32 * (SMO_WARPS / 4));
        phase_a();   // the solver warp joins phase A once its subproblem is done
        __syncthreads();
        mark(5);
        wmark(-1);
        // ---- phase B / a3: epilogue of every chunk (buffered dots, or computed now) ----------
        // chunks [0, nA) have buffered dots; the streamed ones [nA, nchunks) are handed out
        // first so that their X reads start together and no streamed chunk forms the tail
        const int nA = nitems == 0 ? 0 : (nsl > 1 ? nchunks : (sh.next_chunk < nbuf ? sh.next_chunk : nbuf));
        const int nS = nchunks - nA;
        for (;;) {
            int tk = 0;
            if (lane == 0) tk = atomicAdd(&sh.next_chunk2, 1);
            tk = __shfl_sync(FULL, tk, 0);
            if (tk >= nchunks) break;
            const int ch = tk < nS ? nA + tk : tk - nS;
            const int64_t lrow = cta_begin + (int64_t)ch * rows_per_chunk + lane * RPT;
            const int64_t li0 = lane_on ? lrow : cta_end;   // idle lanes: past the CTA's rows
            float acc[RPT][SVM_WS];
            int ekmode = kmode;   // the epilogue's kernel-value source
            if (kmode == 2 && ch >= nA) {
                zero_acc<RPT>(acc);   // (unused: K comes from the cache)
            } else if (ch < nA) {
                if (kmode == 2) ekmode = 3;   // the buffer holds cached K values

                const int lr = lane_on ? (int)(lrow - cta_begin) : 0;
#pragma unroll
                for (int r = 0; r < SVM_WS; ++r) {
                    const float* src = sDot + (size_t)r * dbuf_rows + lr;
                    if constexpr (RPT == 4) {
                        const float4 dv = *reinterpret_cast<const float4*>(src);
                        acc[0][r] = dv.x; acc[1][r] = dv.y; acc[2][r] = dv.z; acc[3][r] = dv.w;
                    } else if constexpr (RPT == 2) {
                        const float2 dv = *reinterpret_cast<const float2*>(src);
                        acc[0][r] = dv.x; acc[1][r] = dv.y;
                    } else {
                        acc[0][r] = *src;
                    }
                }
                for (int q = 1; q < nsl; ++q) {   // slice partials, added in slice order
#pragma unroll
                    for (int r = 0; r < SVM_WS; ++r)
#pragma unroll
                        for (int j = 0; j < RPT; ++j)
                            acc[j][r] += sDot[(size_t)(q * SVM_WS + r) * dbuf_rows + lr + j];
                }
            } else if constexpr (CSR) {
                csr_dots(ch, li0, acc);
            } else if (tma) {
                const uint64_t T = (uint64_t)t * nchunks + ch;
                dots_tile<RPT>(tma_acquire(T), d, lane, sXW, acc);
                tma_release(T);
            } else if (XS || !a.x_ring) {
                dots_dense<RPT>(xbase + (li0 - cta_begin), xld, d, li0 < cta_end, sXW, acc);
            } else {
                dots_dense_async<RPT>(xbase + (li0 - cta_begin), xld, d, li0 < cta_end, sXW, xring, acc);
            }
            wmark(0);
            uint64_t ku[2 * RPT], kl[2 * RPT];
            row_epilogue<RPT, RBFK>(a, v, sh, li0, cta_end, true, acc, ku, kl, ekmode, kcache);
            wmark(2);
            merge_chunk_rows<RPT>(ku, kl, wlu, wll, lane, a.ncopy);
            wmark(3);
        }
        }   // !wide
        wmark(4);
        finish_lists(wlu, wll);
        mark(6);
        wmark(5);
        if (!a.pass_only) publish(tag + 1);
        if (reporter && tid == 0) x_pub = (uint32_t)clock();
        mark(7);
    }
}

// Debug / parity view of the pass: K[i * nr + r] = K(x_i, x_rows[r]) for all local rows.
template <bool CSR>
__global__ void __launch_bounds__(256) kernel_rows_kernel(const SmoArgs a, const int64_t* rows,
                                                          int nr, float* K)
{
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    float* sXW = reinterpret_cast<float*>(dyn_smem);
    __shared__ float xn[SVM_WS];
    const int d = (int)a.d;
    constexpr int WS = CSR ? WSTR_CSR : SVM_WS;
    for (int i = threadIdx.x; i < d * WS; i += blockDim.x) sXW[i] = 0.0f;
    __syncthreads();
    if constexpr (!CSR) {
        for (int i = threadIdx.x; i < d * SVM_WS; i += blockDim.x) {
            int r = i / d, k = i - r * d;
            if (r < nr) sXW[k * SVM_WS + r] = a.peer_XR[0][rows[r] * a.d + k];
        }
    } else {
        for (int r = 0; r < nr; ++r) {
            int64_t b = a.peer_indptr[0][rows[r]], e = a.peer_indptr[0][rows[r] + 1];
            for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x) {
                const int k = a.peer_indices[0][p];
                const float v = a.peer_vals[0][p];
                sXW[k * WS + r] = v;
                if (v != 0.0f) atomicOr(reinterpret_cast<unsigned int*>(sXW + csr_mask_slot(k)), 1u << r);
            }
        }
    }
    if (threadIdx.x < SVM_WS) xn[threadIdx.x] = threadIdx.x < nr ? a.xnorm[rows[threadIdx.x]] : 0.0f;
    __syncthreads();
    int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= a.n_local) return;
    float acc[1][SVM_WS];
    if constexpr (CSR) dots_csr(a.indptr, a.indices, a.vals, li, true, sXW, acc);
    else dots_dense<1>(a.XT + li, a.n_pad, d, true, sXW, acc);
    float xi = a.xnorm[li];
    for (int r = 0; r < nr; ++r) K[li * nr + r] = kernel_from_dot(a.kp, acc[0][r], xi, xn[r]);
}


// ================================================================ batched one-vs-rest (8(f) #1)
// One iteration = k_ovr_solve (one CTA per problem: merge its candidates -> W, stop test, K_WW,
// subproblem, alpha / status of W, coefficients and its 16 columns of the U operand) followed by
// k_ovr_pass (one CTA per 128 training rows: D = X_rows X_U^T on tcgen05 3xTF32 into TMEM, then per
// problem the kernel values of its 16 columns, the G update and the tile's top-8 candidates).
// Each problem follows exactly the single-problem iteration of P:53 (same selection, subproblem and
// update rules); only the X pass is shared.
constexpr int OVR_THREADS = 512;

__device__ __forceinline__ void ovr_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0, spins = 0;
    uint64_t t0 = 0;
    for (;;) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (ok) return;
        if (++spins == 1024) {   // watchdog: a lost stage must fail the launch, not hang the GPU
            spins = 0;
            const uint64_t now = gtimer_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 5000000000ull) __trap();
        }
    }
}

// Pipelined persistent pass (one CTA per SM).  A CTA walks groups of OVR_T = 2 contiguous 128-row
// tiles; per group the features stream in K-chunks of OVR_KCH:
//   producer warp   : cp.async.bulk of the raw feature-major X chunk ([kch][256 rows]) and of the
//                     U chunk (hi | lo, pre-split by k_ovr_solve) into mbarrier rings;
//   converter warps : raw fp32 -> (hi, lo) tf32 split in the K-major core layout of the A operand;
//   MMA warp        : 3xTF32 (lo.hi, hi.lo, hi.hi) per 8-feature k-step, D[tile] in TMEM columns
//                     tile * NU (+ p * 16 for problem p), tcgen05.commit releases the slots;
//   epilogue warps  : per problem the kernel values of its 16 columns, G update, the tile's top-8.
// X is read from HBM exactly once per pass; the stages of consecutive chunks / groups overlap.
// Warp roles of k_ovr_pass
constexpr int OVR_W_A = 0, OVR_W_B = 1, OVR_W_MMA = 2, OVR_W_EPI = 3, OVR_EPI = 16;
constexpr int OVR_PASS_THREADS = (OVR_W_EPI + OVR_EPI) * 32;
constexpr int OVR_MAXRING = 8;                       // A / U ring slots (runtime a.na, a.nb <= this)
constexpr int OVR_ATILE = 2 * 128 * OVR_KCH;         // fp16 elements of one A chunk (hi | lo)

__device__ __forceinline__ void ovr_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void ovr_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void epi_bar()   // named barrier of the epilogue warps only
{
    asm volatile("bar.sync 1, %0;" ::"n"(OVR_EPI * 32) : "memory");
}
// wait with back-off (long waits of the epilogue warps: their spinning would take issue slots)
__device__ __forceinline__ void ovr_wait_sleep(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0;
    uint64_t t0 = 0;
    for (uint32_t spins = 0;; ++spins) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (ok) return;
        __nanosleep(32);
        if ((spins & 1023) == 1023) {
            const uint64_t now = gtimer_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 5000000000ull) __trap();
        }
    }
}

// Operand tiles of the batched pass: X (and U) are pre-split once into fp16 pairs
//   xs = sigma x,  h = fp16_rn(xs),  l = fp16_rn(xs - h)      (sigma a power of two)
// in the K-major SWIZZLE_NONE core layout of kind::f16 (core matrix 8 rows x 8 k = 128 B).
// D = hA hB + hA lB + lA hB (three kind::f16 MMAs, fp32 accumulation in TMEM) ~= sigma^2 x.u with
// the error of the dropped lA lB term (~2^-24 relative, the 3xTF32 level); the products of two
// 11-bit significands are exact in fp32.
__device__ __forceinline__ int kmaj16_off(int r, int k) { return ((r >> 3) * (OVR_KCH / 8) + (k >> 3)) * 64 + (r & 7) * 8 + (k & 7); }

// XH[tile][kc][hi | lo][128 x KCH] from row-major X (one pass at setup; rows >= n, k >= d are 0)
__global__ void k_ovr_xh(const float* __restrict__ XR, int64_t n, int64_t d, int nct, int nkc, float sigma,
                         uint16_t* __restrict__ XH)
{
    const int64_t total = (int64_t)nct * nkc * 16 * (OVR_KCH / 8) * 8;   // (tile, kc, row group, kq, row)
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int r7 = (int)(t & 7), kq = (int)((t >> 3) % (OVR_KCH / 8));
        const int64_t rest = (t >> 3) / (OVR_KCH / 8);
        const int rg = (int)(rest & 15);
        const int64_t tk = rest >> 4;                     // tile * nkc + kc
        const int kc = (int)(tk % nkc);
        const int64_t tile = tk / nkc;
        const int r = rg * 8 + r7;
        const int64_t row = tile * 128 + r;
        const int64_t f0 = (int64_t)kc * OVR_KCH + kq * 8;
        uint16_t h[8], l[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float x = (row < n && f0 + j < d) ? XR[row * d + f0 + j] : 0.0f;
            f16_split(x, sigma, h[j], l[j]);
        }
        uint16_t* base = XH + (size_t)tk * OVR_ATILE;
        const int off = kmaj16_off(r, kq * 8);
        uint4 hv, lv;
        hv.x = h[0] | ((uint32_t)h[1] << 16); hv.y = h[2] | ((uint32_t)h[3] << 16);
        hv.z = h[4] | ((uint32_t)h[5] << 16); hv.w = h[6] | ((uint32_t)h[7] << 16);
        lv.x = l[0] | ((uint32_t)l[1] << 16); lv.y = l[2] | ((uint32_t)l[3] << 16);
        lv.z = l[4] | ((uint32_t)l[5] << 16); lv.w = l[6] | ((uint32_t)l[7] << 16);
        *reinterpret_cast<uint4*>(base + off) = hv;
        *reinterpret_cast<uint4*>(base + 128 * OVR_KCH + off) = lv;
    }
}

// max |X| as float bits (non-negative floats order as unsigned integers)
__global__ void k_absmax(const float* __restrict__ X, int64_t count, unsigned int* __restrict__ out)
{
    float m = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(X[i]));
    m = fmaxf(m, __shfl_xor_sync(FULL, m, 16));
    m = fmaxf(m, __shfl_xor_sync(FULL, m, 8));
    m = fmaxf(m, __shfl_xor_sync(FULL, m, 4));
    m = fmaxf(m, __shfl_xor_sync(FULL, m, 2));
    m = fmaxf(m, __shfl_xor_sync(FULL, m, 1));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// Pipelined persistent pass (one CTA per SM) over 128-row tiles t = blockIdx.x + j gridDim.x:
//   producer    : per stage (K-chunk of 32 features) one cp.async.bulk of the tile's pre-split X
//   (warp 0)      (16 KB) and one of U (hi | lo, written by k_ovr_solve) into an mbarrier ring;
//                 the first stages' X is issued before griddepcontrol.wait (PDL), U after it;
//   (warp 1 idle: the epilogue warps' TMEM lane quadrant is warp mod 4)
//   MMA warp    : 3 kind::f16 MMAs per 16 features (M = 128, N = |U|), D[tile] in TMEM
//                 columns (j & 1) NU (double-buffered), tcgen05.commit releases the slots;
//   16 epilogue : per problem the kernel values of its 16 columns, G update, the tile's top-8;
//     warps       tile j's epilogue overlaps tile j + 1's MMAs.
// X is read from HBM exactly once per pass (4 B per element, as fp32).
__global__ void __launch_bounds__(OVR_PASS_THREADS, 1) k_ovr_pass(const OvrArgs a)
{
    extern __shared__ __align__(1024) unsigned char ovr_smem[];
    const int NU = a.NU, NA = a.na, NB = a.nb;
    const int bslot = 2 * NU * OVR_KCH;                                   // fp16 elements per U slot
    uint16_t* As = reinterpret_cast<uint16_t*>(ovr_smem);                 // [NA][hi | lo][128 x KCH]
    uint16_t* Bs = As + (size_t)NA * OVR_ATILE;                           // [NB][hi | lo][NU x KCH]
    float* sCoef = reinterpret_cast<float*>(Bs + (size_t)NB * bslot);     // [NU]
    float* sNorm = sCoef + OVR_MAXP * 16;                                 // [NU]
    uint64_t* wl = reinterpret_cast<uint64_t*>(sNorm + OVR_MAXP * 16);    // [P][2][128] tile keys
    uint64_t* bars = wl + (size_t)a.P * 2 * 128;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * OVR_MAXRING + 4);
    const uint32_t b_af = su32(bars), b_ae = b_af + 8 * OVR_MAXRING;
    const uint32_t b_bf = b_ae + 8 * OVR_MAXRING, b_be = b_bf + 8 * OVR_MAXRING;
    const uint32_t b_accf = b_be + 8 * OVR_MAXRING, b_acce = b_accf + 16;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nct = a.nct, nkc = a.nkc;
    long long pw0 = 0, pw1 = 0, pw2 = 0;   // profile: cycles in the role's waits / work

    // programmatic dependent launch: the next kernel (the solve) may be scheduled now; this grid's
    // reads of the solve's outputs (U, coefficients, G, status) wait for it (griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == OVR_W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_holder)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < NA; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_af + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_ae + 8 * i), "r"(1));
        }
        for (int i = 0; i < NB; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_bf + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_be + 8 * i), "r"(1));
        }
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_accf + 8 * i), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b_acce + 8 * i), "r"(OVR_EPI));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_holder;
    long long tp = clock64();
#define OVR_MARK(acc) { const long long _n = clock64(); acc += _n - tp; tp = _n; }

    if (warp == OVR_W_A) {
        // ---------------- producer: stage = (X chunk of the tile, U chunk), two bulk copies --------
        if (lane == 0) {
            const uint32_t abytes = (uint32_t)(OVR_ATILE * 2), bbytes = (uint32_t)(bslot * 2);
            int sa = 0;
            uint32_t pe = 1;   // parity of use u = c / NA >= 1 is (u - 1) & 1
            int c = 0;
            // X does not depend on the previous kernel: the first NA stages' X chunks are issued
            // before griddepcontrol.wait, their U chunks (written by the solve) after it
            const int npre = min(NA, (int)((nct - blockIdx.x + gridDim.x - 1) / gridDim.x) * nkc);
            for (int j = 0; j < npre; ++j) {
                const int t = blockIdx.x + (j / nkc) * gridDim.x, kc = j % nkc;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b_af + 8 * j), "r"(abytes + bbytes) : "memory");
                ovr_bulk(su32(As + (size_t)j * OVR_ATILE), a.XH + ((size_t)t * nkc + kc) * OVR_ATILE, abytes, b_af + 8 * j);
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
            for (int j = 0; j < npre; ++j)
                ovr_bulk(su32(Bs + (size_t)j * bslot), a.Uh + (size_t)(j % nkc) * bslot, bbytes, b_af + 8 * j);
            for (int t = blockIdx.x; t < nct; t += gridDim.x)
                for (int kc = 0; kc < nkc; ++kc, ++c) {
                    if (c >= npre) {
                        if (c >= NA) ovr_wait(b_ae + 8 * sa, pe);
                        OVR_MARK(pw0)
                        const uint32_t bar = b_af + 8 * sa;
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(abytes + bbytes) : "memory");
                        ovr_bulk(su32(As + (size_t)sa * OVR_ATILE), a.XH + ((size_t)t * nkc + kc) * OVR_ATILE, abytes, bar);
                        ovr_bulk(su32(Bs + (size_t)sa * bslot), a.Uh + (size_t)kc * bslot, bbytes, bar);
                        OVR_MARK(pw1)
                    }
                    if (++sa == NA) { sa = 0; pe ^= 1u; }
                }
        }
    } else if (warp == OVR_W_B) {
        // (spare warp)
    } else if (warp == OVR_W_MMA) {
        // ---------------- MMA issuer ------------------------------------------------------------
        // (a lone thread issues the MMAs: its scalar instruction stream bounds the issue rate, so
        // descriptors are precomputed, slots advance by counters and one commit releases a stage)
        if (lane == 0) {
            const uint32_t idesc = (1u << 4) | ((uint32_t)(NU >> 3) << 17) | (8u << 24);   // f32 D, f16 A/B, K-major
            const uint32_t sbo = (uint32_t)(OVR_KCH / 8) * 128u;
            const uint64_t a_desc0 = umma_desc_kmajor(su32(As), sbo), b_desc0 = umma_desc_kmajor(su32(Bs), sbo);
            const uint64_t a_step = (uint64_t)(OVR_ATILE * 2 / 16), b_step = (uint64_t)(bslot * 2 / 16);
            const uint64_t a_lo = (uint64_t)(128 * OVR_KCH * 2 / 16), b_lo = (uint64_t)(NU * OVR_KCH * 2 / 16);
            int sa = 0, j = 0;
            uint32_t pa = 0;
            for (int t = blockIdx.x; t < nct; t += gridDim.x, ++j) {
                const int ab = j & 1;
                if (j >= 2) ovr_wait(b_acce + 8 * ab, (uint32_t)(((j >> 1) - 1) & 1));   // TMEM half drained
                OVR_MARK(pw1)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dcol = tmem + (uint32_t)(ab * NU);
                for (int kc = 0; kc < nkc; ++kc) {
                    ovr_wait(b_af + 8 * sa, pa);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint64_t ah = a_desc0 + (uint64_t)sa * a_step, bh = b_desc0 + (uint64_t)sa * b_step;
                    const uint32_t acc0 = kc > 0 ? 1u : 0u;
#pragma unroll
                    for (int ks = 0; ks < OVR_KCH / 16; ++ks) {   // h.h, h.l, l.h; +256 B per k-step
                        const uint64_t ks16 = (uint64_t)(ks * 16);
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(dcol), "l"(ah + ks16), "l"(bh + ks16), "r"(idesc), "r"(ks > 0 ? 1u : acc0));
                        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                                     ::"r"(dcol), "l"(ah + ks16), "l"(bh + b_lo + ks16), "r"(idesc));
                        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                                     ::"r"(dcol), "l"(ah + a_lo + ks16), "l"(bh + ks16), "r"(idesc));
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b_ae + 8 * sa) : "memory");
                    if (++sa == NA) { sa = 0; pa ^= 1u; }
                }
                OVR_MARK(pw0)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b_accf + 8 * ab) : "memory");
            }
        }
    } else {
        // ---------------- epilogue -------------------------------------------------------------
        // TMEM half drained first (all of this warp's problems), then per problem the kernel values,
        // G update and candidate keys of its 32 rows -> shared keys [p][side][128]; then one warp
        // per (problem, side) selects the tile's top-8 of 128 keys.
        constexpr int PPW = OVR_MAXP / 4;      // problems per warp at most
        const int e = warp - OVR_W_EPI;        // 0 .. OVR_EPI - 1
        const int q = warp & 3;                // TMEM lane quadrant of this warp
        const int pi = e >> 2;                 // problems p = pi, pi + 4, ...
        const int np = (a.P - pi + 3) >> 2;    // this warp's problem count (warp-uniform)
        const float isg = a.inv_sigma2;
        uint64_t* tkeys = wl;                  // [P][2][128]
        asm volatile("griddepcontrol.wait;" ::: "memory");   // the solve's outputs are complete
        for (int i = tid - OVR_W_EPI * 32; i < NU; i += OVR_EPI * 32) { sCoef[i] = a.ucoef[i]; sNorm[i] = a.unorm[i]; }
        epi_bar();
        int j = 0;
        for (int t = blockIdx.x; t < nct; t += gridDim.x, ++j) {
            const int ab = j & 1;
            const int64_t i = (int64_t)t * 128 + q * 32 + lane;
            const bool valid = i < a.n;
            float g0[PPW];
            uint32_t st0[PPW];
#pragma unroll
            for (int k = 0; k < PPW; ++k) {    // operands of the update, loaded before the wait
                const int p = pi + 4 * k;
                g0[k] = 0.0f;
                st0[k] = 0;
                if (k < np && valid) { g0[k] = a.G[p][i]; st0[k] = a.status[p][i]; }
            }
            const float xn = valid ? a.xnorm[i] : 0.0f;
            ovr_wait_sleep(b_accf + 8 * ab, (uint32_t)((j >> 1) & 1));
            OVR_MARK(pw0)
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t v[PPW][16];
#pragma unroll
            for (int k = 0; k < PPW; ++k) {
                if (k >= np) break;   // warp-uniform
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * NU + (pi + 4 * k) * 16);
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(v[k][0]), "=r"(v[k][1]), "=r"(v[k][2]), "=r"(v[k][3]), "=r"(v[k][4]), "=r"(v[k][5]), "=r"(v[k][6]), "=r"(v[k][7]),
                               "=r"(v[k][8]), "=r"(v[k][9]), "=r"(v[k][10]), "=r"(v[k][11]), "=r"(v[k][12]), "=r"(v[k][13]), "=r"(v[k][14]), "=r"(v[k][15])
                             : "r"(ta));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");   // TMEM half free
            __syncwarp();
            if (lane == 0) ovr_arrive(b_acce + 8 * ab);
#pragma unroll
            for (int k = 0; k < PPW; ++k) {
                if (k >= np) break;
                const int p = pi + 4 * k;
                uint64_t ku = 0ull, kl = 0ull;
                if (valid) {
                    float S = 0.0f;
#pragma unroll
                    for (int r = 0; r < 16; ++r)
                        S = fmaf(sCoef[p * 16 + r], kernel_from_dot(a.kpp[p], __uint_as_float(v[k][r]) * isg, xn, sNorm[p * 16 + r]), S);
                    const uint32_t st = st0[k];
                    const float yv = (st & ST_YPOS) ? 1.0f : -1.0f;
                    const float gn = fmaf(yv, S, g0[k]);
                    a.G[p][i] = gn;
                    const float sc = -yv * gn;
                    const uint64_t lo = (uint64_t)(0xffffffffu - (uint32_t)i);
                    if (st_in_up(st)) ku = ((uint64_t)ord_f32(sc) << 32) | lo;
                    if (st_in_low(st)) kl = ((uint64_t)ord_f32(-sc) << 32) | lo;
                }
                tkeys[(p * 2 + 0) * 128 + q * 32 + lane] = ku;
                tkeys[(p * 2 + 1) * 128 + q * 32 + lane] = kl;
            }
            epi_bar();
            // the tile's top-8 per problem and side: each lane sorts its 4 keys, 8 rounds of warp max
            for (int ps = e; ps < 2 * a.P; ps += OVR_EPI) {
                const uint64_t* K = tkeys + ps * 128;
                uint64_t kk[4] = {lds_u64(K + lane), lds_u64(K + 32 + lane), lds_u64(K + 64 + lane), lds_u64(K + 96 + lane)};
                sort_desc<4>(kk);
                uint64_t mine = 0ull;
#pragma unroll 1
                for (int r = 0; r < 8; ++r) {
                    const uint64_t best = warp_max_u64(kk[0]);
                    if (lane == r) mine = best;
                    if (best == 0ull) break;   // the rest of the list stays 0 (empty)
                    if (kk[0] == best) { kk[0] = kk[1]; kk[1] = kk[2]; kk[2] = kk[3]; kk[3] = 0ull; }
                }
                if (lane < 8) a.cand[((size_t)ps * nct + t) * 8 + lane] = mine;
            }
            epi_bar();
            OVR_MARK(pw1)
        }
    }
#undef OVR_MARK
    if (a.prof && blockIdx.x == 0 && lane == 0) {
        long long* o = a.prof + 3 * warp;
        atomicAdd(reinterpret_cast<unsigned long long*>(o), (unsigned long long)pw0);
        atomicAdd(reinterpret_cast<unsigned long long*>(o + 1), (unsigned long long)pw1);
        atomicAdd(reinterpret_cast<unsigned long long*>(o + 2), (unsigned long long)pw2);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == OVR_W_MMA) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

__global__ void __launch_bounds__(OVR_THREADS, 1) k_ovr_solve(const OvrArgs a)
{
    extern __shared__ __align__(1024) unsigned char ovr_smem[];
    float* sXW = reinterpret_cast<float*>(ovr_smem);   // dynamic shared memory: the fp64 X_W below
    __shared__ SmoShared sh;
    __shared__ uint64_t gm[16][8];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = blockIdx.x;
    const int d = (int)a.d;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");   // the previous pass's candidates and G
    if (a.done[p]) {
        if (tid < 16) a.ucoef[p * 16 + tid] = 0.0f;
        return;
    }
    long long t0 = clock64();
    long long* prof = (a.prof && p == 0 && tid == 0) ? a.prof + 96 : nullptr;
#define SOLVE_MARK(k) { if (prof) { const long long _n = clock64(); prof[k] += _n - t0; t0 = _n; } }
    // ---- a1: the tiles' sorted top-8 lists -> this problem's top-8 per side.  Warps 0-7 take the
    // up side, 8-15 the low side; a lane folds its lists into one sorted register list (top-8 of
    // a union of two sorted lists = sort(max(a_i, b_{7-i})), a bitonic merge), the warp selects
    // its top-8 over the lanes (8 rounds of 64-bit warp max), one warp per side merges the 8 warps.
    {
        const int side = warp >> 3, sw = warp & 7;
        const uint64_t* cl = a.cand + ((size_t)p * 2 + side) * a.nct * 8;
        uint64_t top[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) top[k] = 0ull;
        for (int l = sw * 32 + lane; l < a.nct; l += 256) {
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(cl + (size_t)l * 8);
            uint64_t b[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) { const ulonglong2 v = src[k]; b[2 * k] = v.x; b[2 * k + 1] = v.y; }
#pragma unroll
            for (int k = 0; k < 8; ++k) top[k] = top[k] > b[7 - k] ? top[k] : b[7 - k];
            // bitonic sequence -> descending (three half-cleaner stages)
#pragma unroll
            for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if ((k & h) == 0) {
                        const uint64_t x = top[k], y = top[k + h];
                        top[k] = x > y ? x : y;
                        top[k + h] = x > y ? y : x;
                    }
        }
        uint64_t mine = 0ull;
#pragma unroll 1
        for (int r = 0; r < 8; ++r) {
            const uint64_t best = warp_max_u64(top[0]);
            if (lane == r) mine = best;
            if (best == 0ull) break;
            if (top[0] == best) {
#pragma unroll
                for (int k = 0; k < 7; ++k) top[k] = top[k + 1];
                top[7] = 0ull;
            }
        }
        if (lane < 8) gm[warp][lane] = mine;
        __syncthreads();
        if (sw == 0) {
            uint64_t* out = side == 0 ? sh.win_up : sh.win_low;
            int32_t* srcs = side == 0 ? sh.win_up_src : sh.win_low_src;
            lane_list_merge(8, [&](int l, int j) { return lds_u64(&gm[side * 8 + l][j]); },
                            [&](int l, int j) { return l; }, out, srcs, lane);
        }
        __syncthreads();
    }
    SOLVE_MARK(0)
    // ---- W: sorted union of the 8 + 8 winners, deduplicated (one copy per row: C-SVC) ---------
    if (warp == 0) {
        uint64_t key = 0;
        if (lane < 8) key = sh.win_up[lane];
        else if (lane < 16) key = sh.win_low[lane - 8];
        const uint64_t g = key ? key_index(key) : ~0ull;
        bool valid = key != 0;
        uint64_t gj[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) gj[j] = __shfl_sync(FULL, g, j);
        if (lane >= 8 && lane < 16) {
#pragma unroll
            for (int j = 0; j < 8; ++j) valid = valid && gj[j] != g;
        }
        valid = valid && lane < 16;
        const uint32_t vm = __ballot_sync(FULL, valid);
        int rank = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) rank += (((vm >> j) & 1u) && gj[j] < g) ? 1 : 0;
        const int nw = __popc(vm);
        if (valid) {
            sh.w_gidx[rank] = (int64_t)g;
            sh.w_slot[rank] = rank;
            sh.r_row[rank] = (int64_t)g;
        }
        if (lane == 0) {
            sh.nw = nw;
            sh.nr = nw;
            const uint64_t ku0 = sh.win_up[0], kl0 = sh.win_low[0];
            sh.m_up = ku0 ? (double)unord_f32((uint32_t)(ku0 >> 32)) : -INFINITY;
            sh.M_low = kl0 ? -(double)unord_f32((uint32_t)(kl0 >> 32)) : INFINITY;
            sh.stop = (sh.m_up - sh.M_low <= a.tol) || (a.iters[p] >= a.max_iter) || nw == 0;
        }
    }
    __syncthreads();
    if (sh.stop) {
        if (tid == 0) {
            a.done[p] = 1;
            a.mup[p] = sh.m_up;
            a.mlow[p] = sh.M_low;
        }
        if (tid < 16) a.ucoef[p * 16 + tid] = 0.0f;
        return;
    }
    const int nw = sh.nw, nr = sh.nr;
    // payloads of W, X_W rows, norms
    if (tid < nw) {
        const int64_t g = sh.w_gidx[tid];
        sh.w_alpha[tid] = a.alpha[p][g];
        sh.w_G[tid] = (double)a.G[p][g];
        sh.w_y[tid] = (a.status[p][g] & ST_YPOS) ? 1 : -1;
    }
    // X_W in fp64 (fp32 inputs, exact), feature-major [dp4][24] (row stride 24 doubles: the
    // m8n8k4 fragment loads of four k-rows fall into two disjoint bank halves).  Thread t gathers
    // row r = t % 16 at features k = t / 16 + 32 j: the 32 lanes of a warp store 2 consecutive
    // 16-double rows (conflict-free); rows >= nr and features >= d are 0.
    double* sW64 = reinterpret_cast<double*>(sXW);
    const int dp4 = (d + 3) & ~3;
    {
        const int r = tid & 15, kb = tid >> 4;
        const float* src = r < nr ? a.XR + sh.r_row[r] * a.d : nullptr;
        for (int k0 = kb; k0 < dp4; k0 += 32 * 32) {   // all loads in flight (one round trip, d <= 1024)
            float x[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const int k = k0 + u * 32;
                x[u] = (src && k < d) ? __ldg(src + k) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const int k = k0 + u * 32;
                if (k < dp4) sW64[k * 24 + r] = (double)x[u];
            }
        }
        if (tid < nr) sh.xn[tid] = a.xnorm[sh.r_row[tid]];
    }
    if (tid >= nr && tid < SVM_WS) sh.xn[tid] = 0.0f;
    __syncthreads();
    SOLVE_MARK(1)
    // ---- K_WW in fp64: Gram X_W X_W^T on the fp64 tensor cores (mma.sync m8n8k4, three 8x8 tiles
    // x 5 k-parts = 15 warps, fixed summation order), then K from the Gram entries (RBF: the
    // distance G_aa + G_bb - 2 G_ab, clamped at 0; 0 exactly on the diagonal) --------------------
    {
        __shared__ double gpart[5][3][64];
        __shared__ double gram[SVM_WS * SVM_WS];
        if (warp < 15) {
            const int t = warp / 5, part = warp - t * 5;
            const int I = t == 2 ? 1 : 0, J = t == 0 ? 0 : 1;
            const int nsteps = dp4 >> 2;
            double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
            const int ra = I * 8 + (lane >> 2), rb = J * 8 + (lane >> 2), kk = lane & 3;
            int s = part;
            for (; s + 5 < nsteps; s += 10) {   // two accumulator pairs: independent DMMA chains
                const double a0 = sW64[(4 * s + kk) * 24 + ra], b0 = sW64[(4 * s + kk) * 24 + rb];
                const double a1 = sW64[(4 * (s + 5) + kk) * 24 + ra], b1 = sW64[(4 * (s + 5) + kk) * 24 + rb];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c0), "+d"(c1) : "d"(a0), "d"(b0));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(e0), "+d"(e1) : "d"(a1), "d"(b1));
            }
            if (s < nsteps) {
                const double a0 = sW64[(4 * s + kk) * 24 + ra], b0 = sW64[(4 * s + kk) * 24 + rb];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c0), "+d"(c1) : "d"(a0), "d"(b0));
            }
            gpart[part][t][(lane >> 2) * 8 + (lane & 3) * 2] = c0 + e0;
            gpart[part][t][(lane >> 2) * 8 + (lane & 3) * 2 + 1] = c1 + e1;
        }
        __syncthreads();
        SOLVE_MARK(5)
        if (tid < SVM_WS * SVM_WS) {
            int ra = tid >> 4, rb = tid & 15;
            const bool sw = (ra >> 3) > (rb >> 3);
            const int I = sw ? rb >> 3 : ra >> 3, J = sw ? ra >> 3 : rb >> 3;
            const int t = I == 0 ? (J == 0 ? 0 : 1) : 2;
            const int e = sw ? (rb & 7) * 8 + (ra & 7) : (ra & 7) * 8 + (rb & 7);
            double g = 0.0;
            for (int part = 0; part < 5; ++part) g += gpart[part][t][e];
            gram[tid] = g;
        }
        __syncthreads();
        if (tid < SVM_WS * SVM_WS) {
            const int ra = tid >> 4, rb = tid & 15;
            if (ra < nr && rb < nr) {
                double v = gram[tid];
                if (a.kpp[p].kernel == 2) {
                    v = ra == rb ? 0.0 : gram[ra * 17] + gram[rb * 17] - 2.0 * gram[tid];
                    v = v > 0.0 ? v : 0.0;
                }
                sh.kr[tid] = kernel_fp64_from(v, a.kpp[p]);
            }
        }
        __syncthreads();
        SOLVE_MARK(6)
        if (tid < SVM_WS * SVM_WS) {
            const int pa = tid >> 4, pb = tid & 15;
            double kab = 0.0, ie = 0.0;
            if (pa < nw && pb < nw) {
                kab = sh.kr[pa * SVM_WS + pb];
                const double eta = sh.kr[pa * SVM_WS + pa] + sh.kr[pb * SVM_WS + pb] - 2.0 * kab;
                ie = 1.0 / (eta < 1e-12 ? 1e-12 : eta);
            }
            sh.kpos[tid] = kab;
            sh.inv_eta[tid] = ie;
        }
        __syncthreads();
    }
    SOLVE_MARK(2)
    // ---- a2: the subproblem (one warp), then alpha / status of W and the coefficients --------
    if (warp == 0) {
        const int steps = solve_subproblem(sh, nw, a.Cp[p], a.inner_tol, a.inner_max, lane);
        if (lane == 0) SOLVE_MARK(3)
        __syncwarp();
        if (lane < SVM_WS) {
            float c = 0.0f;
            if (lane < nw) {
                const double da = sh.w_anew[lane] - sh.w_alpha[lane];
                c = (float)((double)sh.w_y[lane] * da);
                const int64_t g = sh.w_gidx[lane];
                a.alpha[p][g] = sh.w_anew[lane];
                a.status[p][g] = make_status(sh.w_y[lane], sh.w_anew[lane], a.Cp[p]);
            }
            a.ucoef[p * 16 + lane] = c;
            a.unorm[p * 16 + lane] = sh.xn[lane];
        }
        if (lane == 0) {
            a.iters[p] += 1;
            a.inner_total[p] += steps;
        }
    }
    // ---- this problem's 16 columns of the U operand, all K-chunks (fp16 hi | lo, k_ovr_pass) ----
    {
        const int NU = a.NU;
        const int total = a.nkc * OVR_KCH * 16;
        for (int e = tid; e < total; e += OVR_THREADS) {
            const int f = e >> 4, r = e & 15;
            const int kc = f / OVR_KCH, k = f - kc * OVR_KCH;
            const float x = f < d ? (float)sW64[f * 24 + r] : 0.0f;   // exact (fp32 promoted)
            uint16_t h, l;
            f16_split(x, a.sigma, h, l);
            uint16_t* base = a.Uh + (size_t)kc * 2 * NU * OVR_KCH;
            base[kmaj16_off(p * 16 + r, k)] = h;
            base[NU * OVR_KCH + kmaj16_off(p * 16 + r, k)] = l;
        }
    }
    SOLVE_MARK(4)
#undef SOLVE_MARK
}
}  // namespace

int smo_ring_bytes(int rpt) { return SMO_THREADS * 4 * rpt * (rpt == 1 ? pf_x<1>() : rpt == 2 ? pf_x<2>() : pf_x<4>()); }
int smo_csr_stage_bytes() { return SMO_WARPS * CSR_CAP * 6; }
int smo_sell_bytes(int spc, int64_t d) { return (int)(4 * (((spc + 4) & ~3) + ((d + 4) & ~3))); }
int smo_csr_w_extra_bytes(int64_t d) { return (int)(d * 4 * (WSTR_CSR - SVM_WS)); }

int smo_smem_bytes(int64_t d, int world, int nblk, int64_t x_rows)
{
    (void)world;   // the rank level (<= SVM_MAX_RANKS lists) lives in static shared memory
    const int64_t L = nblk;
    return (int)(((d * 16 + 3) & ~3) * 4 + L * 8 * 8 * 2 + 4 * d * x_rows);  // + 64 B per buffered row
}

// persisting-L2 limit of the caller, saved by launch_smo and restored by smo_l2_restore (one
// training at a time per thread; thread_local so concurrent trainings do not mix their values)
static thread_local size_t g_l2_saved = 0;
static thread_local bool g_l2_raised = false;
void smo_l2_restore()
{
    if (!g_l2_raised) return;
    g_l2_raised = false;
    // demote this library's persisting lines only when nobody else had a set-aside (a reset
    // would also demote the caller's); otherwise shrinking the set-aside back releases them
    if (g_l2_saved == 0) cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_saved);
    cudaGetLastError();
}

static const void* smo_pick(const SmoArgs& a)
{
    const bool rbf = a.kp.kernel == 2;
#define SMO_PICK(CSR_, RPT_, XS_) \
    (rbf ? (const void*)smo_persistent<CSR_, RPT_, XS_, true> : (const void*)smo_persistent<CSR_, RPT_, XS_, false>)
    if (a.XT == nullptr) return SMO_PICK(true, 1, false);
    if (a.x_in_smem)
        return a.rpt == 4 ? SMO_PICK(false, 4, true) : a.rpt == 2 ? SMO_PICK(false, 2, true) : SMO_PICK(false, 1, true);
    return a.rpt == 4 ? SMO_PICK(false, 4, false) : a.rpt == 2 ? SMO_PICK(false, 2, false) : SMO_PICK(false, 1, false);
#undef SMO_PICK
}

// Dynamic shared memory available to the persistent kernel variant `a` selects: the device's
// per-block opt-in maximum minus that variant's static shared memory (SmoShared) and 1 KB of slack.
int smo_dyn_smem_cap(const SmoArgs& a)
{
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, smo_pick(a)) != cudaSuccess) { cudaGetLastError(); return 200 * 1024; }
    return optin - (int)fa.sharedSizeBytes - 1024;
}

cudaError_t launch_smo(const SmoArgs& a, int smem_bytes, cudaStream_t st)
{
    void* args[] = {const_cast<SmoArgs*>(&a)};
    const void* fn = smo_pick(a);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.virt ? a.nblk * a.world : a.nblk);   // virtual ranks: all in this launch
    cfg.blockDim = dim3(SMO_THREADS);
    cfg.dynamicSmemBytes = (size_t)smem_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
    // X streamed from HBM every iteration (not resident in shared memory): an L2 access-policy
    // window marks this rank's X^T as persisting, so the part that fits the L2 set-aside stays
    // in L2 across iterations (c4: X = 108 MB against a 126 MB L2).  Arithmetic is unchanged.
    size_t persist_max = 0, window_max = 0;
    {
        int dev = 0, pm = 0, wm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&pm, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&wm, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        persist_max = (size_t)pm;
        window_max = (size_t)wm;
    }
    const size_t xbytes = a.XT ? (size_t)a.d * (size_t)a.n_pad * sizeof(float) : 0;
    const bool persist = a.XT && !a.x_in_smem && persist_max > 0 && window_max > 0 &&
                         !getenv("SVMB200_NO_L2PERSIST");
    // the L2 set-aside is raised for this launch only: smo_l2_restore (after the loop) puts the
    // caller's limit back
    if (persist) {
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        g_l2_saved = cur;
        g_l2_raised = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist_max) == cudaSuccess;
        cudaGetLastError();
    }
    if (persist && g_l2_raised) {
        const size_t win = std::min(xbytes, window_max);
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = const_cast<float*>(a.XT);
        attr[na].val.accessPolicyWindow.num_bytes = win;
        attr[na].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)persist_max / (double)win);
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    svm_note_launches(1);
    return cudaLaunchKernelExC(&cfg, fn, args);   // (run_loop demotes the persisting lines after the loop)
}

cudaError_t launch_kernel_rows(const SmoArgs& a, const int64_t* rows, int nr, float* K,
                               cudaStream_t st)
{
    int smem = (int)(a.d * 4 * (a.XT == nullptr ? WSTR_CSR : SVM_WS));
    int grid = (int)((a.n_local + 255) / 256);
    if (a.XT == nullptr) {
        cudaFuncSetAttribute(kernel_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        svm_note_launches(1);
        kernel_rows_kernel<true><<<grid, 256, smem, st>>>(a, rows, nr, K);
    } else {
        cudaFuncSetAttribute(kernel_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        svm_note_launches(1);
        kernel_rows_kernel<false><<<grid, 256, smem, st>>>(a, rows, nr, K);
    }
    return cudaGetLastError();
}

// launch with programmatic stream serialization (PDL): the kernel may start while the previous
// kernel on the stream finishes; it orders its dependent reads with griddepcontrol.wait
static cudaError_t ovr_launch(void (*kern)(OvrArgs), int grid, int block, int smem, cudaStream_t st, const OvrArgs& a)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = getenv("SVMB200_NO_PDL") ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// shared memory of k_ovr_pass for ring depths (na, nb)
static int ovr_pass_smem_n(int NU, int na, int nb)
{
    return (na * OVR_ATILE + nb * 2 * NU * OVR_KCH) * 2 + 2 * OVR_MAXP * 16 * 4 + (NU / 16) * 2 * 128 * 8 +
           (4 * OVR_MAXRING + 4) * 8 + 16;
}
// ring depths: as deep as the shared memory allows (static: 1 KB; 227 KB per CTA in total)
static void ovr_rings(int NU, int* na, int* nb)
{
    const int cap = 225 * 1024;
    *na = 2;
    while (*na < OVR_MAXRING && ovr_pass_smem_n(NU, *na + 1, *na + 1) <= cap) ++*na;
    *nb = *na;   // one stage = (X chunk, U chunk)
}
int ovr_pass_smem(const OvrArgs& a)
{
    int na, nb;
    ovr_rings(a.NU, &na, &nb);
    return ovr_pass_smem_n(a.NU, na, nb);
}

cudaError_t launch_ovr_pass(const OvrArgs& a0, cudaStream_t st)
{
    const int nsm = svm_device_sms();
    OvrArgs a = a0;
    ovr_rings(a.NU, &a.na, &a.nb);
    const int smem = ovr_pass_smem_n(a.NU, a.na, a.nb);
    // (a per-launch attribute call: kernel attributes are per device, and this costs ~1 us)
    cudaError_t e = cudaFuncSetAttribute(k_ovr_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    svm_note_launches(1);
    return ovr_launch(k_ovr_pass, std::min(nsm, a.nct), OVR_PASS_THREADS, smem, st, a);
}

// Setup of the batched pass: sigma = 2^e with max|X| sigma < 2^14 (fp16 range with margin), and the
// pre-split operand copy XH of X (one HBM pass).
cudaError_t ovr_prepare(OvrArgs& a, unsigned int* scratch, cudaStream_t st)
{
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return e;
    svm_note_launches(2);
    k_absmax<<<4 * 148, 256, 0, st>>>(a.XR, a.n * a.d, scratch);
    unsigned int mb = 0;
    e = cudaMemcpyAsync(&mb, scratch, sizeof mb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    float mx = 0;
    memcpy(&mx, &mb, sizeof mx);
    f16_sigma(mx, &a.sigma, &a.inv_sigma2);
    k_ovr_xh<<<8 * 148, 256, 0, st>>>(a.XR, a.n, a.d, a.nct, a.nkc, a.sigma, a.XH);
    return cudaGetLastError();
}

cudaError_t launch_absmax(const float* X, int64_t count, unsigned int* out, cudaStream_t st)
{
    svm_note_launches(1);
    k_absmax<<<4 * 148, 256, 0, st>>>(X, count, out);
    return cudaGetLastError();
}

static int ovr_solve_smem(const OvrArgs& a) { return (int)(((a.d + 3) & ~3) * 24 * 8); }   // fp64 X_W
cudaError_t launch_ovr_solve_prepare(const OvrArgs& a)
{
    return cudaFuncSetAttribute(k_ovr_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, ovr_solve_smem(a));
}
cudaError_t launch_ovr_solve(const OvrArgs& a, cudaStream_t st)
{
    const int smem = ovr_solve_smem(a);
    cudaError_t e = launch_ovr_solve_prepare(a);
    if (e != cudaSuccess) return e;
    svm_note_launches(1);
    return ovr_launch(k_ovr_solve, a.P, OVR_THREADS, smem, st, a);
}
