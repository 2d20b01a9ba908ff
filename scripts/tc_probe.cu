// Standalone check of the tcgen05 TF32 path used by predict: one 128 x 64 x K product,
// operands in shared memory in the canonical MN-major SWIZZLE_NONE layout (core matrix =
// 8 k-rows x 16 B of 4 consecutive M (or N) elements), accumulator in TMEM, read back with
// tcgen05.ld.32x32b.  Compared with a CPU product of the tf32-truncated inputs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/tc_probe scripts/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 48, KG = K / 8;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MN-major, no swizzle: core matrix (g, kg) = 8 k-rows x 4 consecutive MN elements (16 B per row)
// at byte offset (g * KG + kg) * 128; SBO = KG * 128 (next MN group), LBO = 128 (next k group).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void k_probe(const float* A, const float* B, float* D, uint32_t idesc, int mode)
{
    // A: [K][M] (MN-major in global: M contiguous), B: [K][N]
    __shared__ __align__(1024) float sA[M * K];
    __shared__ __align__(1024) float sB[N * K];
    __shared__ uint32_t tmem_holder;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (mode != 2) {
    for (int e = tid; e < K * (M / 4); e += blockDim.x) {
        const int k = e / (M / 4), g = e % (M / 4);
        const float4 v = *reinterpret_cast<const float4*>(A + k * M + 4 * g);
        *reinterpret_cast<float4*>(reinterpret_cast<char*>(sA) + (g * KG + k / 8) * 128 + (k % 8) * 16) = v;
    }
    for (int e = tid; e < K * (N / 4); e += blockDim.x) {
        const int k = e / (N / 4), g = e % (N / 4);
        const float4 v = *reinterpret_cast<const float4*>(B + k * N + 4 * g);
        *reinterpret_cast<float4*>(reinterpret_cast<char*>(sB) + (g * KG + k / 8) * 128 + (k % 8) * 16) = v;
    }
    } else {   // K-major: core (row group r/8, k chunk k/4) = 8 rows x 4 k at ((r/8) * K/4 + k/4) * 128
        for (int e = tid; e < K * M; e += blockDim.x) {
            const int k = e / M, r = e % M;
            *reinterpret_cast<float*>(reinterpret_cast<char*>(sA) + ((r / 8) * (K / 4) + k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4) = A[k * M + r];
        }
        for (int e = tid; e < K * N; e += blockDim.x) {
            const int k = e / N, r = e % N;
            *reinterpret_cast<float*>(reinterpret_cast<char*>(sB) + ((r / 8) * (K / 4) + k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4) = B[k * N + r];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_holder)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_holder;
    if (tid == 0) printf("tmem base 0x%08x\n", tmem);
    {   // pre-fill D with 7.0 to tell "MMA did not run" from "MMA wrote zeros"
        const uint32_t sv = __float_as_uint(7.0f);
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
        for (int c = 0; c < 64; c += 4)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta + c), "r"(sv), "r"(sv), "r"(sv), "r"(sv));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (tid == 0 && mode == 2) {
        for (int ks = 0; ks < K / 8; ++ks) {
            const uint64_t da = make_desc(su32(sA) + ks * 256, 128, (K / 4) * 128);
            const uint64_t db = make_desc(su32(sB) + ks * 256, 128, (K / 4) * 128);
            const uint32_t acc = ks > 0 ? 1u : 0u;
            const uint32_t id2 = idesc & ~((1u << 15) | (1u << 16));   // K-major A and B
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(id2), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
    }
    if (tid == 0 && mode == 0) {
        for (int kg = 0; kg < KG; ++kg) {
            const uint64_t da = make_desc(su32(sA) + kg * 128, 128, KG * 128);
            const uint64_t db = make_desc(su32(sB) + kg * 128, 128, KG * 128);
            const uint32_t acc = kg > 0 ? 1u : 0u;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
    }
    if (tid == 0 && mode == 1) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&mbar)) : "memory");
    // wait for the MMAs
    {
        uint32_t ok = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(su32(&mbar)), "r"(0) : "memory");
        } while (!ok);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // each warp reads its 32 lanes (rows) x 64 columns
    uint32_t v[64];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#define LD16(o) asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
    : "=r"(v[o+0]), "=r"(v[o+1]), "=r"(v[o+2]), "=r"(v[o+3]), "=r"(v[o+4]), "=r"(v[o+5]), "=r"(v[o+6]), "=r"(v[o+7]), \
      "=r"(v[o+8]), "=r"(v[o+9]), "=r"(v[o+10]), "=r"(v[o+11]), "=r"(v[o+12]), "=r"(v[o+13]), "=r"(v[o+14]), "=r"(v[o+15]) \
    : "r"(taddr + o))
    LD16(0); LD16(16); LD16(32); LD16(48);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int c = 0; c < N; ++c) D[row * N + c] = __uint_as_float(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }

int main()
{
    float *hA = new float[K * M], *hB = new float[K * N], *hD = new float[M * N];
    srand(3);
    for (int i = 0; i < K * M; ++i) hA[i] = (rand() / (float)RAND_MAX - 0.5f) * 2;
    for (int i = 0; i < K * N; ++i) hB[i] = (rand() / (float)RAND_MAX - 0.5f) * 2;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 4 * K * M); cudaMalloc(&dB, 4 * K * N); cudaMalloc(&dD, 4 * M * N);
    cudaMemcpy(dA, hA, 4 * K * M, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 4 * K * N, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 4 * M * N);
    // c_format F32 (bit 4), a/b format TF32 (2 at bits 7, 10), a/b MN-major (bits 15, 16),
    // n_dim = N >> 3 at bit 17, m_dim = M >> 4 at bit 24
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const int mode = getenv("MODE") ? atoi(getenv("MODE")) : 0;
    k_probe<<<1, 128>>>(dA, dB, dD, idesc, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(hD, dD, 4 * M * N, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)tf32_trunc(hA[k * M + m]) * tf32_trunc(hB[k * N + n]);
            const double err = fabs(ref - hD[m * N + n]);
            if (err > 1e-3 && bad++ < 5) printf("  m %d n %d gpu %g ref %g\n", m, n, hD[m * N + n], ref);
            maxerr = fmax(maxerr, err); maxref = fmax(maxref, fabs(ref));
        }
    printf("max |err| %.3g (max |ref| %.3g), bad %d\n", maxerr, maxref, bad);
    return 0;
}
