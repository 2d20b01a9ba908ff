// tcgen05.mma issue-rate microbenchmark (B200): one CTA per SM, one thread issues back-to-back
// M=128 MMAs from shared-memory operands (K-major SWIZZLE_NONE) into TMEM; reports cycles per MMA
// and the implied dense rate for kind::tf32 (K=8) and kind::f16 (bf16 inputs, K=16) at several N.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tc_rate scripts/tc_rate.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo)
{
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int CE, int NS>
__global__ void k_rate(int kind, int N, int iters, long long* out)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t holder;
    __shared__ __align__(8) uint64_t bar, bar2;
    const int tid = threadIdx.x;
    for (int i = tid; i < 8 * (128 + 256) * 64 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.0f;
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&holder)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = holder;
    if (tid == 0) {
        const uint32_t fmt = kind == 0 ? ((2u << 7) | (2u << 10)) : ((1u << 7) | (1u << 10));
        const uint32_t idesc = (1u << 4) | fmt | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const uint32_t a0 = su32(sm), b0 = a0 + 8 * 128 * 64;   // slots of A: 128 rows x 64 B of K (2 k-steps)
        const uint32_t sbo = 4 * 128;                     // KC = 4 core matrices per 8-row group
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int sl = NS == 1 ? 0 : (i / 6) % NS;
            const uint32_t a = a0 + sl * 128 * 64, b = b0 + sl * 256 * 64;
            const uint64_t da = desc(a + (i & 1) * 256, sbo), db = desc(b + (i & 1) * 256, sbo);
            if (kind == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(i));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(i));
            if (CE && (i % CE) == CE - 1)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)) : "memory");
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(su32(&bar)) : "memory");
        long long t2 = clock64();
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main()
{
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    long long* d;
    cudaMalloc(&d, nsm * 2 * sizeof(long long));
    long long h[2 * 256];
    const int smem = 8 * (128 + 256) * 64;

    const int iters = 4096;
    auto run = [&](auto kern, int kind, int N, int ce, int ns) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            kern<<<nsm, 128, smem>>>(kind, N, iters, d);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); exit(1); }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h, d, nsm * 2 * sizeof(long long), cudaMemcpyDeviceToHost);
            if (rep == 0) continue;
            const int K = kind == 0 ? 8 : 16;
            const double flop = 2.0 * 128 * N * K * iters * nsm;
            printf("%s N=%3d commit/%d slots %d: issue %.1f cyc/MMA, complete %.1f cyc/MMA (SM 0); %.0f TFLOP/s dense\n",
                   kind == 0 ? "tf32" : "bf16", N, ce, ns, (double)h[0] / iters, (double)h[1] / iters, flop / ms / 1e9);
        }
    };
    run(k_rate<0, 1>, 1, 160, 0, 1);
    run(k_rate<0, 8>, 1, 160, 0, 8);
    run(k_rate<6, 1>, 1, 160, 6, 1);
    run(k_rate<12, 1>, 1, 160, 12, 1);
    run(k_rate<24, 1>, 1, 160, 24, 1);
    run(k_rate<6, 8>, 1, 160, 6, 8);
    run(k_rate<0, 1>, 1, 128, 0, 1);
    run(k_rate<0, 1>, 1, 256, 0, 1);
    run(k_rate<6, 1>, 1, 256, 6, 1);
    return 0;
}
