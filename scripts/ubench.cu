// Latency microbenchmarks of the primitives on the working-set loop's critical path (B200).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acq_gpu(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#define N 256
__global__ void bench(long long* out, uint32_t* flag, double* dsink, unsigned* usink, int seed)
{
    int lane = threadIdx.x & 31;
    long long t0, t1;
    // 1 redux chain (full warp, converged)
    unsigned v = lane + seed;
    __syncwarp();
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __reduce_max_sync(0xffffffffu, v + lane) ;
    t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / N;
    usink[threadIdx.x] = v;
    // 2 shfl chain
    v = lane + seed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
    t1 = clock64();
    if (threadIdx.x == 0) out[1] = (t1 - t0) / N;
    usink[threadIdx.x] += v;
    // 3 dfma chain
    double x = seed * 0.5 + lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) x = fma(x, 0.999, 0.25);
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = (t1 - t0) / N;
    dsink[threadIdx.x] = x;
    // 4 dsetp + select chain
    double y = seed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) y = (y > 0.5 * i) ? y - 1.0 : y + 2.0;
    t1 = clock64();
    if (threadIdx.x == 0) out[3] = (t1 - t0) / N;
    dsink[threadIdx.x] += y;
    // 5 ld.acquire.sys on a set flag (dependent chain through the address)
    uint32_t idx = 0;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) idx = ld_acq_sys(flag + (idx & 1));
    t1 = clock64();
    if (threadIdx.x == 0) out[4] = (t1 - t0) / 64;
    // 6 ld.acquire.gpu
    t0 = clock64();
    for (int i = 0; i < 64; ++i) idx = ld_acq_gpu(flag + (idx & 1));
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = (t1 - t0) / 64;
    // 7 ld.relaxed.gpu
    t0 = clock64();
    for (int i = 0; i < 64; ++i) idx = ld_relaxed_gpu(flag + (idx & 1));
    t1 = clock64();
    if (threadIdx.x == 0) out[6] = (t1 - t0) / 64;
    usink[threadIdx.x] += idx;
    // 8 __syncthreads chain
    t0 = clock64();
    for (int i = 0; i < 64; ++i) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) out[7] = (t1 - t0) / 64;
    // 9 __threadfence chain
    t0 = clock64();
    for (int i = 0; i < 64; ++i) { __threadfence(); flag[2 + (threadIdx.x & 1)] = i; }
    t1 = clock64();
    if (threadIdx.x == 0) out[8] = (t1 - t0) / 64;
    // 10 fp64 division chain
    double z = 3.0 + seed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) z = 1.0 / (z + 1.0);
    t1 = clock64();
    if (threadIdx.x == 0) out[9] = (t1 - t0) / N;
    dsink[threadIdx.x] += z;
    // 11 u64 compare-select chain
    unsigned long long u = seed + lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) u = (u > (unsigned long long)i * 7919ull) ? u - 3 : u + 5;
    t1 = clock64();
    if (threadIdx.x == 0) out[10] = (t1 - t0) / N;
    usink[threadIdx.x] += (unsigned)u;
    // 12 smem LDS.64 dependent chain
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    int j = lane & 7;
    t0 = clock64();
    for (int i = 0; i < N; ++i) j = ((int)sm[j] + 1) & 63;
    t1 = clock64();
    if (threadIdx.x == 0) out[11] = (t1 - t0) / N;
    usink[threadIdx.x] += j;
    // 13 __threadfence_system chain
    t0 = clock64();
    for (int i = 0; i < 16; ++i) { __threadfence_system(); flag[2 + (threadIdx.x & 1)] = i; }
    t1 = clock64();
    if (threadIdx.x == 0) out[12] = (t1 - t0) / 16;
    // 14 exp fp64 chain
    double e = 0.1 * seed;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) e = exp(-e);
    t1 = clock64();
    if (threadIdx.x == 0) out[13] = (t1 - t0) / 64;
    dsink[threadIdx.x] += e;
}

// cross-CTA flag ping-pong: CTA 0 and CTA k alternately bump a flag -> round-trip latency
__global__ void pingpong(volatile uint32_t* f, long long* out, int iters, int peer)
{
    if (threadIdx.x != 0) return;
    if (blockIdx.x != 0 && blockIdx.x != peer) return;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (blockIdx.x == 0) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(2 * i + 1) : "memory");
            while (ld_acq_gpu((const uint32_t*)f + 1) != (uint32_t)(2 * i + 1)) {}
        } else {
            while (ld_acq_gpu((const uint32_t*)f) != (uint32_t)(2 * i + 1)) {}
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f + 1), "r"(2 * i + 1) : "memory");
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main()
{
    long long* out;
    uint32_t* flag;
    double* ds;
    unsigned* us;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&flag, 64);
    cudaMalloc(&ds, 1024 * 8);
    cudaMalloc(&us, 1024 * 4);
    cudaMemset(flag, 0, 64);
    cudaMemset(out, 0, 64 * 8);
    for (int threads : {32, 512}) {
        bench<<<1, threads>>>(out, flag, ds, us, 1);
        cudaDeviceSynchronize();
        bench<<<1, threads>>>(out, flag, ds, us, 1);
        long long h[16];
        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        const char* names[] = {"redux.max", "shfl.xor", "dfma", "dsetp+sel", "ld.acquire.sys",
                               "ld.acquire.gpu", "ld.relaxed.gpu", "__syncthreads", "__threadfence+st",
                               "fp64 1/x", "u64 cmp+sel", "lds.64 chase", "__threadfence_system+st",
                               "exp fp64"};
        printf("threads=%d\n", threads);
        for (int i = 0; i < 14; ++i) printf("  %-24s %lld cycles\n", names[i], h[i]);
    }
    for (int peer : {1, 74, 147}) {
        cudaMemset(flag, 0, 64);
        pingpong<<<148, 32>>>(flag, out, 1000, peer);
        cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("flag round trip CTA0<->CTA%d: %lld cycles\n", peer, h);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
