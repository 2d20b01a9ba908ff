// FP32 FMA issue rate on sm_100a: 3-register FFMA vs packed FFMA2 vs the kernel's pattern
// (x broadcast against 16 W columns), independent accumulators, 16 warps per SM (one CTA of 512
// threads per SM, like the persistent kernel).  Prints FMA lanes per cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fma_rate scripts/fma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, float a, float b, long long* cyc)
{
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = threadIdx.x * 1e-7f + i;
    float w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = b + i * 1e-3f;
    float x[4] = {a, a + 1.f, a + 2.f, a + 3.f};
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {   // scalar FFMA: acc[j][r] += x[j] * w[r]
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int r = 0; r < 16; ++r) acc[j * 16 + r] = fmaf(x[j], w[r], acc[j * 16 + r]);
        } else {           // packed FFMA2 over column pairs
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int r = 0; r < 16; r += 2) {
                    float2 c = __ffma2_rn(make_float2(x[j], x[j]), make_float2(w[r], w[r + 1]),
                                          make_float2(acc[j * 16 + r], acc[j * 16 + r + 1]));
                    acc[j * 16 + r] = c.x;
                    acc[j * 16 + r + 1] = c.y;
                }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] += 1e-9f;
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * nsm * 512);
    cudaMalloc(&cyc, sizeof(long long) * nsm);
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<nsm, 512>>>(out, iters, 1.0f, 2.0f, cyc);
            else k<1><<<nsm, 512>>>(out, iters, 1.0f, 2.0f, cyc);
            cudaDeviceSynchronize();
        }
        long long c = 0;
        cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        const double fma = 64.0 * iters * 512;   // FMA lanes per CTA
        printf("%s: %.1f FMA lanes / cycle / SM (%lld cycles)\n", mode == 0 ? "FFMA  " : "FFMA2 ", fma / (double)c, c);
    }
    return 0;
}
