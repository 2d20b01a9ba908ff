// REDUX / SHFL / VOTE throughput with W concurrent warps on one SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(long long* out, unsigned* sink, int iters)
{
    unsigned v = threadIdx.x * 7 + 1, acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned a, b, c, d;
        if (OP == 0) { a = __reduce_max_sync(~0u, v); b = __reduce_max_sync(~0u, v + 1); c = __reduce_max_sync(~0u, v + 2); d = __reduce_max_sync(~0u, v + 3); }
        else if (OP == 1) { a = __shfl_xor_sync(~0u, v, 1); b = __shfl_xor_sync(~0u, v + 1, 2); c = __shfl_xor_sync(~0u, v + 2, 4); d = __shfl_xor_sync(~0u, v + 3, 8); }
        else { a = __ballot_sync(~0u, v & 1); b = __ballot_sync(~0u, v & 2); c = __ballot_sync(~0u, v & 4); d = __ballot_sync(~0u, v & 8); }
        acc += a ^ b ^ c ^ d;
        v += acc & 1;
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = acc;
}
int main()
{
    long long* o; unsigned* s; cudaMalloc(&o, 8); cudaMalloc(&s, 4096);
    const char* nm[3] = {"redux", "shfl", "ballot"};
    for (int op = 0; op < 3; ++op)
        for (int w : {1, 4, 16}) {
            int it = 4096;
            for (int rep = 0; rep < 2; ++rep) {
                if (op == 0) k<0><<<1, 32 * w>>>(o, s, it);
                if (op == 1) k<1><<<1, 32 * w>>>(o, s, it);
                if (op == 2) k<2><<<1, 32 * w>>>(o, s, it);
            }
            cudaDeviceSynchronize();
            long long c; cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
            printf("%-6s warps=%2d: %.1f cycles per op per warp (4 independent per iteration) -> SM throughput %.2f ops/cycle\n",
                   nm[op], w, c / (4.0 * it), 4.0 * it * w / c);
        }
    return 0;
}
