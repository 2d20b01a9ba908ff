// Microbenchmark: global_merge<5>-style tournament of L = 148 sorted 8-lists in shared memory
// (one warp), and the 64-bit warp max it is built on.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o scripts/ubench_merge scripts/ubench_merge.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
constexpr unsigned FULL = 0xffffffffu;
__device__ __forceinline__ uint64_t lds_u64(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k)
{
    uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    uint32_t mh = __reduce_max_sync(FULL, hi);
    uint32_t ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    return ((uint64_t)mh << 32) | ml;
}
template <int MAXK>
__device__ __forceinline__ void global_merge(const uint64_t* keys, int L, uint64_t* out, int32_t* src, int lane)
{
    uint64_t cur[MAXK], nxt[MAXK];
    int hd[MAXK];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
        int l = lane + 32 * k;
        cur[k] = l < L ? lds_u64(keys + l * 8) : 0;
        nxt[k] = l < L ? lds_u64(keys + l * 8 + 1) : 0;
        hd[k] = 0;
    }
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
        uint64_t lb = cur[0];
#pragma unroll
        for (int k = 1; k < MAXK; ++k) lb = cur[k] > lb ? cur[k] : lb;
        uint64_t best = warp_max_u64(lb);
        if (best == 0) { if (lane < 8 && lane >= r) { out[lane] = 0; src[lane] = -1; } break; }
        if (lb == best) {
#pragma unroll
            for (int k = 0; k < MAXK; ++k) {
                if (cur[k] == best) {
                    int l = lane + 32 * k;
                    out[r] = best; src[r] = l * 8 + hd[k]; ++hd[k];
                    cur[k] = nxt[k];
                    nxt[k] = hd[k] + 1 < 8 ? lds_u64(keys + l * 8 + hd[k] + 1) : 0;
                }
            }
        }
    }
}
__global__ void k(const uint64_t* gk, int L, long long* cyc, uint64_t* res)
{
    __shared__ uint64_t keys[160 * 8];
    __shared__ uint64_t out[8];
    __shared__ int32_t src[8];
    for (int i = threadIdx.x; i < L * 8; i += 32) keys[i] = gk[i];
    __syncwarp();
    long long tot = 0, totm = 0;
    for (int rep = 0; rep < 100; ++rep) {
        __syncwarp();
        long long t0 = clock64();
        global_merge<5>(keys, L, out, src, threadIdx.x);
        __syncwarp();
        uint64_t v = *(volatile uint64_t*)&out[7];
        asm volatile("" ::"l"(v));
        long long t1 = clock64();
        tot += t1 - t0;
        uint64_t x = keys[threadIdx.x * 3];
        long long t2 = clock64();
        for (int i = 0; i < 8; ++i) x = warp_max_u64(x ^ (uint64_t)i);
        asm volatile("" ::"l"(x));
        long long t3 = clock64();
        totm += t3 - t2;
        if (threadIdx.x == 0) res[0] = x;
    }
    if (threadIdx.x == 0) { cyc[0] = tot / 100; cyc[1] = totm / 100; for (int i = 0; i < 8; ++i) res[1 + i] = out[i]; }
}
int main()
{
    const int L = 148;
    uint64_t* h = new uint64_t[L * 8];
    srand(5);
    for (int l = 0; l < L; ++l) {
        uint64_t v = ((uint64_t)rand() << 32) | rand();
        for (int j = 0; j < 8; ++j) { h[l * 8 + j] = v; v -= (uint64_t)(rand() % 1000 + 1) << 20; }
    }
    uint64_t *d, *r; long long* c;
    cudaMalloc(&d, 8 * L * 8); cudaMalloc(&r, 8 * 9); cudaMalloc(&c, 16);
    cudaMemcpy(d, h, 8 * L * 8, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(d, L, c, r);
    long long hc[2];
    cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
    printf("global_merge<5> L=%d: %lld cycles; 8 dependent warp_max_u64: %lld cycles (%s)\n", L, hc[0], hc[1],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
