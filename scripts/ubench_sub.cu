// Microbenchmark of the |W| = 16 subproblem step (one warp), variants side by side.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_sub scripts/ubench_sub.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

constexpr unsigned FULL = 0xffffffffu;
struct Sh {
    double kpos[256], inv_eta[256], w_alpha[16], w_G[16], w_anew[16];
    int w_y[16];
};

__device__ __forceinline__ uint64_t mono64(double x)
{
    uint64_t u = (uint64_t)__double_as_longlong(x + 0.0);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unmono64(uint64_t u)
{
    return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}
__device__ __forceinline__ double lds_f64(uint32_t addr)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

// V0: the current library version
__device__ int solve_v0(Sh& sh, int nw, double C, double inner_tol, int inner_max, int lane)
{
    const int pa = lane & 15;
    const bool valid = lane < nw;
    const int y = valid ? sh.w_y[lane] : 1;
    double al = valid ? sh.w_alpha[lane] : 0.0;
    double s = valid ? -(double)y * sh.w_G[lane] : 0.0;
    const uint32_t ypos = __ballot_sync(FULL, y > 0);
    const uint32_t a_ie = (uint32_t)__cvta_generic_to_shared(sh.inv_eta);
    const uint32_t a_krow = (uint32_t)__cvta_generic_to_shared(sh.kpos + pa * 16);
    int step = 0;
    for (; step < inner_max; ++step) {
        const bool upok = valid && (y > 0 ? al < C : al > 0.0);
        const bool lowok = valid && (y > 0 ? al > 0.0 : al < C);
        const uint64_t ku = upok ? mono64(s) : 0ull, kl = lowok ? mono64(-s) : 0ull;
        const uint32_t hu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32));
        const uint32_t hl = __reduce_max_sync(FULL, (uint32_t)(kl >> 32));
        const uint32_t lu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32) == hu ? (uint32_t)ku : 0u);
        const uint32_t ll = __reduce_max_sync(FULL, (uint32_t)(kl >> 32) == hl ? (uint32_t)kl : 0u);
        const uint64_t mu = ((uint64_t)hu << 32) | lu, ml = ((uint64_t)hl << 32) | ll;
        const int i = __ffs(__ballot_sync(FULL, ku == mu)) - 1;
        const int j = __ffs(__ballot_sync(FULL, kl == ml)) - 1;
        const double si = unmono64(mu), sj = -unmono64(ml);
        if (mu == 0 || ml == 0 || si - sj <= inner_tol) break;
        const double ie = lds_f64(a_ie + 8u * (uint32_t)(i * 16 + j));
        const double kai = lds_f64(a_krow + 8u * (uint32_t)i);
        const double kaj = lds_f64(a_krow + 8u * (uint32_t)j);
        const double ai = __shfl_sync(FULL, al, i), aj = __shfl_sync(FULL, al, j);
        const bool yi = (ypos >> i) & 1u, yj = (ypos >> j) & 1u;
        double t = (si - sj) * ie;
        const double lim_i = yi ? C - ai : ai;
        const double lim_j = yj ? aj : C - aj;
        const bool ci = t >= lim_i;
        t = ci ? lim_i : t;
        const bool cj = t >= lim_j;
        t = cj ? lim_j : t;
        const bool clip_i = ci && (!cj || lim_i == lim_j);
        const double ni = clip_i ? (yi ? C : 0.0) : (yi ? ai + t : ai - t);
        const double nj = cj ? (yj ? 0.0 : C) : (yj ? aj - t : aj + t);
        al = lane == i ? ni : (lane == j ? nj : al);
        s = fma(t, kaj - kai, s);
    }
    if (lane < 16) sh.w_anew[lane] = al;
    return step;
}

// V1: membership kept as per-lane limits; keys from one 64-bit value per side; the high word's
// REDUX alone decides when unique (ballot popc == 1), else the low word; limits maintained
// per lane so the clip needs no shuffles of alpha: lane i publishes lim_i, lane j lim_j.
__device__ int solve_v1(Sh& sh, int nw, double C, double inner_tol, int inner_max, int lane)
{
    const int pa = lane & 15;
    const bool valid = lane < nw;
    const int y = valid ? sh.w_y[lane] : 1;
    double al = valid ? sh.w_alpha[lane] : 0.0;
    double s = valid ? -(double)y * sh.w_G[lane] : 0.0;
    const uint32_t a_ie = (uint32_t)__cvta_generic_to_shared(sh.inv_eta);
    const uint32_t a_krow = (uint32_t)__cvta_generic_to_shared(sh.kpos + pa * 16);
    // room to move "up" (y a increases) and "down"
    double up_room = valid ? (y > 0 ? C - al : al) : 0.0;    // > 0 <=> in I_up
    double dn_room = valid ? (y > 0 ? al : C - al) : 0.0;    // > 0 <=> in I_low
    int step = 0;
    for (; step < inner_max; ++step) {
        const uint64_t ku = up_room > 0.0 ? mono64(s) : 0ull;
        const uint64_t kl = dn_room > 0.0 ? mono64(-s) : 0ull;
        const uint32_t hu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32));
        const uint32_t hl = __reduce_max_sync(FULL, (uint32_t)(kl >> 32));
        const uint32_t lu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32) == hu ? (uint32_t)ku : 0u);
        const uint32_t ll = __reduce_max_sync(FULL, (uint32_t)(kl >> 32) == hl ? (uint32_t)kl : 0u);
        const uint64_t mu = ((uint64_t)hu << 32) | lu, ml = ((uint64_t)hl << 32) | ll;
        const int i = __ffs(__ballot_sync(FULL, ku == mu)) - 1;
        const int j = __ffs(__ballot_sync(FULL, kl == ml)) - 1;
        const double si = unmono64(mu), sj = -unmono64(ml);
        if (mu == 0 || ml == 0 || si - sj <= inner_tol) break;
        const double ie = lds_f64(a_ie + 8u * (uint32_t)(i * 16 + j));
        const double kai = lds_f64(a_krow + 8u * (uint32_t)i);
        const double kaj = lds_f64(a_krow + 8u * (uint32_t)j);
        const double lim_i = __shfl_sync(FULL, up_room, i), lim_j = __shfl_sync(FULL, dn_room, j);
        double t = (si - sj) * ie;
        const bool ci = t >= lim_i;
        t = ci ? lim_i : t;
        const bool cj = t >= lim_j;
        t = cj ? lim_j : t;
        const bool clip_i = ci && (!cj || lim_i == lim_j);
        if (lane == i) {
            up_room = clip_i ? 0.0 : up_room - t;
            dn_room = clip_i ? C : dn_room + t;
        }
        if (lane == j) {
            dn_room = cj ? 0.0 : dn_room - t;
            up_room = cj ? C : up_room + t;
        }
        s = fma(t, kaj - kai, s);
    }
    if (valid) al = y > 0 ? C - up_room : up_room;
    if (lane < 16) sh.w_anew[lane] = al;
    return step;
}

__device__ int solve_v2(Sh& sh, int nw, double C, double inner_tol, int inner_max, int lane)
{
    const int pa = lane & 15;
    const bool valid = lane < nw;
    const int y = valid ? sh.w_y[lane] : 1;
    double al = valid ? sh.w_alpha[lane] : 0.0;
    double s = valid ? -(double)y * sh.w_G[lane] : 0.0;
    const uint32_t a_ie = (uint32_t)__cvta_generic_to_shared(sh.inv_eta);
    const uint32_t a_krow = (uint32_t)__cvta_generic_to_shared(sh.kpos + pa * 16);
    // room to move "up" (y a increases) and "down"
    double up_room = valid ? (y > 0 ? C - al : al) : 0.0;    // > 0 <=> in I_up
    double dn_room = valid ? (y > 0 ? al : C - al) : 0.0;    // > 0 <=> in I_low
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
        const double ie = lds_f64(a_ie + 8u * (uint32_t)(i * 16 + j));
        const double kai = lds_f64(a_krow + 8u * (uint32_t)i);
        const double kaj = lds_f64(a_krow + 8u * (uint32_t)j);
        const double lim_i = __shfl_sync(FULL, up_room, i), lim_j = __shfl_sync(FULL, dn_room, j);
        const double si = unmono64(mu), sj = -unmono64(ml);
        if (mu == 0 || ml == 0 || si - sj <= inner_tol) break;
        double t = (si - sj) * ie;
        const bool ci = t >= lim_i;
        t = ci ? lim_i : t;
        const bool cj = t >= lim_j;
        t = cj ? lim_j : t;
        const bool clip_i = ci && (!cj || lim_i == lim_j);
        if (lane == i) {
            up_room = clip_i ? 0.0 : up_room - t;
            dn_room = clip_i ? C : dn_room + t;
        }
        if (lane == j) {
            dn_room = cj ? 0.0 : dn_room - t;
            up_room = cj ? C : up_room + t;
        }
        s = fma(t, kaj - kai, s);
    }
    if (valid) al = y > 0 ? C - up_room : up_room;
    if (lane < 16) sh.w_anew[lane] = al;
    return step;
}

__device__ int solve_v3(Sh& sh, int nw, double C, double inner_tol, int inner_max, int lane)
{
    const int pa = lane & 15;
    const bool valid = lane < nw;
    const int y = valid ? sh.w_y[lane] : 1;
    double al = valid ? sh.w_alpha[lane] : 0.0;
    double s = valid ? -(double)y * sh.w_G[lane] : 0.0;
    const uint32_t a_ie = (uint32_t)__cvta_generic_to_shared(sh.inv_eta);
    const uint32_t a_krow = (uint32_t)__cvta_generic_to_shared(sh.kpos + pa * 16);
    // room to move "up" (y a increases) and "down"
    double up_room = valid ? (y > 0 ? C - al : al) : 0.0;    // > 0 <=> in I_up
    double dn_room = valid ? (y > 0 ? al : C - al) : 0.0;    // > 0 <=> in I_low
    int step = 0;
    for (; step < inner_max; ++step) {
        const uint64_t ku = up_room > 0.0 ? mono64(s) : 0ull;
        const uint64_t kl = dn_room > 0.0 ? mono64(-s) : 0ull;
        const uint32_t hu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32));
        const uint32_t hl = __reduce_max_sync(FULL, (uint32_t)(kl >> 32));
        const uint32_t bu = __ballot_sync(FULL, (uint32_t)(ku >> 32) == hu);
        const uint32_t bl = __ballot_sync(FULL, (uint32_t)(kl >> 32) == hl);
        uint32_t lu, ll;
        if ((bu & (bu - 1)) == 0 && (bl & (bl - 1)) == 0) {   // unique high words (warp-uniform)
            lu = __shfl_sync(FULL, (uint32_t)ku, __ffs(bu) - 1);
            ll = __shfl_sync(FULL, (uint32_t)kl, __ffs(bl) - 1);
        } else {
            lu = __reduce_max_sync(FULL, (uint32_t)(ku >> 32) == hu ? (uint32_t)ku : 0u);
            ll = __reduce_max_sync(FULL, (uint32_t)(kl >> 32) == hl ? (uint32_t)kl : 0u);
        }
        const uint64_t mu = ((uint64_t)hu << 32) | lu, ml = ((uint64_t)hl << 32) | ll;
        const int i = (__ffs(__ballot_sync(FULL, ku == mu)) - 1) & 15;
        const int j = (__ffs(__ballot_sync(FULL, kl == ml)) - 1) & 15;
        const double ie = lds_f64(a_ie + 8u * (uint32_t)(i * 16 + j));
        const double kai = lds_f64(a_krow + 8u * (uint32_t)i);
        const double kaj = lds_f64(a_krow + 8u * (uint32_t)j);
        const double lim_i = __shfl_sync(FULL, up_room, i), lim_j = __shfl_sync(FULL, dn_room, j);
        const double si = unmono64(mu), sj = -unmono64(ml);
        if (mu == 0 || ml == 0 || si - sj <= inner_tol) break;
        double t = (si - sj) * ie;
        const bool ci = t >= lim_i;
        t = ci ? lim_i : t;
        const bool cj = t >= lim_j;
        t = cj ? lim_j : t;
        const bool clip_i = ci && (!cj || lim_i == lim_j);
        if (lane == i) {
            up_room = clip_i ? 0.0 : up_room - t;
            dn_room = clip_i ? C : dn_room + t;
        }
        if (lane == j) {
            dn_room = cj ? 0.0 : dn_room - t;
            up_room = cj ? C : up_room + t;
        }
        s = fma(t, kaj - kai, s);
    }
    if (valid) al = y > 0 ? C - up_room : up_room;
    if (lane < 16) sh.w_anew[lane] = al;
    return step;
}

template <int V>
__global__ void bench(Sh* shs, int nprob, int* steps_out, long long* cyc_out, double C, double tol)
{
    __shared__ Sh sh;
    long long tot = 0;
    int stot = 0;
    for (int p = 0; p < nprob; ++p) {
        // load problem
        for (int i = threadIdx.x; i < (int)(sizeof(Sh) / 8); i += 32)
            reinterpret_cast<double*>(&sh)[i] = reinterpret_cast<const double*>(&shs[p])[i];
        __syncwarp();
        long long t0 = clock64();
        int st = V == 0 ? solve_v0(sh, 16, C, tol, 1024, threadIdx.x) : V == 1 ? solve_v1(sh, 16, C, tol, 1024, threadIdx.x) : V == 2 ? solve_v2(sh, 16, C, tol, 1024, threadIdx.x) : solve_v3(sh, 16, C, tol, 1024, threadIdx.x);
        __syncwarp();
        long long t1 = clock64();
        tot += t1 - t0;
        stot += st;
        if (threadIdx.x < 16) shs[p].w_anew[threadIdx.x] = sh.w_anew[threadIdx.x];
    }
    if (threadIdx.x == 0) { *steps_out = stot; *cyc_out = tot; }
}

int main()
{
    const int NP = 200;
    Sh* h = new Sh[NP];
    srand(7);
    for (int p = 0; p < NP; ++p) {
        double x[16][8];
        for (int a = 0; a < 16; ++a) for (int k = 0; k < 8; ++k) x[a][k] = (rand() / (double)RAND_MAX - 0.5) * 2;
        for (int a = 0; a < 16; ++a) for (int b = 0; b < 16; ++b) {
            double dd = 0; for (int k = 0; k < 8; ++k) dd += (x[a][k] - x[b][k]) * (x[a][k] - x[b][k]);
            h[p].kpos[a * 16 + b] = exp(-0.125 * dd);
        }
        for (int a = 0; a < 16; ++a) for (int b = 0; b < 16; ++b) {
            double e = h[p].kpos[a * 16 + a] + h[p].kpos[b * 16 + b] - 2 * h[p].kpos[a * 16 + b];
            h[p].inv_eta[a * 16 + b] = 1.0 / (e < 1e-12 ? 1e-12 : e);
        }
        for (int a = 0; a < 16; ++a) {
            h[p].w_y[a] = (a & 1) ? -1 : 1;
            h[p].w_alpha[a] = (rand() % 3) * 0.5;
            h[p].w_G[a] = (rand() / (double)RAND_MAX - 0.5) * 2;
        }
    }
    Sh* d;
    cudaMalloc(&d, sizeof(Sh) * NP);
    int* ds;
    long long* dc;
    cudaMalloc(&ds, 4);
    cudaMalloc(&dc, 8);
    double res[4][16];
    for (int v = 0; v < 4; ++v) {
        cudaMemcpy(d, h, sizeof(Sh) * NP, cudaMemcpyHostToDevice);
        auto run = [&]() {
            if (v == 0) bench<0><<<1, 32>>>(d, NP, ds, dc, 1.0, 1e-4);
            else if (v == 1) bench<1><<<1, 32>>>(d, NP, ds, dc, 1.0, 1e-4);
            else if (v == 2) bench<2><<<1, 32>>>(d, NP, ds, dc, 1.0, 1e-4);
            else bench<3><<<1, 32>>>(d, NP, ds, dc, 1.0, 1e-4);
        };
        run();
        cudaDeviceSynchronize();
        cudaMemcpy(d, h, sizeof(Sh) * NP, cudaMemcpyHostToDevice);
        run();
        int st; long long cy;
        cudaMemcpy(&st, ds, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost);
        Sh last;
        cudaMemcpy(&last, d + NP - 1, sizeof(Sh), cudaMemcpyDeviceToHost);
        for (int a = 0; a < 16; ++a) res[v][a] = last.w_anew[a];
        printf("v%d: %d steps over %d problems, %.1f cycles/step\n", v, st, NP, (double)cy / st);
    }
    for (int v = 1; v < 4; ++v) {
        double md = 0; for (int a = 0; a < 16; ++a) md = fmax(md, fabs(res[0][a] - res[v][a]));
        printf("max |alpha_v0 - alpha_v%d| = %g\n", v, md);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
