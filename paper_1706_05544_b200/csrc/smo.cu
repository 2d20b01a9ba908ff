// smo.cu -- the persistent working-set kernel: the hot loop of Rgtsvm's optimizer.
//
// One cooperative launch runs the whole loop of P:53 ("iteratively optimizing 16 heuristically
// selected dual space coefficients ... until convergence").  Every CTA owns a contiguous slice of
// training rows and, per iteration:
//   a1  merges the 8+8 candidates every CTA (of every rank) published into the working set W
//       ("picking 16 dual space coefficients based on which partial derivatives ... are the
//       largest, subject to dual space constraints") -- redundantly and identically
//       in every CTA, so no CTA waits on a single solver;
//   a2  solves the |W|-variable subproblem in fp64 on warp 0 ("optimized based on the local
//       gradient"; P:69 for eps-SVR) WHILE the other 15 warps already stream X and form
//       the kernel rows K(x_i, X_W) for their first rows;
//   a3  finishes the fused pass G_i += y_i sum_r c_r K(x_i, x_r) ("calculating the gradient for
//       all dual space coefficients"; "the responses terms are updated") and keeps a
//       running per-warp top-8 of the new scores, so the n x |W| kernel block is never stored;
//   and publishes its CTA top-8 up / top-8 low keys + payloads into every rank's receive buffer
//   with a release flag (the one-shot all-gather of SURVEY 8(e), fused into the pass).
// DESIGN.md has the layout, the roofline and what differs from the paper's GTSVM design.
#include "svm_internal.cuh"

#include <float.h>
#include <math.h>

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads)
{
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 64-bit warp max from two 32-bit REDUX reductions (all lanes participate).
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k)
{
    uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    uint32_t mh = __reduce_max_sync(FULL, hi);
    uint32_t ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    return ((uint64_t)mh << 32) | ml;
}

// Running top-8 of a warp: lane l < 8 holds the l-th largest key offered so far (0 = empty).
struct WarpTop8 {
    uint64_t v;
    __device__ __forceinline__ void reset() { v = 0; }
    __device__ __forceinline__ uint64_t thresh() const { return __shfl_sync(FULL, v, 7); }
    __device__ __forceinline__ void insert(uint64_t k, int lane)
    {
        uint64_t prev = __shfl_up_sync(FULL, v, 1);
        if (lane < 8 && k > v) v = (lane == 0 || prev > k) ? k : prev;
    }
    // Offer one key per lane (0 = none).  Keys are unique, so the result is exact.
    __device__ __forceinline__ void offer(uint64_t key, int lane)
    {
        uint64_t th = thresh();
        unsigned b = __ballot_sync(FULL, key > th);
        while (b) {
            int src = __ffs(b) - 1;
            uint64_t k = __shfl_sync(FULL, key, src);
            insert(k, lane);
            th = thresh();
            b &= ~(1u << src);
            b &= __ballot_sync(FULL, key > th);
        }
    }
};

template <int RPT>
__device__ __forceinline__ void zero_acc(float (&acc)[RPT][SVM_WS])
{
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
        for (int r = 0; r < SVM_WS; ++r) acc[j][r] = 0.0f;
}

// Dense kernel-row dot products: acc[j][r] = x_{li+j} . x_{W_r} for RPT consecutive rows.
// X is feature-major (one coalesced 4*RPT-byte load per lane per feature); X_W^T sits in shared
// memory as [d][16] and is read with 4 broadcast LDS.128 per feature, feeding 16*RPT FFMA.
template <int RPT>
__device__ __forceinline__ void dots_dense(const float* __restrict__ XT, int64_t n_pad, int d,
                                           int64_t li, bool active, const float* sXW,
                                           float (&acc)[RPT][SVM_WS])
{
    zero_acc<RPT>(acc);
    if (!active) return;
    const float* p = XT + li;
    const float4* w4 = reinterpret_cast<const float4*>(sXW);
#pragma unroll 4
    for (int k = 0; k < d; ++k) {
        float x[RPT];
        if constexpr (RPT == 4) {
            float4 v = __ldg(reinterpret_cast<const float4*>(p));
            x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
        } else {
            x[0] = __ldg(p);
        }
        p += n_pad;
        float4 wv[4] = {w4[4 * k], w4[4 * k + 1], w4[4 * k + 2], w4[4 * k + 3]};
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                acc[j][4 * q + 0] = fmaf(x[j], wv[q].x, acc[j][4 * q + 0]);
                acc[j][4 * q + 1] = fmaf(x[j], wv[q].y, acc[j][4 * q + 1]);
                acc[j][4 * q + 2] = fmaf(x[j], wv[q].z, acc[j][4 * q + 2]);
                acc[j][4 * q + 3] = fmaf(x[j], wv[q].w, acc[j][4 * q + 3]);
            }
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
        float4 wv[4] = {w4[4 * k], w4[4 * k + 1], w4[4 * k + 2], w4[4 * k + 3]};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            acc[0][4 * q + 0] = fmaf(v, wv[q].x, acc[0][4 * q + 0]);
            acc[0][4 * q + 1] = fmaf(v, wv[q].y, acc[0][4 * q + 1]);
            acc[0][4 * q + 2] = fmaf(v, wv[q].z, acc[0][4 * q + 2]);
            acc[0][4 * q + 3] = fmaf(v, wv[q].w, acc[0][4 * q + 3]);
        }
    }
}

// Shared state of one persistent CTA (static part; X_W and the staged keys are dynamic).
struct SmoShared {
    uint64_t warp_up[SMO_WARPS][8], warp_low[SMO_WARPS][8];
    uint64_t cta_up[8], cta_low[8];
    uint64_t win_up[8], win_low[8];      // merged global winners (keys)
    int32_t win_up_src[8], win_low_src[8];
    int64_t w_gidx[SVM_WS];              // working set, ascending dual index
    int32_t w_src[SVM_WS];               // payload slot of each position
    int32_t w_slot[SVM_WS];              // distinct-row slot of each position
    int64_t r_row[SVM_WS];               // distinct rows (global)
    double kr[SVM_WS * SVM_WS];          // K between distinct rows, fp64
    double qww[SVM_WS * SVM_WS];         // Q_WW = y_a y_b K
    double w_alpha[SVM_WS], w_G[SVM_WS], w_dalpha[SVM_WS], w_anew[SVM_WS];
    int32_t w_y[SVM_WS];
    float c[SVM_WS];                     // c_r = sum_{a: row r} y_a dalpha_a
    float xn[SVM_WS];                    // |x_r|^2 of the distinct rows
    int32_t nw, nr, stop, timeout, next_chunk, inner_steps;
    double m_up, M_low;
};

// Per-row epilogue shared by the scan (do_update = false) and the pass.
template <int RPT>
__device__ __forceinline__ void row_epilogue(const SmoArgs& a, const SmoShared& sh,
                                             int64_t li0, int64_t cta_end, bool do_update,
                                             const float (&acc)[RPT][SVM_WS], WarpTop8& up,
                                             WarpTop8& low, int lane)
{
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        int64_t li = li0 + j;
        bool valid = li < cta_end;
        float S = 0.0f;
        if (valid && do_update) {
            float xn = __ldg(a.xnorm + li);
#pragma unroll
            for (int r = 0; r < SVM_WS; ++r)
                S = fmaf(sh.c[r], kernel_from_dot(a.kp, acc[j][r], xn, sh.xn[r]), S);
        }
        for (int c = 0; c < a.ncopy; ++c) {
            uint64_t ku = 0, kl = 0;
            if (valid) {
                int64_t idx = (int64_t)c * a.n_pad + li;
                uint32_t st = a.status[idx];
                float yv = (st & ST_YPOS) ? 1.0f : -1.0f;
                float g = a.G[idx];
                if (do_update) {
                    g = fmaf(yv, S, g);
                    a.G[idx] = g;
                }
                float s = -yv * g;
                uint64_t gidx = (uint64_t)c * (uint64_t)a.n_global + (uint64_t)(a.row0 + li);
                if (st_in_up(st)) ku = make_key(s, gidx);
                if (st_in_low(st)) kl = make_key(-s, gidx);
            }
            up.offer(ku, lane);
            low.offer(kl, lane);
        }
    }
}

// Merge SMO_WARPS sorted warp lists into the CTA top-8 (one warp).
__device__ __forceinline__ void cta_merge(const uint64_t (*lists)[8], uint64_t* out, int lane)
{
    int idx = 0;
    uint64_t head = lane < SMO_WARPS ? lists[lane][0] : 0;
    for (int r = 0; r < 8; ++r) {
        uint64_t best = warp_max_u64(head);
        if (lane == 0) out[r] = best;
        if (best == 0) {
            for (int q = r + 1 + lane; q < 8; q += 32) out[q] = 0;
            break;
        }
        if (head == best && lane < SMO_WARPS) {
            ++idx;
            head = idx < 8 ? lists[lane][idx] : 0;
        }
    }
}

// Global merge of L sorted 8-lists (staged in shared memory as keys[L][8]) into the top-8 (one
// warp).  src receives list * 8 + position of each winner.
__device__ __forceinline__ void global_merge(const uint64_t* keys, uint8_t* head, int L,
                                             uint64_t* out, int32_t* src, int lane)
{
    for (int l = lane; l < L; l += 32) head[l] = 0;
    __syncwarp();
    uint64_t best_local = 0;
    int best_list = -1;
    for (int l = lane; l < L; l += 32) {
        uint64_t k = keys[l * 8];
        if (k > best_local) { best_local = k; best_list = l; }
    }
    for (int r = 0; r < 8; ++r) {
        uint64_t best = warp_max_u64(best_local);
        if (best == 0) {
            if (lane < 8 && lane >= r) { out[lane] = 0; src[lane] = -1; }
            break;
        }
        if (best_local == best) {  // unique owner
            int h = head[best_list];
            out[r] = best;
            src[r] = best_list * 8 + h;
            head[best_list] = (uint8_t)(h + 1);
            best_local = 0;
            best_list = -1;
            for (int l = lane; l < L; l += 32) {
                int hh = head[l];
                uint64_t k = hh < 8 ? keys[l * 8 + hh] : 0;
                if (k > best_local) { best_local = k; best_list = l; }
            }
        }
        __syncwarp();
    }
}

__device__ __forceinline__ int owner_rank(const SmoArgs& a, int64_t row)
{
    int r = 0;
    while (r + 1 < a.world && row >= a.rank_row0[r + 1]) ++r;
    return r;
}

template <bool CSR, int RPT>
__global__ void __launch_bounds__(SMO_THREADS, 1) smo_persistent(const SmoArgs a)
{
    extern __shared__ __align__(16) unsigned char dyn_smem[];
    __shared__ SmoShared sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = a.world * a.nblk;
    const int d = (int)a.d;
    float* sXW = reinterpret_cast<float*>(dyn_smem);                       // [d][16]
    uint64_t* sKU = reinterpret_cast<uint64_t*>(dyn_smem + (size_t)d * 64);  // [L][8]
    uint64_t* sKL = sKU + (size_t)L * 8;                                    // [L][8]
    uint8_t* sHeadU = reinterpret_cast<uint8_t*>(sKL + (size_t)L * 8);      // [L]
    uint8_t* sHeadL = sHeadU + L;

    const int64_t cta_begin = (int64_t)blockIdx.x * a.rows_per_cta;
    const int64_t cta_end = min(cta_begin + a.rows_per_cta, a.n_local);
    const int rows_per_chunk = 32 * RPT;
    const int nchunks = cta_end > cta_begin
                            ? (int)((cta_end - cta_begin + rows_per_chunk - 1) / rows_per_chunk)
                            : 0;
    const int slot = a.rank * a.nblk + blockIdx.x;
    const bool sys = a.world > 1;
    const bool reporter = blockIdx.x == 0;  // CTA 0 of every rank reports for its rank

    // ---- publish: CTA top-8 lists -> every rank's receive buffer, then the release flag ------
    auto publish = [&](uint32_t tag) {
        const int par = tag & 1;
        if (tid < 16) {
            uint64_t k = tid < 8 ? sh.cta_up[tid] : sh.cta_low[tid - 8];
            CandPay pay = {0.0, 0.0f, 0u};
            if (k) {
                uint64_t g = key_index(k);
                int c = g >= (uint64_t)a.n_global ? 1 : 0;
                int64_t li = (int64_t)(g - (uint64_t)c * a.n_global) - a.row0;
                int64_t idx = (int64_t)c * a.n_pad + li;
                pay.alpha = a.alpha[idx];
                pay.G = a.G[idx];
                pay.status = a.status[idx];
            }
            size_t off = ((size_t)par * L + slot) * 16 + tid;
            for (int r = 0; r < a.world; ++r) {
                a.peer_keys[r][off] = k;
                a.peer_pay[r][off] = pay;
            }
            if (sys) __threadfence_system(); else __threadfence();
        }
        __syncthreads();
        if (tid == 0) {
            for (int r = 0; r < a.world; ++r) {
                if (sys) st_release_sys(a.peer_flags[r] + slot, tag);
                else st_release_gpu(a.peer_flags[r] + slot, tag);
            }
        }
    };

    // ---- per-warp lists -> CTA lists ---------------------------------------------------------
    auto finish_lists = [&](WarpTop8& up, WarpTop8& low) {
        if (lane < 8) {
            sh.warp_up[warp][lane] = up.v;
            sh.warp_low[warp][lane] = low.v;
        }
        __syncthreads();
        if (warp == 0) cta_merge(sh.warp_up, sh.cta_up, lane);
        else if (warp == 1) cta_merge(sh.warp_low, sh.cta_low, lane);
        __syncthreads();
    };

    // ---- prologue: scan the current (alpha, G) and publish tag0 + 1 ---------------------------
    {
        WarpTop8 up, low;
        up.reset();
        low.reset();
        float acc[RPT][SVM_WS];
        zero_acc<RPT>(acc);
        for (int ch = warp; ch < nchunks; ch += SMO_WARPS) {
            int64_t li0 = cta_begin + (int64_t)ch * rows_per_chunk + lane * RPT;
            row_epilogue<RPT>(a, sh, li0, cta_end, false, acc, up, low, lane);
        }
        finish_lists(up, low);
        publish(a.tag0 + 1);
    }

    for (int64_t t = 0;; ++t) {
        const uint32_t tag = a.tag0 + 1 + (uint32_t)t;
        const int par = tag & 1;
        // ---- wait until every CTA of every rank published `tag` ------------------------------
        if (tid == 0) sh.timeout = 0;
        __syncthreads();
        for (int sl = tid; sl < L; sl += SMO_THREADS) {
            const uint32_t* f = a.peer_flags[a.rank] + sl;
            uint64_t t0 = 0;
            int spins = 0;
            while ((int32_t)(ld_acquire_sys(f) - tag) < 0) {
                if (++spins == 1024) {
                    spins = 0;
                    uint64_t now = globaltimer_ns();
                    if (t0 == 0) t0 = now;
                    else if (now - t0 > a.timeout_ns) { sh.timeout = 1; break; }
                }
            }
        }
        __syncthreads();
        if (sh.timeout) {
            if (reporter && tid == 0) a.info->error = 1;
            return;
        }
        // ---- stage the published keys (L2, bypassing L1) ------------------------------------
        {
            const ulonglong2* src =
                reinterpret_cast<const ulonglong2*>(a.peer_keys[a.rank] + (size_t)par * L * 16);
            for (int i = tid; i < L * 8; i += SMO_THREADS) {
                int l = i >> 3, w = i & 7;  // 8 x 16B per slot: 4 up, 4 low
                ulonglong2 v = __ldcg(src + i);
                uint64_t* dst = w < 4 ? sKU + l * 8 + 2 * w : sKL + l * 8 + 2 * (w - 4);
                dst[0] = v.x;
                dst[1] = v.y;
            }
        }
        __syncthreads();
        // ---- a1: global merge (warp 0: I_up top-8, warp 1: I_low top-8) ----------------------
        if (warp == 0) global_merge(sKU, sHeadU, L, sh.win_up, sh.win_up_src, lane);
        else if (warp == 1) global_merge(sKL, sHeadL, L, sh.win_low, sh.win_low_src, lane);
        __syncthreads();
        if (warp == 0) {
            // W = sorted union of |W|/2 up winners and |W|/2 low winners, deduplicated.
            const int half = a.q >> 1;
            uint64_t key = 0;
            int32_t src = -1;
            if (lane < 8 && lane < half) { key = sh.win_up[lane]; src = sh.win_up_src[lane]; }
            else if (lane >= 8 && lane < 16 && lane - 8 < half) {
                key = sh.win_low[lane - 8];
                src = sh.win_low_src[lane - 8];
                if (src >= 0) src = (src >> 3) * 16 + 8 + (src & 7);
            }
            if (lane < 8 && src >= 0) src = (src >> 3) * 16 + (src & 7);
            uint64_t g = key ? key_index(key) : ~0ull;
            bool valid = key != 0;
            // drop low entries already chosen by the up half
            for (int j = 0; j < 8; ++j) {
                uint64_t gj = __shfl_sync(FULL, g, j);
                if (lane >= 8 && valid && gj == g) valid = false;
            }
            int rank = 0;
            for (int j = 0; j < 16; ++j) {
                uint64_t gj = __shfl_sync(FULL, g, j);
                bool vj = __shfl_sync(FULL, valid, j);
                rank += (vj && gj < g) ? 1 : 0;
            }
            unsigned vb = __ballot_sync(FULL, valid && lane < 16);
            if (valid && lane < 16) {
                sh.w_gidx[rank] = (int64_t)g;
                sh.w_src[rank] = src;
            }
            if (lane == 0) {
                sh.nw = __popc(vb);
                uint64_t ku = sh.win_up[0], kl = sh.win_low[0];
                sh.m_up = ku ? (double)unord_f32((uint32_t)(ku >> 32)) : -INFINITY;
                sh.M_low = kl ? -(double)unord_f32((uint32_t)(kl >> 32)) : INFINITY;
                sh.stop = (sh.m_up - sh.M_low <= a.tol) || (t >= a.max_iter) || sh.nw == 0;
                sh.next_chunk = 0;
            }
        }
        __syncthreads();
        if (sh.stop) {
            if (reporter && tid == 0) {
                a.info->iterations = t;
                a.info->m_up = sh.m_up;
                a.info->M_low = sh.M_low;
                a.info->converged = (sh.m_up - sh.M_low <= a.tol) ? 1 : 0;
            }
            return;
        }
        // ---- a2 setup: payloads, distinct rows, X_W^T into shared memory ----------------------
        const int nw = sh.nw;
        if (warp == 0) {
            int64_t g = 0, row = -1;
            if (lane < nw) {
                g = sh.w_gidx[lane];
                const CandPay* pp = a.peer_pay[a.rank] + (size_t)par * L * 16 + sh.w_src[lane];
                double al = __ldcg(&pp->alpha);
                float gv = __ldcg(&pp->G);
                uint32_t st = __ldcg(&pp->status);
                sh.w_alpha[lane] = al;
                sh.w_G[lane] = (double)gv;
                sh.w_y[lane] = (st & ST_YPOS) ? 1 : -1;
                row = g >= a.n_global ? g - a.n_global : g;
            }
            // distinct rows in position order (eps-SVR may select both copies of one row)
            int slot_r = -1;
            int nr = 0;
            for (int j = 0; j < nw; ++j) {
                int64_t rj = __shfl_sync(FULL, row, j);
                bool first = true;
                for (int k = 0; k < j; ++k) first &= (__shfl_sync(FULL, row, k) != rj);
                if (first) {
                    if (lane == 0) sh.r_row[nr] = rj;
                    if (lane == j) slot_r = nr;
                    ++nr;
                } else if (lane == j) {
                    for (int k = 0; k < nr; ++k)
                        if (sh.r_row[k] == rj) slot_r = k;
                }
                __syncwarp();
            }
            if (lane < nw) sh.w_slot[lane] = slot_r;
            if (lane == 0) sh.nr = nr;
        }
        __syncthreads();
        const int nr = sh.nr;
        if constexpr (!CSR) {
            for (int i = tid; i < d * SVM_WS; i += SMO_THREADS) {
                int r = i / d, k = i - r * d;
                float v = 0.0f;
                if (r < nr) {
                    int64_t row = sh.r_row[r];
                    int o = owner_rank(a, row);
                    v = a.peer_XR[o][(row - a.rank_row0[o]) * a.d + k];
                }
                sXW[k * SVM_WS + r] = v;
            }
        } else {
            for (int i = tid; i < d * SVM_WS; i += SMO_THREADS) sXW[i] = 0.0f;
            __syncthreads();
            for (int r = warp; r < nr; r += SMO_WARPS) {
                int64_t row = sh.r_row[r];
                int o = owner_rank(a, row);
                int64_t lr = row - a.rank_row0[o];
                int64_t b = a.peer_indptr[o][lr], e = a.peer_indptr[o][lr + 1];
                for (int64_t p = b + lane; p < e; p += 32)
                    sXW[a.peer_indices[o][p] * SVM_WS + r] = a.peer_vals[o][p];
            }
        }
        if (tid < SVM_WS) {
            float xn = 0.0f;
            if (tid < nr) {
                int64_t row = sh.r_row[tid];
                int o = owner_rank(a, row);
                xn = a.peer_xnorm[o][row - a.rank_row0[o]];
            }
            sh.xn[tid] = xn;
        }
        __syncthreads();
        // ---- Q_WW in fp64 (warps 0-3) -> warp 0 solves; other warps start the pass ------------
        if (warp < 4) {
            const int npairs = nr * (nr + 1) / 2;
            for (int p = tid; p < npairs; p += 128) {
                int r = 0, rem = p;
                while (rem >= nr - r) { rem -= nr - r; ++r; }
                int s = r + rem;
                double acc0 = 0.0, acc1 = 0.0;
                int k = 0;
                if (a.kp.kernel == 2) {
                    for (; k + 1 < d; k += 2) {
                        double t0 = (double)sXW[k * SVM_WS + r] - (double)sXW[k * SVM_WS + s];
                        double t1 = (double)sXW[(k + 1) * SVM_WS + r] -
                                    (double)sXW[(k + 1) * SVM_WS + s];
                        acc0 = fma(t0, t0, acc0);
                        acc1 = fma(t1, t1, acc1);
                    }
                    if (k < d) {
                        double t0 = (double)sXW[k * SVM_WS + r] - (double)sXW[k * SVM_WS + s];
                        acc0 = fma(t0, t0, acc0);
                    }
                } else {
                    for (; k + 1 < d; k += 2) {
                        acc0 = fma((double)sXW[k * SVM_WS + r], (double)sXW[k * SVM_WS + s], acc0);
                        acc1 = fma((double)sXW[(k + 1) * SVM_WS + r],
                                   (double)sXW[(k + 1) * SVM_WS + s], acc1);
                    }
                    if (k < d)
                        acc0 = fma((double)sXW[k * SVM_WS + r], (double)sXW[k * SVM_WS + s], acc0);
                }
                double kv = kernel_fp64_from(acc0 + acc1, a.kp);
                sh.kr[r * SVM_WS + s] = kv;
                sh.kr[s * SVM_WS + r] = kv;
            }
            named_bar_sync(2, 128);
        }

        WarpTop8 up, low;
        up.reset();
        low.reset();
        if (warp == 0) {
            // ---- a2: the |W|-variable subproblem, max-violating pair steps in fp64 -----------
            const int pa = lane & 15;
            const bool valid = pa < nw;
            const double C = a.C;
            int ya = valid ? sh.w_y[pa] : 1;
            double al = valid ? sh.w_alpha[pa] : 0.0;
            double Ga = valid ? sh.w_G[pa] : 0.0;
            const double a_old = al;
            if (lane < nw) {
                for (int b = 0; b < nw; ++b)
                    sh.qww[lane * SVM_WS + b] =
                        (double)(ya * sh.w_y[b]) * sh.kr[sh.w_slot[lane] * SVM_WS + sh.w_slot[b]];
            }
            __syncwarp();
            int step = 0;
            for (; step < a.inner_max; ++step) {
                double s = -(double)ya * Ga;
                bool upok = valid && (ya > 0 ? al < C : al > 0.0);
                bool lowok = valid && (ya > 0 ? al > 0.0 : al < C);
                double v = lane < 16 ? (upok ? s : -INFINITY) : (lowok ? -s : -INFINITY);
                int p = pa;
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) {
                    double vo = __shfl_xor_sync(FULL, v, off);
                    int po = __shfl_xor_sync(FULL, p, off);
                    if (vo > v || (vo == v && po < p)) { v = vo; p = po; }
                }
                double si = __shfl_sync(FULL, v, 0);
                int i = __shfl_sync(FULL, p, 0);
                double msj = __shfl_sync(FULL, v, 16);
                int j = __shfl_sync(FULL, p, 16);
                double sj = -msj;
                if (si == -INFINITY || msj == -INFINITY || si - sj <= a.inner_tol) break;
                int yi = __shfl_sync(FULL, ya, i), yj = __shfl_sync(FULL, ya, j);
                double ai = __shfl_sync(FULL, al, i), aj = __shfl_sync(FULL, al, j);
                double eta = sh.qww[i * SVM_WS + i] + sh.qww[j * SVM_WS + j] -
                             2.0 * (double)yi * (double)yj * sh.qww[i * SVM_WS + j];
                if (eta < 1e-12) eta = 1e-12;
                double tt = (si - sj) / eta;
                double lim_i = yi > 0 ? C - ai : ai;
                double lim_j = yj > 0 ? aj : C - aj;
                bool clip_i = false, clip_j = false;
                if (tt >= lim_i) { tt = lim_i; clip_i = true; }
                if (tt >= lim_j) { tt = lim_j; clip_j = true; clip_i = clip_i && (lim_i == lim_j); }
                if (pa == i) {
                    al += (double)yi * tt;
                    if (clip_i) al = yi > 0 ? C : 0.0;
                }
                if (pa == j) {
                    al -= (double)yj * tt;
                    if (clip_j) al = yj > 0 ? 0.0 : C;
                }
                if (valid)
                    Ga += sh.qww[pa * SVM_WS + i] * ((double)yi * tt) -
                          sh.qww[pa * SVM_WS + j] * ((double)yj * tt);
            }
            if (lane < nw) {
                sh.w_dalpha[lane] = al - a_old;
                sh.w_anew[lane] = al;
            }
            __syncwarp();
            if (lane < SVM_WS) {
                double cr = 0.0;
                for (int b = 0; b < nw; ++b)
                    if (sh.w_slot[b] == lane) cr += (double)sh.w_y[b] * sh.w_dalpha[b];
                sh.c[lane] = lane < nr ? (float)cr : 0.0f;
            }
            // owner writes alpha and status of its W entries (before the pass reads status)
            if (lane < nw) {
                int64_t g = sh.w_gidx[lane];
                int c = g >= a.n_global ? 1 : 0;
                int64_t row = g - (int64_t)c * a.n_global;
                int64_t li = row - a.row0;
                if (li >= cta_begin && li < cta_end) {
                    int64_t idx = (int64_t)c * a.n_pad + li;
                    a.alpha[idx] = al;
                    a.status[idx] = make_status(ya, al, C);
                }
            }
            if (reporter) {
                if (lane < nw) {
                    a.info->last_w[lane] = sh.w_gidx[lane];
                    a.info->last_dalpha[lane] = sh.w_dalpha[lane];
                }
                if (lane == 0) {
                    a.info->last_nw = nw;
                    a.info->last_inner = step;
                    a.info->inner_total += step;
                }
            }
            __threadfence_block();
            named_bar_arrive(1, SMO_THREADS);
            // warp 0 now joins the pass
            for (;;) {
                int ch = 0;
                if (lane == 0) ch = atomicAdd(&sh.next_chunk, 1);
                ch = __shfl_sync(FULL, ch, 0);
                if (ch >= nchunks) break;
                int64_t li0 = cta_begin + (int64_t)ch * rows_per_chunk + lane * RPT;
                float acc[RPT][SVM_WS];
                if constexpr (CSR) dots_csr(a.indptr, a.indices, a.vals, li0, li0 < cta_end, sXW, acc);
                else dots_dense<RPT>(a.XT, a.n_pad, d, li0, li0 < cta_end, sXW, acc);
                row_epilogue<RPT>(a, sh, li0, cta_end, true, acc, up, low, lane);
            }
        } else {
            // ---- a3: the fused kernel-row + gradient pass (first chunk overlaps a2) -----------
            bool waited = false;
            for (;;) {
                int ch = 0;
                if (lane == 0) ch = atomicAdd(&sh.next_chunk, 1);
                ch = __shfl_sync(FULL, ch, 0);
                if (ch >= nchunks) break;
                int64_t li0 = cta_begin + (int64_t)ch * rows_per_chunk + lane * RPT;
                float acc[RPT][SVM_WS];
                if constexpr (CSR) dots_csr(a.indptr, a.indices, a.vals, li0, li0 < cta_end, sXW, acc);
                else dots_dense<RPT>(a.XT, a.n_pad, d, li0, li0 < cta_end, sXW, acc);
                if (!waited) {
                    named_bar_sync(1, SMO_THREADS);
                    waited = true;
                }
                row_epilogue<RPT>(a, sh, li0, cta_end, true, acc, up, low, lane);
            }
            if (!waited) named_bar_sync(1, SMO_THREADS);
        }
        finish_lists(up, low);
        publish(tag + 1);
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
    for (int i = threadIdx.x; i < d * SVM_WS; i += blockDim.x) sXW[i] = 0.0f;
    __syncthreads();
    if constexpr (!CSR) {
        for (int i = threadIdx.x; i < d * SVM_WS; i += blockDim.x) {
            int r = i / d, k = i - r * d;
            if (r < nr) sXW[k * SVM_WS + r] = a.peer_XR[0][rows[r] * a.d + k];
        }
    } else {
        for (int r = 0; r < nr; ++r) {
            int64_t b = a.peer_indptr[0][rows[r]], e = a.peer_indptr[0][rows[r] + 1];
            for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x)
                sXW[a.peer_indices[0][p] * SVM_WS + r] = a.peer_vals[0][p];
        }
    }
    if (threadIdx.x < SVM_WS) xn[threadIdx.x] = threadIdx.x < nr ? a.xnorm[rows[threadIdx.x]] : 0.0f;
    __syncthreads();
    int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= a.n_local) return;
    float acc[1][SVM_WS];
    if constexpr (CSR) dots_csr(a.indptr, a.indices, a.vals, li, true, sXW, acc);
    else dots_dense<1>(a.XT, a.n_pad, d, li, true, sXW, acc);
    float xi = a.xnorm[li];
    for (int r = 0; r < nr; ++r) K[li * nr + r] = kernel_from_dot(a.kp, acc[0][r], xi, xn[r]);
}

}  // namespace

int smo_smem_bytes(int64_t d, int world, int nblk)
{
    int L = world * nblk;
    return (int)(d * 64 + (int64_t)L * 8 * 8 * 2 + 2 * L + 16);
}

cudaError_t launch_smo(const SmoArgs& a, int smem_bytes, cudaStream_t st)
{
    void* args[] = {const_cast<SmoArgs*>(&a)};
    const void* fn;
    if (a.XT == nullptr) fn = (const void*)smo_persistent<true, 1>;
    else if (a.rpt == 4) fn = (const void*)smo_persistent<false, 4>;
    else fn = (const void*)smo_persistent<false, 1>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel(fn, dim3(a.nblk), dim3(SMO_THREADS), args,
                                       (size_t)smem_bytes, st);
}

cudaError_t launch_kernel_rows(const SmoArgs& a, const int64_t* rows, int nr, float* K,
                               cudaStream_t st)
{
    int smem = (int)(a.d * 64);
    int grid = (int)((a.n_local + 255) / 256);
    if (a.XT == nullptr) {
        cudaFuncSetAttribute(kernel_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kernel_rows_kernel<true><<<grid, 256, smem, st>>>(a, rows, nr, K);
    } else {
        cudaFuncSetAttribute(kernel_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kernel_rows_kernel<false><<<grid, 256, smem, st>>>(a, rows, nr, K);
    }
    return cudaGetLastError();
}
