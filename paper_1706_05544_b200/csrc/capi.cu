// capi.cu -- the host engine behind include/svmb200.h (the C ABI): validation, problem building
// (a0), the working-set loop driver around the persistent kernel (a1-a3), certification and bias
// (a4), model assembly (a5) and batched predict (a6).  Every arithmetic step of the path runs in
// the CUDA kernels of smo.cu / layout.cu / predict.cu; this file allocates, copies and launches.
//
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.  Readings and layouts: DESIGN.md.
#include "../../include/svmb200.h"
#include "layout.cuh"

#include <dlfcn.h>

#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

// ================================================================ launch counter
#include <atomic>
#include <mutex>
static std::atomic<long long> g_launches{0};
void svm_note_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
extern "C" int64_t svm_launch_count(void) { return (int64_t)g_launches.load(); }

// ================================================================ errors
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? SVM_ENOMEM : SVM_ECUDA,         \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,  \
                        __LINE__);                                                        \
        }                                                                                 \
    } while (0)

#define TRY(expr)                   \
    do {                            \
        int rc_ = (expr);           \
        if (rc_ != SVM_OK) return rc_; \
    } while (0)

// ================================================================ device memory (RAII)
// Device buffers come from the stream-ordered pool (cudaMallocAsync on the legacy stream): no
// device-wide synchronisation on free, and repeated trainings reuse pooled memory.  Every entry
// point synchronises its stream before returning, so pool reuse never races user work.
// The library's device buffers come from a PRIVATE stream-ordered pool per device (the default
// pool and the caller's allocators are left alone).  Its release threshold keeps up to
// min(16 GiB, 1/8 of the device) of freed memory cached for the next training (the kernel-column
// cache alone takes up to 12 GiB): with threshold 0
// every synchronize returned it to the OS and the next training re-mapped it, which made single
// trainings 10-30% slower at random (c2: +40 ms, c4: +1.2 s measured); beyond the bound, freed
// memory goes back to the device at the next synchronize, so a host framework sharing the GPU
// never loses more than the bound to this library.
cudaMemPool_t svm_mem_pool()
{
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) { cudaGetLastError(); return nullptr; }
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps pp = {};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &pp) != cudaSuccess) { cudaGetLastError(); return nullptr; }
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        uint64_t thr = std::min<uint64_t>(16ull << 30, (uint64_t)tot / 8);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        cudaGetLastError();
        pools[dev] = pool;
    }
    return pools[dev];
}

struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    bool plain = false;  // cudaMalloc'd (exportable with cudaIpcGetMemHandle; pool memory is not)
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release()
    {
        if (p) {
            if (plain) cudaFree(p);
            else cudaFreeAsync(p, 0);
        }
        p = nullptr;
        bytes = 0;
        plain = false;
    }
    // Re-allocate an existing buffer as plain cudaMalloc memory (for peer export), keeping data.
    int make_plain()
    {
        if (!p || plain) return SVM_OK;
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(SVM_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
        }
        cudaMemcpy(q, p, bytes, cudaMemcpyDeviceToDevice);
        cudaFreeAsync(p, 0);
        cudaDeviceSynchronize();
        p = q;
        plain = true;
        return SVM_OK;
    }
    int alloc(size_t b)
    {
        release();
        if (b == 0) b = 16;
        cudaMemPool_t pool = svm_mem_pool();
        cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, b, pool, 0) : cudaMallocAsync(&p, b, 0);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return fail(SVM_ENOMEM, "cudaMallocAsync(%zu bytes) failed: %s", b, cudaGetErrorString(e));
        }
        bytes = b;
        return SVM_OK;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

static bool is_device_ptr(const void* p)
{
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// copy n elements of T from (host or device) src into a new device buffer
template <class T>
static int to_device(DBuf& dst, const T* src, int64_t n, cudaStream_t st)
{
    TRY(dst.alloc(sizeof(T) * (size_t)std::max<int64_t>(n, 1)));
    if (n > 0)
        CK(cudaMemcpyAsync(dst.p, src, sizeof(T) * n,
                           is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    return SVM_OK;
}

template <class T>
static int to_host(std::vector<T>& dst, const T* src, int64_t n, cudaStream_t st)
{
    dst.resize((size_t)std::max<int64_t>(n, 0));
    if (n > 0) {
        CK(cudaMemcpyAsync(dst.data(), src, sizeof(T) * n,
                           is_device_ptr(src) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    return SVM_OK;
}

static int sm_count()
{
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 1;
}

static double now_ms()
{
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ================================================================ parameters
extern "C" int svm_params_default(svm_params* p, int64_t d)
{
    if (!p || d < 1) return fail(SVM_EINVAL, "svm_params_default: NULL params or d < 1");
    memset(p, 0, sizeof *p);
    p->type = SVM_C_CLASSIFICATION;
    p->kernel = SVM_RADIAL;
    p->cost = 1.0;
    p->gamma = 1.0 / (double)d;
    p->degree = 3;
    p->coef0 = 0.0;
    p->epsilon = 0.1;
    p->tolerance = 1e-3;          // e1071 default
    p->working_set = 16;
    p->max_iter = 0;
    p->layout = SVM_ROW_MAJOR;
    p->certify = -1;
    p->stream = nullptr;
    return SVM_OK;
}

static int check_params(const svm_params* p, int64_t n, int64_t d)
{
    if (!p) return fail(SVM_EINVAL, "params is NULL");
    if (n < 2) return fail(SVM_EINVAL, "need n >= 2 training rows (got %lld)", (long long)n);
    if (d < 1) return fail(SVM_EINVAL, "need d >= 1 features (got %lld)", (long long)d);
    if (d > 3072) return fail(SVM_EINVAL, "d = %lld exceeds the fused pass limit of 3072", (long long)d);
    if (p->type != SVM_C_CLASSIFICATION && p->type != SVM_EPS_REGRESSION)
        return fail(SVM_EINVAL, "type must be SVM_C_CLASSIFICATION or SVM_EPS_REGRESSION");
    if (p->kernel < SVM_LINEAR || p->kernel > SVM_SIGMOID) return fail(SVM_EINVAL, "bad kernel");
    if (!(p->cost > 0.0) || !std::isfinite(p->cost)) return fail(SVM_EINVAL, "cost must be > 0");
    if (!std::isfinite(p->gamma)) return fail(SVM_EINVAL, "gamma must be finite");
    if (p->kernel == SVM_POLYNOMIAL && p->degree < 1) return fail(SVM_EINVAL, "degree must be >= 1");
    if (!(p->epsilon >= 0.0) || !std::isfinite(p->epsilon)) return fail(SVM_EINVAL, "epsilon must be >= 0");
    if (!(p->tolerance > 0.0) || !std::isfinite(p->tolerance))
        return fail(SVM_EINVAL, "tolerance must be > 0");
    if (p->working_set < 2 || p->working_set > SVM_WS || (p->working_set & 1))
        return fail(SVM_EINVAL, "working_set must be even and in [2, 16] (got %d)", p->working_set);
    if (p->layout != SVM_ROW_MAJOR && p->layout != SVM_COL_MAJOR) return fail(SVM_EINVAL, "bad layout");
    if (!(p->coef0 == p->coef0)) return fail(SVM_EINVAL, "coef0 is NaN");
    return SVM_OK;
}

static KParams kparams(const svm_params* p, int64_t d)
{
    KParams k;
    k.kernel = p->kernel;
    k.degree = p->degree;
    k.gamma64 = p->gamma > 0.0 ? p->gamma : 1.0 / (double)d;
    k.coef064 = p->coef0;
    k.gamma = (float)k.gamma64;
    k.coef0 = (float)p->coef0;
    return k;
}

// ================================================================ training data on the device
struct Data {
    int64_t n = 0, d = 0, n_pad = 0, rows_per_cta = 0, nnz = 0;
    int nblk = 0;
    bool csr = false;
    DBuf XT, XR_own, norms, indptr_own, indices_own, vals_own;
    DBuf sell_idx, sell_val, sell_gptr;   // CSR in slices of 32 rows for the pass (build_sell)
    int sell_spc = 0;
    const float* XR = nullptr;            // row-major rows (owned or borrowed)
    const int64_t* indptr = nullptr;      // CSR (owned or borrowed)
    const int32_t* indices = nullptr;
    const float* vals = nullptr;
};

static int pick_nblk(int64_t n)
{
    const char* env = getenv("SVMB200_NBLK");
    int sms = sm_count();
    if (env && atoi(env) > 0) return std::min(atoi(env), sms);
    int64_t want = (n + 255) / 256;  // >= 256 rows per CTA before using more SMs
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, sms));
}

static void set_geometry(Data& D, int64_t n, int nblk)
{
    D.nblk = nblk;
    int64_t per = (n + nblk - 1) / nblk;
    D.rows_per_cta = (per + 3) / 4 * 4;
    D.n_pad = D.rows_per_cta * nblk;
}

static int check_bad_flag(DBuf& flag, cudaStream_t st, int code, const char* what)
{
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h) return fail(code, "%s", what);
    return SVM_OK;
}

static int build_dense(Data& D, const float* X, int64_t n, int64_t d, int layout, int nblk,
                       cudaStream_t st)
{
    if (!X) return fail(SVM_EINVAL, "X is NULL");
    D.n = n;
    D.d = d;
    D.csr = false;
    set_geometry(D, n, nblk);
    TRY(D.XT.alloc(sizeof(float) * D.n_pad * d));
    TRY(D.norms.alloc(sizeof(float) * D.n_pad));
    bool dev = is_device_ptr(X);
    DBuf tmp;
    const float* Xd = X;
    if (!dev) {
        TRY(tmp.alloc(sizeof(float) * n * d));
        CK(cudaMemcpyAsync(tmp.p, X, sizeof(float) * n * d, cudaMemcpyHostToDevice, st));
        Xd = tmp.as<float>();
    }
    if (layout == SVM_ROW_MAJOR) {
        CK(lay_rowmajor_to_XT(Xd, n, d, D.XT.as<float>(), D.n_pad, st));
        if (dev) D.XR = X;  // borrowed for the call
        else {
            D.XR_own.p = tmp.p;  // keep the uploaded row-major copy
            D.XR_own.bytes = tmp.bytes;
            tmp.p = nullptr;
            D.XR = D.XR_own.as<float>();
        }
    } else {
        CK(lay_colmajor_to_XT(Xd, n, d, D.XT.as<float>(), D.n_pad, st));
        TRY(D.XR_own.alloc(sizeof(float) * n * d));
        CK(lay_XT_to_rowmajor(D.XT.as<float>(), n, d, D.n_pad, D.XR_own.as<float>(), st));
        D.XR = D.XR_own.as<float>();
    }
    DBuf bad;
    TRY(bad.alloc(sizeof(int)));
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    CK(lay_check_finite(D.XT.as<float>(), D.n_pad * d, bad.as<int>(), st));
    TRY(check_bad_flag(bad, st, SVM_ENONFINITE, "X contains a non-finite value"));
    CK(lay_norms_XT(D.XT.as<float>(), n, d, D.n_pad, D.norms.as<float>(), st));
    return SVM_OK;
}

// The pass's copy of a CSR matrix (SmoArgs::sell_*, layout.cu k_sell_fill): the rows of every
// 32-row warp chunk of every CTA interleaved lane by lane in groups of 4 nonzeros, so that a warp
// streams its chunk with coalesced 8- and 16-byte loads and no shared-memory staging.  Built for
// the CTA geometry of D (a virtual-rank launch partitions the rows identically).  Column indices
// are stored as u16 (the pass stages X_W^T [d][20] in shared memory, so d is far below 65536).
static int build_sell(Data& D, cudaStream_t st)
{
    D.sell_spc = 0;
    if (D.d > 65534 || getenv("SVMB200_CSR_STAGED")) return SVM_OK;   // per-warp staging path
    const int spc = (int)((D.rows_per_cta + 31) / 32);
    const int64_t ns = (int64_t)D.nblk * spc;
    DBuf len;
    TRY(len.alloc(sizeof(int64_t) * ns));
    CK(lay_sell_len(D.indptr, D.n, D.rows_per_cta, spc, ns, len.as<int64_t>(), st));
    std::vector<int64_t> h(ns + 1, 0);
    CK(cudaMemcpyAsync(h.data() + 1, len.p, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < ns; ++i) h[i + 1] += h[i];
    TRY(D.sell_gptr.alloc(sizeof(int64_t) * (ns + 1)));
    CK(cudaMemcpyAsync(D.sell_gptr.p, h.data(), sizeof(int64_t) * (ns + 1), cudaMemcpyHostToDevice, st));
    const int64_t groups = std::max<int64_t>(h[ns], 1);
    // skewed row lengths pad every slice to its longest row: beyond 4x the CSR bytes (+64 MB) the
    // per-warp staging path, which reads only the real nonzeros, is kept instead
    if ((double)groups * 32 * 24 > 4.0 * 8.0 * (double)D.nnz + 64.0 * (1 << 20)) return SVM_OK;
    TRY(D.sell_idx.alloc(sizeof(uint2) * groups * 32));
    TRY(D.sell_val.alloc(sizeof(float4) * groups * 32));
    CK(lay_sell_fill(D.indptr, D.indices, D.vals, D.n, D.d, D.rows_per_cta, spc, ns,
                     D.sell_gptr.as<int64_t>(), D.sell_idx.as<uint2>(), D.sell_val.as<float4>(), st));
    CK(cudaStreamSynchronize(st));   // h is freed on return
    D.sell_spc = spc;
    return SVM_OK;
}

static int build_csr(Data& D, const int64_t* indptr, const int32_t* indices, const float* data,
                     int64_t n, int64_t d, int nblk, cudaStream_t st)
{
    if (!indptr || !indices || !data) return fail(SVM_EINVAL, "CSR arrays must not be NULL");
    D.n = n;
    D.d = d;
    D.csr = true;
    set_geometry(D, n, nblk);
    // nnz from indptr[n]
    int64_t nnz = 0, first = 0;
    if (is_device_ptr(indptr)) {
        CK(cudaMemcpyAsync(&nnz, indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&first, indptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else {
        nnz = indptr[n];
        first = indptr[0];
    }
    if (first != 0 || nnz < 0) return fail(SVM_EINVAL, "CSR indptr[0] must be 0 and indptr[n] >= 0");
    D.nnz = nnz;
    if (is_device_ptr(indptr)) D.indptr = indptr;
    else { TRY(to_device(D.indptr_own, indptr, n + 1, st)); D.indptr = D.indptr_own.as<int64_t>(); }
    if (is_device_ptr(indices)) D.indices = indices;
    else { TRY(to_device(D.indices_own, indices, nnz, st)); D.indices = D.indices_own.as<int32_t>(); }
    if (is_device_ptr(data)) D.vals = data;
    else { TRY(to_device(D.vals_own, data, nnz, st)); D.vals = D.vals_own.as<float>(); }
    DBuf bad;
    TRY(bad.alloc(sizeof(int)));
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    CK(lay_check_csr(D.indptr, D.indices, n, d, nnz, bad.as<int>(), st));
    TRY(check_bad_flag(bad, st, SVM_EINVAL,
                       "CSR invariants violated (indptr non-decreasing, columns strictly increasing "
                       "within a row and < d)"));
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    CK(lay_check_finite(D.vals, nnz, bad.as<int>(), st));
    TRY(check_bad_flag(bad, st, SVM_ENONFINITE, "X contains a non-finite value"));
    TRY(D.norms.alloc(sizeof(float) * D.n_pad));
    CK(lay_norms_csr(D.indptr, D.vals, n, D.n_pad, D.norms.as<float>(), st));
    return build_sell(D, st);
}

// Handles that outlive the call (svm_solver, svm_batch) must not keep the caller's device arrays
// (the header's rule: inputs are borrowed for the call only): copy every borrowed pointer of D
// into a buffer D owns.
static int own_inputs(Data& D, cudaStream_t st)
{
    if (!D.csr && D.XR && !D.XR_own.p) {
        TRY(D.XR_own.alloc(sizeof(float) * D.n * D.d));
        CK(cudaMemcpyAsync(D.XR_own.p, D.XR, sizeof(float) * D.n * D.d, cudaMemcpyDeviceToDevice, st));
        D.XR = D.XR_own.as<float>();
    }
    if (D.csr) {
        if (!D.indptr_own.p) {
            TRY(D.indptr_own.alloc(sizeof(int64_t) * (D.n + 1)));
            CK(cudaMemcpyAsync(D.indptr_own.p, D.indptr, sizeof(int64_t) * (D.n + 1), cudaMemcpyDeviceToDevice, st));
            D.indptr = D.indptr_own.as<int64_t>();
        }
        if (!D.indices_own.p) {
            TRY(D.indices_own.alloc(sizeof(int32_t) * std::max<int64_t>(D.nnz, 1)));
            CK(cudaMemcpyAsync(D.indices_own.p, D.indices, sizeof(int32_t) * D.nnz, cudaMemcpyDeviceToDevice, st));
            D.indices = D.indices_own.as<int32_t>();
        }
        if (!D.vals_own.p) {
            TRY(D.vals_own.alloc(sizeof(float) * std::max<int64_t>(D.nnz, 1)));
            CK(cudaMemcpyAsync(D.vals_own.p, D.vals, sizeof(float) * D.nnz, cudaMemcpyDeviceToDevice, st));
            D.vals = D.vals_own.as<float>();
        }
    }
    return SVM_OK;
}

// ================================================================ one binary problem (Eq. 2)
struct Exchange {
    int L = 0, nbuf = 0;         // CTA lists per rank; buffers (1, or the virtual ranks of a launch)
    DBuf xw, info;               // per buffer: rank level [2][SVM_MAX_RANKS][XW_RANK_SLOT] then the
                                 // local level [2][L][XW_PER_SLOT] (self-tagged words); loop info
    uint32_t epoch = 0;
    static int64_t words(int L_) { return XW_RANK_WORDS + 2 * (int64_t)L_ * XW_PER_SLOT; }
    uint64_t* buf(int r) const { return xw.as<uint64_t>() + r * words(L); }
    int alloc(int L_, int nbuf_ = 1)
    {
        L = L_;
        nbuf = nbuf_;
        xw.release();
        TRY(xw.alloc(sizeof(uint64_t) * words(L) * nbuf));
        if (!info.p) TRY(info.alloc(sizeof(SmoInfo)));
        CK(cudaMemset(xw.p, 0, xw.bytes));
        return SVM_OK;
    }
};

// Stop / certification target as a fraction of the requested tolerance (reading R16,
// SURVEY 8(c) "Proposals"): the certified violation is computed with fp32-accurate kernel values
// (fp64 sums), and at full size it sat up to 1.8e-5 below the fp64-recomputed one (c3, tol 1e-3);
// aiming at 0.95 tol keeps the fp64 violation <= tol.
#define SVM_CERT_MARGIN_DEFAULT 0.95
// (SVMB200_CERT_MARGIN overrides the certification target only, not the loop's first stop: a
// test knob that forces resumptions)
static double cert_margin()
{
    const char* e = getenv("SVMB200_CERT_MARGIN");
    return (e && atof(e) > 0 && atof(e) <= 1) ? atof(e) : SVM_CERT_MARGIN_DEFAULT;
}
#define SVM_CERT_MARGIN cert_margin()

struct Problem {
    int ncopy = 1;
    double C = 1, eps = 0.1, tol = 1e-3;
    int q = 16;
    int64_t max_iter = 0;
    KParams kp;
    DBuf alpha, G, status, yv;   // yv: +-1 labels or z, fp32 [n]
    int64_t iterations = 0;
    double m_up = 0, M_low = 0;
    bool converged = false, certified = false;
    double tol_loop = 0;   // the loop's stop threshold: SVM_CERT_MARGIN tol, lowered after a failed
                           // certification (R16)
    double loop_ms = 0, cert_ms = 0;
    int32_t n_cert = 0;     // certifications run (1 + resumptions when every loop was certified)
    double exch_ms = 0;    // share of loop_ms CTA 0 spent in the candidate exchange
    double exch_hist[SMO_EXCH_BINS] = {};   // per-iteration exchange latency histogram (us units
                                            // after scaling: see exch_percentile)
    double us_per_cycle = 0;                // loop_ms / loop_cycles of the last launch
    int64_t cache_allhit = 0;               // iterations run as kernel-column-cache passes
    int64_t passes = 0;    // X passes of the dominant pass kernel (batched one-vs-rest: k_ovr_pass)
    double pass_ms = 0;    // their device time (CUDA event pairs around each launch)
    SmoInfo last_info;
};

static int problem_init(Problem& P, const Data& D, const float* yv_host, const svm_params* prm,
                        cudaStream_t st)
{
    P.ncopy = prm->type == SVM_EPS_REGRESSION ? 2 : 1;
    P.C = prm->cost;
    P.eps = prm->epsilon;
    P.tol = prm->tolerance;
    P.tol_loop = SVM_CERT_MARGIN_DEFAULT * prm->tolerance;   // DESIGN.md reading R16
    P.q = prm->working_set;
    int64_t m = D.n * P.ncopy;
    P.max_iter = prm->max_iter > 0 ? prm->max_iter : std::max<int64_t>(10 * m, 10000);
    P.kp = kparams(prm, D.d);
    TRY(P.alpha.alloc(sizeof(double) * D.n_pad * P.ncopy));
    TRY(P.G.alloc(sizeof(float) * D.n_pad * P.ncopy));
    TRY(P.status.alloc(D.n_pad * P.ncopy));
    TRY(to_device(P.yv, yv_host, D.n, st));
    CK(lay_init_state(P.yv.as<float>(), D.n, D.n_pad, P.ncopy, P.eps, P.C, P.alpha.as<double>(),
                      P.G.as<float>(), P.status.as<uint8_t>(), st));
    return SVM_OK;
}

// Peer view of a sharded run (world = 1 when NULL).
struct ShardCtx {
    int rank = 0, world = 1;
    int64_t row0 = 0, n_global = 0;
    int64_t rank_row0[SVM_MAX_RANKS + 1] = {};
    const float* XR[SVM_MAX_RANKS] = {};
    const float* norms[SVM_MAX_RANKS] = {};
    const int64_t* indptr[SVM_MAX_RANKS] = {};
    const int32_t* indices[SVM_MAX_RANKS] = {};
    const float* vals[SVM_MAX_RANKS] = {};
    int64_t rpc[SVM_MAX_RANKS] = {};
    uint64_t* xw[SVM_MAX_RANKS] = {};
};

static SmoArgs make_args(const Data& D, Problem& P, Exchange& E, const ShardCtx* sc = nullptr)
{
    SmoArgs a;
    memset(&a, 0, sizeof a);
    a.XT = D.csr ? nullptr : D.XT.as<float>();
    a.indptr = D.indptr;
    a.indices = D.indices;
    a.vals = D.vals;
    a.xnorm = D.norms.as<float>();
    a.n_local = D.n;
    a.n_pad = D.n_pad;
    a.d = D.d;
    a.row0 = 0;
    a.n_global = D.n;
    a.rows_per_cta = D.rows_per_cta;
    a.ncopy = P.ncopy;
    // rows per thread: enough chunks to keep ~12 warps busy, fewer LDS per FMA when rows allow
    a.rpt = D.csr ? 1 : (D.rows_per_cta >= 12 * 128 ? 4 : (D.rows_per_cta >= 6 * 64 ? 2 : 1));
    if (const char* e = getenv("SVMB200_RPT")) {
        int v = atoi(e);
        a.rpt = D.csr ? 1 : (v == 4 ? 4 : (v == 2 ? 2 : 1));
    }
    a.alpha = P.alpha.as<double>();
    a.G = P.G.as<float>();
    a.status = P.status.as<uint8_t>();
    a.C = P.C;
    a.tol = P.tol_loop;
    a.inner_tol = std::max(0.1 * P.tol, 1e-10);  // DESIGN.md reading R2
    a.inner_max = 64 * P.q;
    a.q = P.q;
    a.kp = P.kp;
    a.rank = 0;
    a.world = 1;
    a.virt = 0;
    a.nblk = D.nblk;
    for (int r = 0; r < SVM_MAX_RANKS; ++r) a.rank_nblk[r] = D.nblk;   // equal on every rank
    a.rank_row0[0] = 0;
    a.rank_row0[1] = D.n;
    a.peer_XR[0] = D.XR;
    a.peer_xnorm[0] = D.norms.as<float>();
    a.peer_indptr[0] = D.indptr;
    a.peer_indices[0] = D.indices;
    a.peer_vals[0] = D.vals;
    if (D.csr && D.sell_spc > 0) {
        a.sell_idx = D.sell_idx.as<uint2>();
        a.sell_val = D.sell_val.as<float4>();
        a.sell_gptr = D.sell_gptr.as<int64_t>();
        a.sell_spc = D.sell_spc;
    }
    a.rank_rpc[0] = D.rows_per_cta;
    a.peer_xw[0] = E.buf(0);
    a.timeout_ns = 30ull * 1000000000ull;
    a.overlap = 2;   // (run_loop: 2 for X resident in shared memory, 1 for streamed X)
    a.qww_mma = (!D.csr && getenv("SVMB200_QWW_MMA") && atoi(getenv("SVMB200_QWW_MMA"))) ? 1 : 0;
    if (const char* e = getenv("SVMB200_OVERLAP")) a.overlap = atoi(e);
    a.info = E.info.as<SmoInfo>();
    if (sc && sc->world > 1) {
        a.rank = sc->rank;
        a.world = sc->world;
        a.row0 = sc->row0;
        a.n_global = sc->n_global;
        for (int r = 0; r <= sc->world; ++r) a.rank_row0[r] = sc->rank_row0[r];
        for (int r = 0; r < sc->world; ++r) {
            a.peer_XR[r] = sc->XR[r];
            a.peer_xnorm[r] = sc->norms[r];
            a.peer_indptr[r] = sc->indptr[r];
            a.peer_indices[r] = sc->indices[r];
            a.peer_vals[r] = sc->vals[r];
            a.rank_rpc[r] = sc->rpc[r];
            a.peer_xw[r] = sc->xw[r];
        }
        a.timeout_ns = 60ull * 1000000000ull;
    }
    return a;
}

// Launch variants of the persistent loop beyond plain training (tests and diagnostics).
struct LoopMode {
    int vranks = 1;                     // > 1: that many virtual ranks inside one launch
    const int64_t* pass_rows = nullptr; // pass-only diagnostic: fixed W rows (device) ...
    const float* pass_c = nullptr;      // ... and coefficients (device); max_iter = passes
    int pass_nr = 0;
    double* pass_ms = nullptr;          // out: device time of the pass-only launch
};

// TMA descriptor of X^T [d][n_pad] for the streamed dense pass: dim 0 = rows (contiguous), dim 1
// = features; box = {32 rpt rows, d features} -- one chunk of a CTA per tensor copy.  The encoder
// is the driver's cuTensorMapEncodeTiled, reached through the runtime (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled()
{
    static std::once_flag once;
    static EncodeTiledFn fn = nullptr;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
    });
    return fn;
}
static bool encode_x_map(CUtensorMap* map, const float* XT, int64_t n_pad, int64_t d, int rows)
{
    EncodeTiledFn fn = encode_tiled();
    if (!fn || d > 256 || rows > 256 || (n_pad * 4) % 16 != 0) return false;
    cuuint64_t dims[2] = {(cuuint64_t)n_pad, (cuuint64_t)d};
    cuuint64_t strides[1] = {(cuuint64_t)n_pad * 4};
    cuuint32_t box[2] = {(cuuint32_t)rows, (cuuint32_t)d};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(XT), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Virtual ranks (LoopMode::vranks = P): the launch's D.nblk CTAs form P ranks of D.nblk / P CTAs;
// rank r owns rows [r nblk_r R, (r + 1) nblk_r R) (clipped to n) -- the same rows its CTAs own in a
// one-rank launch, so alpha, G and the iteration count must be bit-identical to it.  Each virtual
// rank has its own exchange buffer; W rows, norms and payloads are gathered from their owner.
static int set_virtual_ranks(SmoArgs& a, const Data& D, Exchange& E, int P)
{
    if (P < 2 || P > SVM_MAX_RANKS || D.nblk % P != 0)
        return fail(SVM_EINVAL, "virtual ranks: %d must be in [2, %d] and divide the %d CTAs", P,
                    SVM_MAX_RANKS, D.nblk);
    const int nb = D.nblk / P;
    if (E.L != nb || E.nbuf != P) TRY(E.alloc(nb, P));
    a.virt = 1;
    a.world = P;
    a.nblk = nb;
    a.rank = 0;
    a.row0 = 0;
    a.n_global = D.n;
    for (int r = 0; r <= P; ++r) a.rank_row0[r] = std::min<int64_t>(D.n, (int64_t)r * nb * D.rows_per_cta);
    for (int r = 0; r < P; ++r) {
        const int64_t o = a.rank_row0[r];
        a.rank_nblk[r] = nb;
        a.rank_rpc[r] = D.rows_per_cta;
        a.peer_XR[r] = D.csr ? nullptr : D.XR + o * D.d;
        a.peer_xnorm[r] = D.norms.as<float>() + o;
        a.peer_indptr[r] = D.csr ? D.indptr + o : nullptr;
        a.peer_indices[r] = D.indices;
        a.peer_vals[r] = D.vals;
        a.peer_xw[r] = E.buf(r);
    }
    return SVM_OK;
}

// Run up to max_iter iterations of the persistent loop; accumulates into P.
static int run_loop(const Data& D, Problem& P, Exchange& E, int64_t max_iter, cudaStream_t st,
                    SmoInfo* info_out, const ShardCtx* sc = nullptr, const LoopMode* mode = nullptr)
{
    const LoopMode M0;
    const LoopMode& M = mode ? *mode : M0;
    if (M.vranks <= 1 && !sc && (E.L != D.nblk || E.nbuf != 1)) TRY(E.alloc(D.nblk));
    SmoArgs a = make_args(D, P, E, sc);
    if (M.vranks > 1) TRY(set_virtual_ranks(a, D, E, M.vranks));
    if (M.pass_rows) {
        a.pass_only = 1;
        a.pass_rows = M.pass_rows;
        a.pass_c = M.pass_c;
        a.pass_nr = M.pass_nr;
    }
    a.tag0 = E.epoch;
    a.max_iter = max_iter;

    CK(cudaMemsetAsync(E.info.p, 0, sizeof(SmoInfo), st));
    const int64_t pos_elems = D.rows_per_cta * P.ncopy;
    const int64_t smem_cap = 200 * 1024;
    int smem = smo_smem_bytes(D.d, a.world, a.nblk, D.csr ? 0 : D.rows_per_cta);
    if (!D.csr && smem <= smem_cap && !getenv("SVMB200_NO_XSMEM")) {
        a.x_in_smem = 1;  // this CTA's X slice stays resident in shared memory
    } else {
        // wide rows streamed from HBM: one row per lane and features split into slices, so that
        // enough (chunk, slice) items keep every warp's loads in flight
        if (!D.csr && D.d >= 256 && !getenv("SVMB200_RPT")) a.rpt = 1;
        a.x_ring = (!D.csr && (a.rpt >= 2 || D.d >= 256)) ? 1 : 0;
        if (const char* e = getenv("SVMB200_XRING")) a.x_ring = (!D.csr && atoi(e)) ? 1 : 0;
        smem = smo_smem_bytes(D.d, a.world, a.nblk, 0) +
               (D.csr ? (a.sell_spc > 0 ? smo_sell_bytes(a.sell_spc, D.d) : smo_csr_stage_bytes()) +
                            smo_csr_w_extra_bytes(D.d)
                      : smo_ring_bytes(a.rpt));
        // dense rows of <= 256 features: the TMA ring (one tensor copy per 32 rpt-row chunk)
        // (opt-in, SVMB200_TMA=1: measured slower than the per-lane ring on c4)
        if (!D.csr && D.d < 256 && getenv("SVMB200_TMA") && atoi(getenv("SVMB200_TMA"))) {
            const int64_t stage = D.d * 32 * a.rpt * 4;
            const int base = smo_smem_bytes(D.d, a.world, a.nblk, 0) + 128;
            int ns = 4;
            if (const char* e = getenv("SVMB200_TMA_STAGES")) ns = std::max(2, std::min(8, atoi(e)));
            while (ns > 2 && base + ns * stage > 150 * 1024) --ns;
            if (base + ns * stage <= 200 * 1024 &&
                encode_x_map(&a.xmap, D.XT.as<float>(), D.n_pad, D.d, 32 * a.rpt)) {
                a.x_tma = 1;
                a.tma_ns = ns;
                a.x_ring = 0;
                smem = base + (int)(ns * stage);
            }
        }
    }
    if (!a.x_in_smem && !D.csr && D.d >= 256 && a.rpt == 1 && D.rows_per_cta <= 14 * 32 &&
        !getenv("SVMB200_NO_WIDE")) {
        // wide streamed rows: CTA-wide bulk-copy pipeline (8 stages of wide_kc features x Rs
        // rows, Rs = 8 mod 32) feeding one-row-per-lane dot products held in registers
        const int64_t ncw = (D.rows_per_cta + 31) / 32, Rs = ncw * 32 + 8;
        const int base = smo_smem_bytes(D.d, a.world, a.nblk, 0);
        int64_t kc = std::min<int64_t>(16, (210 * 1024 - base) / (8 * 4 * Rs));
        if (kc < 4) kc = 0;
        if (kc > 0) {
            a.wide = 1;
            a.wide_kc = (int32_t)kc;
            a.x_ring = 0;
            smem = base + (int)(8 * 4 * kc * Rs);
        }
    }
    // phase-A warps while the subproblem runs: X resident in shared memory (c2, chain-bound) keeps
    // the solver's sub-partition free (2: c2 419 vs 451 ms); streamed X gives it to phase A too
    // (1: c4 3184 vs 3215 ms, c5 857 vs 860 ms per 3,000 iterations; round-2 measurements)
    if (!getenv("SVMB200_OVERLAP")) a.overlap = a.x_in_smem ? 2 : 1;
    const int dyn_cap = smo_dyn_smem_cap(a);   // (opt-in maximum - this variant's static SmoShared)
    if (smem > dyn_cap)
        return fail(SVM_EINVAL, "shared-memory need %d B exceeds the SM (d = %lld, %d + %d lists)",
                    smem, (long long)D.d, a.nblk, a.world);
    // dense (non-wide, non-TMA) chunks of fewer than 32 rpt rows (SVMB200_CHUNK_ROWS = rows, a
    // multiple of 4): opt-in only -- balancing the chunk count to a multiple of the 16 warps with
    // idle lanes measured slower (c4: 56.8 vs 48.6 us per iteration)
    a.chunk_rows = 0;
    if (!D.csr && !a.wide && !a.x_tma) {
        if (const char* e = getenv("SVMB200_CHUNK_ROWS")) {
            const int64_t c = 32 * a.rpt, v = atoll(e) / 4 * 4;
            if (v >= 4 && v < c) a.chunk_rows = (int32_t)v;
        }
    }
    // kernel-column cache: streamed X only (X resident in shared memory costs no
    // HBM; the wide and TMA pipelines consume every chunk of every iteration); up to 8192 columns
    // within min(12 GiB, 20% of the free device memory) -- inside the pool's retained bound, so
    // repeated trainings do not re-map it (c4: 6436 columns = the budget, bench 3.20 s; 3.29 s at 4096;
    // 10240 columns = 20 GB: 3.36 s, re-mapped every training; 16384 = 33 GB: +1.2-3 s).
    // SVMB200_CACHE = slots (0 = off).
    DBuf cdata, ctag, cstamp;
    if (!a.x_in_smem && !a.wide && !a.x_tma && !a.pass_only) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const int64_t col = D.n_pad * (int64_t)sizeof(float);
        const double budget = std::min(12.0 * (1ull << 30), 0.2 * (double)fr);
        int64_t slots = std::min<int64_t>(8192, (int64_t)budget / std::max<int64_t>(col, 1));
        if (const char* e = getenv("SVMB200_CACHE")) slots = std::min<int64_t>(atoll(e), 65536);
        slots = slots / 4 * 4;
        const int nctas = a.virt ? a.nblk * a.world : a.nblk;
        if (slots >= 16) {
            TRY(cdata.alloc((size_t)col * slots));
            TRY(ctag.alloc(sizeof(int32_t) * slots * nctas));
            TRY(cstamp.alloc(sizeof(uint32_t) * slots * nctas));
            CK(cudaMemsetAsync(ctag.p, 0xff, ctag.bytes, st));
            CK(cudaMemsetAsync(cstamp.p, 0, cstamp.bytes, st));
            a.cache_slots = (int32_t)slots;
            a.cache_data = cdata.as<float>();
            a.cache_tag = ctag.as<int32_t>();
            a.cache_stamp = cstamp.as<uint32_t>();
        }
    }
    {   // buffer the dot products of as many rows as fit (64 B per row), whole chunks only
        const int64_t chunk = 32 * a.rpt;
        const int64_t all_rows = (D.rows_per_cta + chunk - 1) / chunk * chunk;
        const int64_t avail = std::min<int64_t>(210 * 1024, dyn_cap) - smem;
        int64_t rows = avail / 64;
        rows = std::min<int64_t>(rows, all_rows);
        rows = rows / chunk * chunk;
        if (getenv("SVMB200_NO_DBUF") || a.wide) rows = 0;
        a.nslice = 1;
        if (!a.x_in_smem && !D.csr && !a.x_tma && D.d >= 256 && rows == all_rows) {
            // feature slices: as many as the partial buffers allow, >= 64 features each, aiming
            // at >= 4 items per warp
            const int64_t nch = all_rows / chunk;
            int64_t ns = std::min<int64_t>({avail / (64 * all_rows), D.d / 64, 8,
                                            (4 * SMO_WARPS + nch - 1) / nch});
            if (const char* e = getenv("SVMB200_NSLICE")) ns = std::min<int64_t>(ns, atoi(e));
            a.nslice = (int32_t)std::max<int64_t>(ns, 1);
        }
        a.dbuf_rows = (int32_t)std::max<int64_t>(rows, 0);
        smem += (int)(64 * a.dbuf_rows * a.nslice);
    }
    if (pos_elems > 65535)
        return fail(SVM_EINVAL, "%lld dual variables per CTA exceed the 16-bit candidate position",
                    (long long)pos_elems);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    cudaError_t le = launch_smo(a, smem, st);
    if (le != cudaSuccess) {
        smo_l2_restore();
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return fail(SVM_ECUDA, "persistent working-set kernel launch failed: %s (smem %d B, %d CTAs)",
                    cudaGetErrorString(le), smem, D.nblk);
    }
    CK(cudaEventRecord(e1, st));
    SmoInfo info;
    CK(cudaMemcpyAsync(&info, E.info.p, sizeof info, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    smo_l2_restore();   // launch_smo's persisting-L2 set-aside -> the caller's limit
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (info.error) return fail(SVM_ETIMEOUT, "working-set exchange timed out (a rank stopped)");
    E.epoch += (uint32_t)info.iterations + 1;
    if (a.pass_only) {   // a diagnostic: the solver's iteration bookkeeping is not advanced
        if (M.pass_ms) *M.pass_ms = ms;
        if (getenv("SVMB200_PROFILE")) {
            const double it = (double)std::max<int64_t>(1, info.iterations);
            fprintf(stderr, "[svmb200] pass-only %lld passes, %.3f ms: worker warp 0 (cycles/pass): B-dots %.0f "
                    "B-epilogue %.0f B-merge %.0f B-tail %.0f finish %.0f\n", (long long)info.iterations, ms,
                    info.phase_cycles[8] / it, info.phase_cycles[10] / it, info.phase_cycles[11] / it,
                    info.phase_cycles[12] / it, info.phase_cycles[13] / it);
        }
        if (info_out) *info_out = info;
        return SVM_OK;
    }
    P.iterations += info.iterations;
    P.m_up = info.m_up;
    P.M_low = info.M_low;
    P.converged = info.converged != 0;
    P.loop_ms += ms;
    if (info.loop_cycles > 0) P.exch_ms += ms * (double)info.exch_cycles / (double)info.loop_cycles;
    P.last_info = info;
    if (info.loop_cycles > 0) {
        P.us_per_cycle = ms * 1e3 / (double)info.loop_cycles;
        for (int b = 0; b < SMO_EXCH_BINS; ++b) P.exch_hist[b] += (double)info.exch_hist[b];
    }
    P.cache_allhit += info.cache_allhit;
    if (a.cache_slots > 0 && getenv("SVMB200_PROFILE"))
        fprintf(stderr, "[svmb200] column cache, %d slots: %lld iterations, row hit rate %.3f, "
                "cache-pass iterations %.3f\n", a.cache_slots, (long long)info.iterations,
                info.cache_lookups ? (double)info.cache_hits / (double)info.cache_lookups : 0.0,
                info.iterations ? (double)info.cache_allhit / (double)info.iterations : 0.0);
    if (getenv("SVMB200_PROFILE")) {
        int clk = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
        double tot = 0;
        for (int i = 0; i < 8; ++i) tot += (double)info.phase_cycles[i];
        fprintf(stderr, "[svmb200] %lld iters, %.1f ms: phases (cycles/iter) wait+stage %.0f merge+W %.0f rows %.0f "
                "qww %.0f sub %.0f A+sync %.0f B+finish %.0f publish %.0f | total %.0f | inner/iter %.1f\n",
                (long long)info.iterations, ms,
                info.phase_cycles[0] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[1] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[2] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[3] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[4] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[5] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[6] / (double)std::max<int64_t>(1, info.iterations),
                info.phase_cycles[7] / (double)std::max<int64_t>(1, info.iterations),
                tot / (double)std::max<int64_t>(1, info.iterations),
                info.inner_total / (double)std::max<int64_t>(1, info.iterations));
        (void)clk;
        const double it = (double)std::max<int64_t>(1, info.iterations);
        fprintf(stderr, "[svmb200]   worker warp 0 (cycles/iter): B-dots %.0f - %.0f B-epilogue %.0f "
                "B-merge %.0f B-tail %.0f finish %.0f | level-1 merge: first call %.0f, warm repeat %.0f\n",
                info.phase_cycles[8] / it, info.phase_cycles[9] / it,
                info.phase_cycles[10] / it, info.phase_cycles[11] / it, info.phase_cycles[12] / it,
                info.phase_cycles[13] / it, info.phase_cycles[14] / it, info.phase_cycles[15] / it);
    }
    if (info_out) *info_out = info;
    return SVM_OK;
}

// q-quantile (cycles, bin midpoint) of an exchange-latency histogram; 0 when empty.
static double exch_percentile(const double* h, double q)
{
    double tot = 0;
    for (int b = 0; b < SMO_EXCH_BINS; ++b) tot += h[b];
    if (tot <= 0) return 0.0;
    double acc = 0;
    for (int b = 0; b < SMO_EXCH_BINS; ++b) {
        acc += h[b];
        if (acc >= q * tot) return exch_bin_mid(b);
    }
    return exch_bin_mid(SMO_EXCH_BINS - 1);
}

// Per-row coefficients of problem P (device, fp64[n]) and the SV flags they imply.
static int problem_coef(const Data& D, const Problem& P, DBuf& coef, DBuf& flag, cudaStream_t st)
{
    TRY(coef.alloc(sizeof(double) * D.n));
    CK(lay_coef(P.alpha.as<double>(), P.status.as<uint8_t>(), D.n, D.n_pad, P.ncopy, P.C,
                coef.as<double>(), flag.as<uint8_t>(), st));
    return SVM_OK;
}

// Stream compaction of flagged rows -> device index list; returns count.
static int compact(const DBuf& flag, int64_t n, DBuf& idx, int64_t* count, cudaStream_t st)
{
    int nb = 0;
    DBuf cnt;
    TRY(cnt.alloc(sizeof(int32_t) * ((n + 1023) / 1024 + 1)));
    CK(lay_count_flags(flag.as<uint8_t>(), n, cnt.as<int32_t>(), &nb, st));
    std::vector<int32_t> hc(nb);
    CK(cudaMemcpyAsync(hc.data(), cnt.p, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int64_t> offs(nb);
    int64_t tot = 0;
    for (int i = 0; i < nb; ++i) { offs[i] = tot; tot += hc[i]; }
    DBuf doffs;
    TRY(to_device(doffs, offs.data(), nb, st));
    TRY(idx.alloc(sizeof(int64_t) * std::max<int64_t>(tot, 1)));
    CK(lay_scatter_flags(flag.as<uint8_t>(), n, doffs.as<int64_t>(), idx.as<int64_t>(), st));
    CK(cudaStreamSynchronize(st));
    *count = tot;
    return SVM_OK;
}

// Feature-major SV block (+ norms) for a given row index list; nsv_pad multiple of 64.
static int gather_rows_T(const Data& D, const DBuf& idx, int64_t nsv, int64_t nsv_pad, DBuf& SVT,
                         DBuf& svn, cudaStream_t st)
{
    TRY(SVT.alloc(sizeof(float) * D.d * nsv_pad));
    TRY(svn.alloc(sizeof(float) * nsv_pad));
    if (!D.csr) {
        CK(lay_gather_sv(D.XT.as<float>(), D.n_pad, D.d, D.norms.as<float>(), idx.as<int64_t>(), nsv,
                         nsv_pad, SVT.as<float>(), svn.as<float>(), st));
    } else {
        CK(cudaMemsetAsync(SVT.p, 0, SVT.bytes, st));
        CK(lay_csr_to_XT(D.indptr, D.indices, D.vals, idx.as<int64_t>(), nsv, 0, SVT.as<float>(),
                         nsv_pad, st));
        // norms of the gathered rows: reuse the SV gather of norms through a dense zero XT is not
        // possible for CSR; gather norms directly
        CK(lay_gather_sv(nullptr, 0, 0, D.norms.as<float>(), idx.as<int64_t>(), nsv, nsv_pad,
                         nullptr, svn.as<float>(), st));
    }
    return SVM_OK;
}

// Decision sums F[i] = sum_s coef_s K(sv_s, x_i) over the TRAINING rows (fp64 accumulation).
static int training_decision(const Data& D, const DBuf& SVT, const DBuf& svn, int64_t nsv,
                             int64_t nsv_pad, const DBuf& coef_sv, const KParams& kp, DBuf& F,
                             cudaStream_t st)
{
    TRY(F.alloc(sizeof(double) * D.n));
    // queries = training rows in feature-major form; dense: X^T (n_pad is a multiple of 4 but the
    // predict tile needs 128) -> process through a padded view when needed
    int64_t nq_pad = (D.n + 127) / 128 * 128;
    DBuf QT, qn;
    const float* qT = nullptr;
    const float* qnorm = nullptr;
    int64_t ld = 0;
    // the certification runs on the fp16-split kernel for every d (as predict does; 3xTF32 only
    // with SVMB200_NO_F16): it reads X^T with any leading dimension, so no padded copy
    const bool f16 = getenv("SVMB200_NO_F16") == nullptr;
    if (!D.csr && (D.n_pad % 128 == 0 || D.d > 128 || f16)) {
        qT = D.XT.as<float>();
        qnorm = D.norms.as<float>();
        ld = D.n_pad;
    } else {
        TRY(QT.alloc(sizeof(float) * D.d * nq_pad));
        TRY(qn.alloc(sizeof(float) * nq_pad));
        CK(cudaMemsetAsync(QT.p, 0, QT.bytes, st));
        CK(cudaMemsetAsync(qn.p, 0, qn.bytes, st));
        if (D.csr) {
            CK(lay_csr_to_XT(D.indptr, D.indices, D.vals, nullptr, D.n, 0, QT.as<float>(), nq_pad, st));
        } else {
            CK(cudaMemcpy2DAsync(QT.p, sizeof(float) * nq_pad, D.XT.p, sizeof(float) * D.n_pad,
                                 sizeof(float) * D.n, D.d, cudaMemcpyDeviceToDevice, st));
        }
        CK(cudaMemcpyAsync(qn.p, D.norms.p, sizeof(float) * D.n, cudaMemcpyDeviceToDevice, st));
        qT = QT.as<float>();
        qnorm = qn.as<float>();
        ld = nq_pad;
    }
    DBuf SVtc;
    const float* svtc = nullptr;
    if (pred_tc_dp(D.d) && !f16) {
        TRY(SVtc.alloc(sizeof(float) * pred_sv_tiles_floats(nsv_pad, D.d, 1)));
        CK(pred_sv_tiles(SVT.as<float>(), nsv_pad, D.d, coef_sv.as<double>(), 1, SVtc.as<float>(), st));
        svtc = SVtc.as<float>();
    }
    CK(pred_decision(qT, qnorm, D.n, ld, SVT.as<float>(), svn.as<float>(), nsv, nsv_pad, D.d,
                     coef_sv.as<double>(), 1, kp, F.as<double>(), st, svtc, /*f16_any_d=*/f16));
    return SVM_OK;
}

struct Reduced {
    double m_up, M_low, free_sum, free_cnt, dual;
};

static int reduce_state(const Data& D, const Problem& P, Reduced* r, cudaStream_t st)
{
    DBuf out;
    TRY(out.alloc(sizeof(double) * 5));
    CK(lay_reduce_state(P.alpha.as<double>(), P.G.as<float>(), P.status.as<uint8_t>(),
                        P.yv.as<float>(), D.n, D.n_pad, P.ncopy, P.eps, P.C, out.as<double>(), st));
    double h[5];
    CK(cudaMemcpyAsync(h, out.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *r = {h[0], h[1], h[2], h[3], h[4]};
    return SVM_OK;
}

static bool want_certify(const svm_params* prm, int64_t n, int64_t nsv, int64_t d)
{
    if (prm->certify == 0) return false;
    if (prm->certify > 0) return true;
    // auto: every BASELINE config (c5: 2e6 x 9.4e5 SVs x 400 = 7.5e14, one fp16-split tcgen05
    // decision pass of a few seconds against a ~100 s training); only far larger problems skip it
    return (double)n * (double)nsv * (double)d <= 2e15;
}

// What a certification leaves for the next one of the same solve: the fp64 decision sums F it
// computed and the coefficients they were computed from.
struct CertState {
    DBuf F, coef;
    bool valid = false;
};

// Certification (a4): recompute G = Q a + p from the support vectors with fp64 accumulation and
// re-measure the violation; returns it in *viol.  With a valid CertState (a resumed loop after an
// earlier certification of the same problem) only the rows whose coefficient changed since then
// enter: F += sum_{s changed} (coef_s - coef'_s) K(x_s, .) -- the same fp64 sums of fp32 kernel
// values as a full recomputation, over the ~16 x (resumed iterations) changed rows instead of
// every SV (c5: 13 k instead of 940 k rows).
static int certify(const Data& D, Problem& P, double* viol, cudaStream_t st, CertState* cs = nullptr)
{
    double t0 = now_ms();
    DBuf coef, flag, idx, SVT, svn, coef_sv, F;
    TRY(flag.alloc(D.n));
    CK(cudaMemsetAsync(flag.p, 0, D.n, st));
    TRY(problem_coef(D, P, coef, flag, st));
    const bool delta = cs && cs->valid && !getenv("SVMB200_FULL_RECERT");
    DBuf dcoef;
    if (delta) {   // coef <- coef - coef', flag <- changed, coef' <- coef
        TRY(dcoef.alloc(sizeof(double) * D.n));
        CK(lay_coef_delta(coef.as<double>(), cs->coef.as<double>(), D.n, dcoef.as<double>(),
                          flag.as<uint8_t>(), st));
        std::swap(coef.p, dcoef.p);
        std::swap(coef.bytes, dcoef.bytes);
        std::swap(coef.plain, dcoef.plain);
    }
    int64_t nsv = 0;
    TRY(compact(flag, D.n, idx, &nsv, st));
    const bool prof = getenv("SVMB200_PROFILE") != nullptr;
    double ta = prof ? (cudaStreamSynchronize(st), now_ms()) : 0;
    int64_t nsv_pad = std::max<int64_t>(64, (nsv + 63) / 64 * 64);
    TRY(gather_rows_T(D, idx, nsv, nsv_pad, SVT, svn, st));
    TRY(coef_sv.alloc(sizeof(double) * nsv_pad));
    CK(lay_gather_coef(coef.as<double>(), idx.as<int64_t>(), nsv, nsv_pad, coef_sv.as<double>(), st));
    double tb = prof ? (cudaStreamSynchronize(st), now_ms()) : 0;
    if (nsv > 0 || !delta) TRY(training_decision(D, SVT, svn, nsv, nsv_pad, coef_sv, P.kp, F, st));
    double tc = prof ? (cudaStreamSynchronize(st), now_ms()) : 0;
    if (delta) {
        if (nsv > 0) CK(lay_add_f64(cs->F.as<double>(), F.as<double>(), D.n, st));
    } else if (cs) {   // keep F and the coefficients for an incremental re-certification
        std::swap(cs->F.p, F.p);
        std::swap(cs->F.bytes, F.bytes);
        std::swap(cs->F.plain, F.plain);
        std::swap(cs->coef.p, coef.p);
        std::swap(cs->coef.bytes, coef.bytes);
        std::swap(cs->coef.plain, coef.plain);
        cs->valid = true;
    }
    const double* Fall = cs ? cs->F.as<double>() : F.as<double>();
    CK(pred_refresh_G(Fall, P.yv.as<float>(), P.status.as<uint8_t>(), D.n, D.n_pad,
                      P.ncopy, P.eps, P.G.as<float>(), st));
    Reduced r;
    TRY(reduce_state(D, P, &r, st));
    if (prof)
        fprintf(stderr, "[svmb200] certify%s: nsv %lld, coef+compact %.1f ms, SV gather %.1f ms, decision %.1f ms, "
                "refresh+reduce %.1f ms, violation %.3g\n", delta ? " (changed rows only)" : "",
                (long long)nsv, ta - t0, tb - ta, tc - tb,
                (cudaStreamSynchronize(st), now_ms()) - tc, r.m_up - r.M_low);
    P.m_up = r.m_up;
    P.M_low = r.M_low;
    *viol = r.m_up - r.M_low;
    P.certified = true;
    P.cert_ms += now_ms() - t0;
    ++P.n_cert;
    return SVM_OK;
}

// The full solve of one problem: loop to tolerance, then certification + resume (a4).
static int certify_resume(const Data& D, Problem& P, Exchange& E, const svm_params* prm,
                          cudaStream_t st);
static int solve_problem(const Data& D, Problem& P, Exchange& E, const svm_params* prm,
                         cudaStream_t st)
{
    TRY(run_loop(D, P, E, P.max_iter, st, nullptr));
    return certify_resume(D, P, E, prm, st);
}

// After a failed certification G has been recomputed from the SVs (fp64 accumulation), so the
// resumed loop starts from an accurate G; it stops below tol by resume_factor() times the measured
// excess (the fp32 drift of the first loop), and at least 1% of tol below the previous stop.
static double resume_factor()
{
    static double f = -1;
    if (f < 0) {
        const char* e = getenv("SVMB200_RESUME_K");
        f = e ? atof(e) : 0.5;
    }
    return f;
}

// Certification (a4, reading R16) and resumption of the persistent loop after a loop stopped.
// Every loop that stops converged is followed by a certification, including the last resumed
// one: the reported state is always the re-measured one (converged = 0 if the last check failed
// after SVM_MAX_RESUMES resumptions).
#define SVM_MAX_RESUMES 4
static int certify_resume(const Data& D, Problem& P, Exchange& E, const svm_params* prm,
                          cudaStream_t st)
{
    CertState cs;
    for (int round = 0;; ++round) {
        if (!P.converged || prm->certify == 0) break;
        if (prm->certify < 0 && round == 0) {  // auto: only when one pass over n x n_SV is affordable
            DBuf coef, flag, idx;
            TRY(flag.alloc(D.n));
            CK(cudaMemsetAsync(flag.p, 0, D.n, st));
            TRY(problem_coef(D, P, coef, flag, st));
            int64_t nsv = 0;
            TRY(compact(flag, D.n, idx, &nsv, st));
            if (!want_certify(prm, D.n, nsv, D.d)) break;
        }
        double viol = 0;
        TRY(certify(D, P, &viol, st, &cs));
        const double target = SVM_CERT_MARGIN * P.tol;
        if (viol <= target) { P.converged = true; break; }
        P.converged = viol <= P.tol;   // (reported if the resumptions run out)
        if (round == SVM_MAX_RESUMES) break;
        // fp32 G stopped just inside the target: resume below it by resume_factor() times the
        // measured excess, and at least 1% of tol below the previous stop
        P.tol_loop = std::min(P.tol_loop - 0.01 * P.tol, target - resume_factor() * (viol - target));
        int64_t left = P.max_iter - P.iterations;
        if (left <= 0) break;
        TRY(run_loop(D, P, E, left, st, nullptr));
    }
    return SVM_OK;
}

// ================================================================ model
struct svm_model {
    svm_model_info info;
    int64_t d = 0, nsv = 0, nsv_pad = 0;
    int n_out = 1, mode = 0;   // mode 0 regression, 1 binary, 2 one-vs-rest
    KParams kp;
    double first_label = 0;
    DBuf SVT, svnorm, coef, b, labels;  // coef fp64 [n_out][nsv_pad]
    DBuf SVtc;                          // tcgen05 SV tiles (built on the first predict, d <= 128)
    std::vector<int64_t> sv_index;
    std::vector<double> coef_host;      // [n_out][nsv]
};

// tcgen05 predict operands: the SVs as [tile][hi | lo][64 * dp] K-major core tiles (d <= 128)
static int build_sv_tiles(svm_model* M, cudaStream_t st)
{
    if (pred_tc_dp(M->d) == 0 || M->nsv_pad == 0) return SVM_OK;
    // predict takes the fp16-split kernel (k_decision_f16) for up to 16 outputs: no tiles needed
    if (M->n_out <= 16 && !getenv("SVMB200_NO_F16")) return SVM_OK;
    TRY(M->SVtc.alloc(sizeof(float) * pred_sv_tiles_floats(M->nsv_pad, M->d, M->n_out)));
    CK(pred_sv_tiles(M->SVT.as<float>(), M->nsv_pad, M->d, M->coef.as<double>(), M->n_out,
                     M->SVtc.as<float>(), st));
    return SVM_OK;
}

static int assemble_model(const Data& D, std::vector<Problem>& probs, const svm_params* prm,
                          svm_model* M, const std::vector<double>& bs, cudaStream_t st)
{
    const int np = (int)probs.size();
    DBuf flag;
    TRY(flag.alloc(D.n));
    CK(cudaMemsetAsync(flag.p, 0, D.n, st));
    std::vector<DBuf> coefs(np);
    for (int p = 0; p < np; ++p) TRY(problem_coef(D, probs[p], coefs[p], flag, st));
    DBuf idx;
    int64_t nsv = 0;
    TRY(compact(flag, D.n, idx, &nsv, st));
    M->nsv = nsv;
    M->nsv_pad = std::max<int64_t>(64, (nsv + 63) / 64 * 64);
    M->d = D.d;
    TRY(gather_rows_T(D, idx, nsv, M->nsv_pad, M->SVT, M->svnorm, st));
    TRY(M->coef.alloc(sizeof(double) * M->nsv_pad * np));
    for (int p = 0; p < np; ++p)
        CK(lay_gather_coef(coefs[p].as<double>(), idx.as<int64_t>(), nsv, M->nsv_pad,
                           M->coef.as<double>() + (int64_t)p * M->nsv_pad, st));
    M->n_out = np;
    TRY(build_sv_tiles(M, st));
    TRY(to_device(M->b, bs.data(), np, st));
    M->sv_index.resize(nsv);
    if (nsv) CK(cudaMemcpyAsync(M->sv_index.data(), idx.p, sizeof(int64_t) * nsv,
                                cudaMemcpyDeviceToHost, st));
    M->coef_host.resize((size_t)nsv * np);
    for (int p = 0; p < np; ++p)
        if (nsv) CK(cudaMemcpyAsync(M->coef_host.data() + (size_t)p * nsv,
                                    M->coef.as<double>() + (int64_t)p * M->nsv_pad,
                                    sizeof(double) * nsv, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    (void)prm;
    return SVM_OK;
}

// ================================================================ training entry points
static int label_problems(const svm_params* prm, const std::vector<float>& y,
                          std::vector<std::vector<float>>& ys, std::vector<double>& labels,
                          int* mode, double* first_label)
{
    int64_t n = (int64_t)y.size();
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(y[i])) return fail(SVM_ENONFINITE, "y[%lld] is not finite", (long long)i);
    if (prm->type == SVM_EPS_REGRESSION) {
        ys.assign(1, y);
        *mode = 0;
        return SVM_OK;
    }
    std::vector<double> order;          // first-appearance order
    std::map<double, int> seen;
    for (float v : y)
        if (seen.emplace((double)v, (int)order.size()).second) {
            order.push_back(v);
            if (order.size() > 64) return fail(SVM_EINVAL, "more than 64 classes");
        }
    if (order.size() < 2) return fail(SVM_EDEGENERATE, "classification labels have a single class");
    labels = order;
    *first_label = order[0];
    if (order.size() == 2) {
        *mode = 1;
        bool pm1 = (order[0] == 1.0 && order[1] == -1.0) || (order[0] == -1.0 && order[1] == 1.0);
        std::vector<float> yb(n);
        double pos = pm1 ? 1.0 : order[0];
        for (int64_t i = 0; i < n; ++i) yb[i] = ((double)y[i] == pos) ? 1.0f : -1.0f;
        if (pm1) labels = {1.0, -1.0};
        else labels = {order[0], order[1]};
        ys.assign(1, yb);
        return SVM_OK;
    }
    *mode = 2;                           // one-vs-rest (BASELINE config 3)
    ys.clear();
    for (double c : order) {
        std::vector<float> yb(n);
        for (int64_t i = 0; i < n; ++i) yb[i] = ((double)y[i] == c) ? 1.0f : -1.0f;
        ys.push_back(std::move(yb));
    }
    return SVM_OK;
}

// Batched one-vs-rest: all binary problems of one dense X iterate together, one
// X pass per iteration on tcgen05 (k_ovr_pass) and one CTA per problem for selection + subproblem
// (k_ovr_solve).  Every problem follows the single-problem iteration of P:53; *handled = false
// when the configuration is not covered (the problems are then solved one after another).
static int solve_batched(const Data& D, std::vector<Problem>& probs, const svm_params* prm,
                         cudaStream_t st, bool* handled)
{
    *handled = false;
    const int P = (int)probs.size();
    if (D.csr || P < 2 || P > OVR_MAXP || probs[0].ncopy != 1 || probs[0].q != SVM_WS ||
        getenv("SVMB200_NO_BATCH"))
        return SVM_OK;
    OvrArgs a;
    memset(&a, 0, sizeof a);
    a.XT = D.XT.as<float>();
    a.XR = D.XR;
    a.xnorm = D.norms.as<float>();
    a.n = D.n;
    a.n_pad = D.n_pad;
    a.d = D.d;
    a.P = P;
    for (int p = 0; p < P; ++p) {
        a.alpha[p] = probs[p].alpha.as<double>();
        a.G[p] = probs[p].G.as<float>();
        a.status[p] = probs[p].status.as<uint8_t>();
    }
    const Problem& P0 = probs[0];
    for (int p = 0; p < P; ++p) {   // per problem (one-vs-rest: all equal; CV grids: per cell)
        a.Cp[p] = probs[p].C;
        a.kpp[p] = probs[p].kp;
    }
    a.tol = P0.tol_loop;
    a.inner_tol = std::max(0.1 * P0.tol, 1e-10);   // DESIGN.md reading R2
    a.inner_max = 64 * P0.q;
    a.max_iter = P0.max_iter;
    a.NU = 16 * P;
    a.kch = OVR_KCH;
    a.nkc = (int)((D.d + a.kch - 1) / a.kch);
    a.nct = (int)((D.n + 127) / 128);
    // k_ovr_solve stages X_W in fp64 [d][24]: 192 B per feature of shared memory
    if (ovr_pass_smem(a) > 227 * 1024 || ((D.d + 3) & ~3) * 192 + 28 * 1024 > 227 * 1024) return SVM_OK;
    DBuf Utc, XH, scratch, unorm, ucoef, cand, done, iters, mup, mlow, inner;
    TRY(Utc.alloc(sizeof(uint16_t) * (size_t)a.nkc * 2 * a.NU * a.kch));
    TRY(XH.alloc(sizeof(uint16_t) * (size_t)a.nct * a.nkc * 2 * 128 * a.kch));
    TRY(scratch.alloc(sizeof(unsigned int)));
    TRY(unorm.alloc(sizeof(float) * a.NU));
    TRY(ucoef.alloc(sizeof(float) * a.NU));
    TRY(cand.alloc(sizeof(uint64_t) * (size_t)P * 2 * a.nct * 8));
    TRY(done.alloc(sizeof(int32_t) * P));
    TRY(iters.alloc(sizeof(int64_t) * P));
    TRY(mup.alloc(sizeof(double) * P));
    TRY(mlow.alloc(sizeof(double) * P));
    TRY(inner.alloc(sizeof(int64_t) * P));
    for (DBuf* b : {&Utc, &unorm, &ucoef, &done, &iters, &inner}) CK(cudaMemsetAsync(b->p, 0, b->bytes, st));
    const bool prof = getenv("SVMB200_PROFILE") != nullptr;
    DBuf profb;
    if (prof) {
        TRY(profb.alloc(sizeof(long long) * 64 * 3));
        CK(cudaMemsetAsync(profb.p, 0, profb.bytes, st));
        a.prof = profb.as<long long>();
    }
    a.Uh = Utc.as<uint16_t>();
    a.XH = XH.as<uint16_t>();
    CK(ovr_prepare(a, scratch.as<unsigned int>(), st));
    a.unorm = unorm.as<float>();
    a.ucoef = ucoef.as<float>();
    a.cand = cand.as<uint64_t>();
    a.done = done.as<int32_t>();
    a.iters = iters.as<int64_t>();
    a.mup = mup.as<double>();
    a.mlow = mlow.as<double>();
    a.inner_total = inner.as<int64_t>();
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // The pass launches are timed with CUDA event pairs on this stream, one launch in every
    // PASS_SAMPLE (an event between two kernels serialises them, which would undo the programmatic
    // dependent launch that overlaps a kernel's prologue with its predecessor's tail):
    // pass_ms = mean sampled duration x passes.  The host polls the done flags every POLL
    // iterations.
    constexpr int NEV = 16, PASS_SAMPLE = 8, POLL = 16;
    cudaEvent_t pev[NEV][2];
    for (int k = 0; k < NEV; ++k)
        for (int j = 0; j < 2; ++j) CK(cudaEventCreate(&pev[k][j]));
    int nrec = 0, nsampled = 0;
    int64_t passes = 0;
    double sampled_ms = 0;
    auto timed_pass = [&]() -> int {
        const bool sample = (passes % PASS_SAMPLE) == 0 && nrec < NEV;
        if (sample) CK(cudaEventRecord(pev[nrec][0], st));
        CK(launch_ovr_pass(a, st));
        if (sample) {
            CK(cudaEventRecord(pev[nrec][1], st));
            ++nrec;
        }
        ++passes;
        return SVM_OK;
    };
    auto drain = [&]() {   // after a stream synchronize
        for (int k = 0; k < nrec; ++k) {
            float t = 0;
            const cudaError_t te = cudaEventElapsedTime(&t, pev[k][0], pev[k][1]);
            if (te != cudaSuccess) { cudaGetLastError(); continue; }
            sampled_ms += t;
            ++nsampled;
        }
        nrec = 0;
    };
    CK(cudaEventRecord(e0, st));
    TRY(timed_pass());   // candidates of the initial state (all coefficients 0)
    // Active-problem compaction: at every host poll, problems that stopped leave the batch -- their
    // final counters are kept on the host, the others move to the leading slots (per-slot state,
    // candidate lists, pointers, gamma / C), and the next launches run with N = 16 x active MMA
    // columns and only the active problems' epilogues.  Each problem's arithmetic is unchanged.
    std::vector<int> orig(P);          // original problem of each slot
    for (int p = 0; p < P; ++p) orig[p] = p;
    std::vector<int32_t> dh(P), fin_done(P, 0);
    std::vector<int64_t> ih(P), fin_iters(P, 0), inh(P), fin_inner(P, 0);
    std::vector<double> uh(P), lh(P), fin_up(P, 0.0), fin_low(P, 0.0);
    const bool compact_ok = getenv("SVMB200_NO_COMPACT") == nullptr;
    const size_t cand_block = (size_t)2 * a.nct * 8;   // u64 keys per problem slot
    for (int64_t it = 0; it <= a.max_iter; ++it) {
        CK(launch_ovr_solve(a, st));
        TRY(timed_pass());
        if ((it % POLL) == POLL - 1) {   // host poll of the done flags
            const int PA = a.P;
            CK(cudaMemcpyAsync(dh.data(), a.done, sizeof(int32_t) * PA, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            drain();
            int active = 0;
            for (int q = 0; q < PA; ++q) active += dh[q] ? 0 : 1;
            if (active == 0) break;
            if (compact_ok && active < PA) {
                CK(cudaMemcpyAsync(ih.data(), a.iters, sizeof(int64_t) * PA, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(uh.data(), a.mup, sizeof(double) * PA, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(lh.data(), a.mlow, sizeof(double) * PA, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(inh.data(), a.inner_total, sizeof(int64_t) * PA, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                std::vector<int> norig;
                std::vector<int64_t> ni, nin;
                std::vector<double> nu, nl;
                for (int q = 0; q < PA; ++q) {
                    const int o = orig[q];
                    if (dh[q]) {   // finished: keep its final counters
                        fin_done[o] = 1; fin_iters[o] = ih[q]; fin_up[o] = uh[q]; fin_low[o] = lh[q];
                        fin_inner[o] = inh[q];
                        continue;
                    }
                    const int nq = (int)norig.size();
                    if (nq != q)   // candidate lists of the last pass follow their problem
                        CK(cudaMemcpyAsync(a.cand + (size_t)nq * cand_block, a.cand + (size_t)q * cand_block,
                                           sizeof(uint64_t) * cand_block, cudaMemcpyDeviceToDevice, st));
                    norig.push_back(o);
                    ni.push_back(ih[q]); nin.push_back(inh[q]); nu.push_back(uh[q]); nl.push_back(lh[q]);
                    a.alpha[nq] = probs[o].alpha.as<double>();
                    a.G[nq] = probs[o].G.as<float>();
                    a.status[nq] = probs[o].status.as<uint8_t>();
                    a.Cp[nq] = probs[o].C;
                    a.kpp[nq] = probs[o].kp;
                }
                std::vector<int32_t> zd(active, 0);
                CK(cudaMemcpyAsync(a.done, zd.data(), sizeof(int32_t) * active, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(a.iters, ni.data(), sizeof(int64_t) * active, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(a.inner_total, nin.data(), sizeof(int64_t) * active, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(a.mup, nu.data(), sizeof(double) * active, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(a.mlow, nl.data(), sizeof(double) * active, cudaMemcpyHostToDevice, st));
                CK(cudaStreamSynchronize(st));
                orig = norig;
                a.P = active;
                a.NU = 16 * active;
            }
        }
    }
    CK(launch_ovr_solve(a, st));   // stop tests of the final state
    CK(cudaEventRecord(e1, st));
    {
        const int PA = a.P;
        CK(cudaMemcpyAsync(dh.data(), a.done, sizeof(int32_t) * PA, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ih.data(), a.iters, sizeof(int64_t) * PA, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(uh.data(), a.mup, sizeof(double) * PA, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(lh.data(), a.mlow, sizeof(double) * PA, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int q = 0; q < PA; ++q) {
            const int o = orig[q];
            fin_done[o] = dh[q]; fin_iters[o] = ih[q]; fin_up[o] = uh[q]; fin_low[o] = lh[q];
        }
        dh = fin_done; ih = fin_iters; uh = fin_up; lh = fin_low;
    }
    drain();
    for (int k = 0; k < NEV; ++k)
        for (int j = 0; j < 2; ++j) cudaEventDestroy(pev[k][j]);
    const double pass_ms = nsampled ? sampled_ms / nsampled * (double)passes : 0.0;
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    probs[0].passes = passes;
    probs[0].pass_ms = pass_ms;
    for (int p = 0; p < P; ++p) {
        Problem& Pp = probs[p];
        Pp.iterations = ih[p];
        Pp.m_up = dh[p] ? uh[p] : 0.0;
        Pp.M_low = dh[p] ? lh[p] : 0.0;
        Pp.converged = dh[p] && (uh[p] - lh[p] <= Pp.tol_loop);
        Pp.loop_ms += ms / P;
    }
    if (prof) {
        std::vector<long long> ph(64 * 3);
        cudaMemcpy(ph.data(), a.prof, sizeof(long long) * ph.size(), cudaMemcpyDeviceToHost);
        const double np = (double)std::max<int64_t>(1, passes);
        auto w = [&](int warp, int k) { return (double)ph[3 * warp + k] / np; };
        fprintf(stderr, "[svmb200] k_ovr_pass CTA 0 per pass (cycles): producer wait %.0f issue %.0f | MMA tiles %.0f wait-TMEM %.0f | epilogue0 wait %.0f work %.0f\n",
                w(0, 0), w(0, 1), w(2, 0), w(2, 1), w(3, 0), w(3, 1));
        const double ns = (double)std::max<int64_t>(1, passes - 1);
        fprintf(stderr, "[svmb200] k_ovr_solve CTA 0 per iteration (cycles): merge %.0f W+rows %.0f K_WW sums %.0f kernel %.0f eta %.0f subproblem %.0f alpha+U %.0f\n",
                ph[96] / ns, ph[97] / ns, ph[101] / ns, ph[102] / ns, ph[98] / ns, ph[99] / ns, ph[100] / ns);
    }
    if (prof) {
        int64_t mx = 0, sum = 0;
        for (int p = 0; p < P; ++p) { mx = std::max(mx, ih[p]); sum += ih[p]; }
        fprintf(stderr, "[svmb200] batched OvR: %d problems, %lld iterations (max), %lld in total, %.1f ms, %.1f us per batched iteration\n",
                P, (long long)mx, (long long)sum, ms, 1e3 * ms / std::max<int64_t>(1, mx));
    }
    *handled = true;
    return SVM_OK;
}

static int train_common(Data& D, const float* y, const svm_params* prm, svm_model** out,
                        double t_start, cudaStream_t st)
{
    std::vector<float> yh;
    TRY(to_host(yh, y, D.n, st));
    std::vector<std::vector<float>> ys;
    std::vector<double> labels;
    int mode = 0;
    double first = 0;
    TRY(label_problems(prm, yh, ys, labels, &mode, &first));
    double t_setup = now_ms() - t_start;
    Exchange E;
    TRY(E.alloc(D.nblk));
    std::vector<Problem> probs(ys.size());
    std::vector<double> bs(ys.size());
    double dual = 0, worst = -INFINITY, loop_ms = 0, cert_ms = 0, pass_ms = 0, exch_ms = 0;
    double xh[SMO_EXCH_BINS] = {}, upc = 0;
    int64_t cache_passes = 0;
    int64_t iters = 0, passes = 0;
    int32_t n_cert = 0;
    bool conv = true, cert = true;
    for (size_t p = 0; p < ys.size(); ++p) TRY(problem_init(probs[p], D, ys[p].data(), prm, st));
    bool batched = false;
    TRY(solve_batched(D, probs, prm, st, &batched));
    for (size_t p = 0; p < ys.size(); ++p) {
        Problem& P = probs[p];
        if (batched) TRY(certify_resume(D, P, E, prm, st));
        else TRY(solve_problem(D, P, E, prm, st));
        Reduced r;
        TRY(reduce_state(D, P, &r, st));
        // bias (sign-corrected; reading R6)
        bs[p] = r.free_cnt > 0 ? r.free_sum / r.free_cnt : 0.5 * (r.m_up + r.M_low);
        if (!std::isfinite(bs[p])) bs[p] = 0.0;
        dual += r.dual;
        worst = std::max(worst, r.m_up - r.M_low);
        iters += P.iterations;
        conv = conv && P.converged;
        cert = cert && P.certified;
        loop_ms += P.loop_ms;
        exch_ms += P.exch_ms;
        cache_passes += P.cache_allhit;
        for (int b = 0; b < SMO_EXCH_BINS; ++b) xh[b] += P.exch_hist[b];
        if (P.us_per_cycle > 0) upc = P.us_per_cycle;
        cert_ms += P.cert_ms;
        n_cert += P.n_cert;
        if (!batched) { passes += P.iterations; pass_ms += P.loop_ms; }
    }
    if (batched) { passes = probs[0].passes; pass_ms = probs[0].pass_ms; }
    svm_model* M = new (std::nothrow) svm_model();
    if (!M) return fail(SVM_ENOMEM, "model allocation failed");
    int rc = assemble_model(D, probs, prm, M, bs, st);
    if (rc != SVM_OK) { delete M; return rc; }
    M->mode = mode;
    M->n_out = (int)probs.size();
    M->kp = probs[0].kp;
    M->first_label = first;
    std::vector<double> lab = labels;
    if (lab.empty()) lab.push_back(0.0);
    rc = to_device(M->labels, lab.data(), (int64_t)lab.size(), st);
    if (rc != SVM_OK) { delete M; return rc; }
    svm_model_info& I = M->info;
    memset(&I, 0, sizeof I);
    I.type = prm->type;
    I.kernel = prm->kernel;
    I.degree = prm->degree;
    I.gamma = M->kp.gamma;
    I.coef0 = prm->coef0;
    I.n_features = D.d;
    I.n_train = D.n;
    I.n_sv = M->nsv;
    I.n_class = mode == 0 ? 0 : (int32_t)labels.size();
    I.n_problem = M->n_out;
    for (size_t i = 0; i < labels.size() && i < 64; ++i) I.labels[i] = labels[i];
    for (size_t i = 0; i < bs.size() && i < 64; ++i) I.b[i] = bs[i];
    I.iterations = iters;
    I.violation = worst;
    I.converged = conv ? 1 : 0;
    I.certified = cert ? 1 : 0;
    I.dual_objective = dual;
    I.loop_ms = loop_ms;
    I.exchange_ms = exch_ms;
    I.exchange_p50_us = exch_percentile(xh, 0.50) * upc;
    I.exchange_p99_us = exch_percentile(xh, 0.99) * upc;
    I.cache_passes = cache_passes;
    I.certifications = n_cert;
    I.certify_ms = cert_ms;
    I.setup_ms = t_setup;
    I.passes = passes;
    I.pass_ms = pass_ms;
    I.batched = batched ? 1 : 0;
    cudaStreamSynchronize(st);
    I.train_ms = now_ms() - t_start;
    *out = M;
    return SVM_OK;
}

extern "C" int svm_train(const float* X, const float* y, int64_t n, int64_t d,
                         const svm_params* params, svm_model** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    double t0 = now_ms();
    TRY(check_params(params, n, d));
    if (!X || !y) return fail(SVM_EINVAL, "X or y is NULL");
    cudaStream_t st = (cudaStream_t)params->stream;
    Data D;
    TRY(build_dense(D, X, n, d, params->layout, pick_nblk(n), st));
    return train_common(D, y, params, out, t0, st);
}

extern "C" int svm_train_csr(const int64_t* indptr, const int32_t* indices, const float* data,
                             const float* y, int64_t n, int64_t d, const svm_params* params,
                             svm_model** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    double t0 = now_ms();
    TRY(check_params(params, n, d));
    if (!y) return fail(SVM_EINVAL, "y is NULL");
    cudaStream_t st = (cudaStream_t)params->stream;
    Data D;
    TRY(build_csr(D, indptr, indices, data, n, d, pick_nblk(n), st));
    return train_common(D, y, params, out, t0, st);
}

// ================================================================ predict
static int predict_common(const svm_model* M, int64_t nq, const float* Xq_dense, int layout,
                          const int64_t* indptr, const int32_t* indices, const float* data,
                          float* decision, float* out)
{
    cudaStream_t st = nullptr;
    const int64_t CH = 65536;  // query rows per chunk
    bool dec_dev = is_device_ptr(decision), out_dev = is_device_ptr(out);
    DBuf hostX, QT, qn, F, ddec, dout;
    const float* Xd = Xq_dense;
    if (Xq_dense && !is_device_ptr(Xq_dense)) {
        TRY(hostX.alloc(sizeof(float) * nq * M->d));
        CK(cudaMemcpyAsync(hostX.p, Xq_dense, sizeof(float) * nq * M->d, cudaMemcpyHostToDevice, st));
        Xd = hostX.as<float>();
    }
    DBuf dptr, didx, dval;
    const int64_t* ip = indptr;
    const int32_t* ix = indices;
    const float* iv = data;
    if (!Xq_dense) {
        int64_t nnz = 0;
        if (is_device_ptr(indptr)) {
            CK(cudaMemcpyAsync(&nnz, indptr + nq, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else nnz = indptr[nq];
        if (!is_device_ptr(indptr)) { TRY(to_device(dptr, indptr, nq + 1, st)); ip = dptr.as<int64_t>(); }
        if (!is_device_ptr(indices)) { TRY(to_device(didx, indices, nnz, st)); ix = didx.as<int32_t>(); }
        if (!is_device_ptr(data)) { TRY(to_device(dval, data, nnz, st)); iv = dval.as<float>(); }
        DBuf bad;
        TRY(bad.alloc(sizeof(int)));
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        CK(lay_check_csr(ip, ix, nq, M->d, nnz, bad.as<int>(), st));
        TRY(check_bad_flag(bad, st, SVM_EINVAL, "query CSR invariants violated"));
    }
    int64_t chunk = std::min<int64_t>(CH, nq);
    int64_t cpad = (chunk + 127) / 128 * 128;
    TRY(QT.alloc(sizeof(float) * M->d * cpad));
    TRY(qn.alloc(sizeof(float) * cpad));
    TRY(F.alloc(sizeof(double) * chunk * M->n_out));
    TRY(ddec.alloc(sizeof(float) * chunk * M->n_out));
    TRY(dout.alloc(sizeof(float) * chunk));
    for (int64_t q0 = 0; q0 < nq; q0 += chunk) {
        int64_t m = std::min(chunk, nq - q0);
        if (Xq_dense) {
            if (layout == SVM_ROW_MAJOR) {
                CK(lay_rowmajor_to_XT(Xd + q0 * M->d, m, M->d, QT.as<float>(), cpad, st));
            } else {
                // column-major queries: column k of the chunk starts at Xd + k * nq + q0
                CK(cudaMemsetAsync(QT.p, 0, QT.bytes, st));
                CK(cudaMemcpy2DAsync(QT.p, sizeof(float) * cpad, Xd + q0, sizeof(float) * nq,
                                     sizeof(float) * m, M->d, cudaMemcpyDeviceToDevice, st));
            }
        } else {
            CK(cudaMemsetAsync(QT.p, 0, QT.bytes, st));
            CK(lay_csr_to_XT(ip, ix, iv, nullptr, m, q0, QT.as<float>(), cpad, st));
        }
        DBuf bad;
        TRY(bad.alloc(sizeof(int)));
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        CK(lay_check_finite(QT.as<float>(), M->d * cpad, bad.as<int>(), st));
        TRY(check_bad_flag(bad, st, SVM_ENONFINITE, "query X contains a non-finite value"));
        CK(lay_norms_XT(QT.as<float>(), m, M->d, cpad, qn.as<float>(), st));
        CK(pred_decision(QT.as<float>(), qn.as<float>(), m, cpad, M->SVT.as<float>(),
                         M->svnorm.as<float>(), M->nsv, M->nsv_pad, M->d, M->coef.as<double>(),
                         M->n_out, M->kp, F.as<double>(), st, M->SVtc.p ? M->SVtc.as<float>() : nullptr,
                         /*f16_any_d=*/true));
        CK(pred_finalize(F.as<double>(), m, M->n_out, M->b.as<double>(), M->mode,
                         M->labels.as<double>(), M->first_label, ddec.as<float>(),
                         dout.as<float>(), st));
        if (decision)
            CK(cudaMemcpyAsync(decision + q0 * M->n_out, ddec.p, sizeof(float) * m * M->n_out,
                               dec_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        if (out)
            CK(cudaMemcpyAsync(out + q0, dout.p, sizeof(float) * m,
                               out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    return SVM_OK;
}

extern "C" int svm_predict(const svm_model* model, const float* Xq, int64_t nq, int64_t d,
                           int32_t layout, float* decision, float* out)
{
    if (!model) return fail(SVM_EINVAL, "model is NULL");
    if (d != model->d) return fail(SVM_EINVAL, "d = %lld does not match the model's %lld",
                                   (long long)d, (long long)model->d);
    if (nq < 0) return fail(SVM_EINVAL, "nq < 0");
    if (nq == 0) return SVM_OK;
    if (!Xq) return fail(SVM_EINVAL, "Xq is NULL");
    if (layout != SVM_ROW_MAJOR && layout != SVM_COL_MAJOR) return fail(SVM_EINVAL, "bad layout");
    return predict_common(model, nq, Xq, layout, nullptr, nullptr, nullptr, decision, out);
}

extern "C" int svm_predict_csr(const svm_model* model, const int64_t* indptr,
                               const int32_t* indices, const float* data, int64_t nq, int64_t d,
                               float* decision, float* out)
{
    if (!model) return fail(SVM_EINVAL, "model is NULL");
    if (d != model->d) return fail(SVM_EINVAL, "d = %lld does not match the model's %lld",
                                   (long long)d, (long long)model->d);
    if (nq < 0) return fail(SVM_EINVAL, "nq < 0");
    if (nq == 0) return SVM_OK;
    if (!indptr || !indices || !data) return fail(SVM_EINVAL, "CSR arrays must not be NULL");
    return predict_common(model, nq, nullptr, SVM_ROW_MAJOR, indptr, indices, data, decision, out);
}

extern "C" int svm_model_get_info(const svm_model* model, svm_model_info* info)
{
    if (!model || !info) return fail(SVM_EINVAL, "NULL model or info");
    *info = model->info;
    return SVM_OK;
}

extern "C" int svm_model_get_sv(const svm_model* model, int64_t* sv_index, double* coef)
{
    if (!model) return fail(SVM_EINVAL, "model is NULL");
    if (sv_index && model->nsv)
        memcpy(sv_index, model->sv_index.data(), sizeof(int64_t) * model->nsv);
    if (coef && !model->coef_host.empty())
        memcpy(coef, model->coef_host.data(), sizeof(double) * model->coef_host.size());
    return SVM_OK;
}

extern "C" void svm_free_model(svm_model* model) { delete model; }

extern "C" const char* svm_last_error(void) { return g_err.c_str(); }

// ================================================================ K-fold CV and grid (8(f) #4)
// SURVEY 8(f) #4 / P:49, P:77-78 ("K-fold cross validation", "tuning parameters"): every (grid
// cell, fold, class) is one Eq. 2 instance on the SAME device X: the held-out rows of the fold
// leave the problem through their status (lay_exclude_fold), the cell's gamma and C are per
// problem.  Classification problems run together through the batched tcgen05 pass (16 per batch,
// one X pass per iteration for all of them, per-problem gamma / C); eps-SVR problems run one after
// another on the persistent kernel.  After the loop every problem is certified (G recomputed from
// its SVs, fp64 sums) -- that G covers the held-out rows too, so the fold model's decision value
// on a held-out row is read off it: SVC f = y (G + 1) + b, SVR f = G+ - eps + z + b.
static double pearson(const std::vector<double>& a, const std::vector<double>& b)
{
    const size_t m = a.size();
    if (m < 2) return NAN;
    double ma = 0, mb = 0;
    for (size_t i = 0; i < m; ++i) { ma += a[i]; mb += b[i]; }
    ma /= (double)m;
    mb /= (double)m;
    double sab = 0, saa = 0, sbb = 0;
    for (size_t i = 0; i < m; ++i) {
        sab += (a[i] - ma) * (b[i] - mb);
        saa += (a[i] - ma) * (a[i] - ma);
        sbb += (b[i] - mb) * (b[i] - mb);
    }
    return (saa > 0 && sbb > 0) ? sab / std::sqrt(saa * sbb) : NAN;
}

extern "C" int svm_cross_validate(const float* X, const float* y, int64_t n, int64_t d,
                                  const svm_params* params, int32_t nfold, const int32_t* fold,
                                  int32_t ngrid, const double* gammas, const double* costs,
                                  svm_cv_result* results, double* cv_decision)
{
    if (!results) return fail(SVM_EINVAL, "results is NULL");
    TRY(check_params(params, n, d));
    if (!X || !y) return fail(SVM_EINVAL, "X or y is NULL");
    if (nfold < 2 || nfold > n) return fail(SVM_EINVAL, "nfold = %d must be in [2, n]", nfold);
    if (ngrid < 1) return fail(SVM_EINVAL, "ngrid must be >= 1");
    cudaStream_t st = (cudaStream_t)params->stream;
    for (int g = 0; g < ngrid; ++g) {
        if (gammas && !(gammas[g] > 0.0) && params->kernel != SVM_LINEAR)
            return fail(SVM_EINVAL, "gammas[%d] must be > 0", g);
        if (costs && !(costs[g] > 0.0)) return fail(SVM_EINVAL, "costs[%d] must be > 0", g);
    }
    // fold ids (host), validated; default round robin i mod nfold
    std::vector<int32_t> fh(n);
    if (fold) TRY(to_host(fh, fold, n, st));
    else for (int64_t i = 0; i < n; ++i) fh[i] = (int32_t)(i % nfold);
    std::vector<int64_t> fcount(nfold, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (fh[i] < 0 || fh[i] >= nfold) return fail(SVM_EINVAL, "fold[%lld] = %d outside [0, nfold)", (long long)i, fh[i]);
        ++fcount[fh[i]];
    }
    for (int f = 0; f < nfold; ++f)
        if (fcount[f] == 0) return fail(SVM_EINVAL, "fold %d is empty", f);
    Data D;
    TRY(build_dense(D, X, n, d, params->layout, pick_nblk(n), st));
    std::vector<float> yh;
    TRY(to_host(yh, y, n, st));
    std::vector<std::vector<float>> ys;
    std::vector<double> labels;
    int mode = 0;
    double first = 0;
    TRY(label_problems(params, yh, ys, labels, &mode, &first));
    const int k = (int)ys.size();
    DBuf dfold;
    TRY(to_device(dfold, fh.data(), n, st));
    // a fold fails when its training split has a single class (classification)
    std::vector<bool> fold_failed(nfold, false);
    if (mode != 0)
        for (int f = 0; f < nfold; ++f) {
            std::map<double, int> seen;
            for (int64_t i = 0; i < n; ++i)
                if (fh[i] != f) seen[(double)yh[i]] = 1;
            fold_failed[f] = seen.size() < 2;
        }
    // held-out decision values [ngrid][n][k]
    std::vector<double> dec((size_t)ngrid * n * k, 0.0);
    std::vector<int64_t> iters(ngrid, 0);
    std::vector<int> conv(ngrid, 1);
    Exchange E;
    TRY(E.alloc(D.nblk));
    struct Item { int g, f, c; };
    std::vector<Item> items;
    for (int g = 0; g < ngrid; ++g)
        for (int f = 0; f < nfold; ++f)
            for (int c = 0; c < k; ++c) items.push_back({g, f, c});
    const int per_batch = mode == 0 ? 1 : OVR_MAXP;
    std::vector<float> Gh(n);
    for (size_t b0 = 0; b0 < items.size(); b0 += per_batch) {
        const size_t b1 = std::min(items.size(), b0 + per_batch);
        std::vector<Problem> probs(b1 - b0);
        std::vector<svm_params> prms(b1 - b0);
        for (size_t j = b0; j < b1; ++j) {
            svm_params pg = *params;
            if (gammas) pg.gamma = gammas[items[j].g];
            if (costs) pg.cost = costs[items[j].g];
            prms[j - b0] = pg;
            Problem& Pr = probs[j - b0];
            TRY(problem_init(Pr, D, ys[items[j].c].data(), &pg, st));
            CK(lay_exclude_fold(dfold.as<int32_t>(), items[j].f, n, D.n_pad, Pr.ncopy,
                                Pr.status.as<uint8_t>(), st));
        }
        bool batched = false;
        if (probs.size() >= 2) TRY(solve_batched(D, probs, &prms[0], st, &batched));
        for (size_t j = b0; j < b1; ++j) {
            Problem& Pr = probs[j - b0];
            const svm_params& pg = prms[j - b0];
            if (batched) TRY(certify_resume(D, Pr, E, &pg, st));
            else TRY(solve_problem(D, Pr, E, &pg, st));
            if (!Pr.certified) {   // the held-out decision values come from a certified G
                double viol = 0;
                const bool c0 = Pr.converged;
                TRY(certify(D, Pr, &viol, st));
                Pr.converged = c0 && viol <= Pr.tol;
            }
            Reduced r;
            TRY(reduce_state(D, Pr, &r, st));
            double b = r.free_cnt > 0 ? r.free_sum / r.free_cnt : 0.5 * (r.m_up + r.M_low);
            if (!std::isfinite(b)) b = 0.0;
            CK(cudaMemcpyAsync(Gh.data(), Pr.G.p, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const Item it = items[j];
            iters[it.g] += Pr.iterations;
            if (!Pr.converged) conv[it.g] = 0;
            const std::vector<float>& yv = ys[it.c];
            for (int64_t i = 0; i < n; ++i) {
                if (fh[i] != it.f) continue;
                const double G = (double)Gh[i];
                const double f = mode == 0 ? G - Pr.eps + (double)yv[i] + b
                                           : (double)yv[i] * (G + 1.0) + b;
                dec[((size_t)it.g * n + i) * k + it.c] = f;
            }
        }
    }
    // metrics per cell: mean over the folds that did not fail
    for (int g = 0; g < ngrid; ++g) {
        svm_cv_result& R = results[g];
        memset(&R, 0, sizeof R);
        R.nfold = nfold;
        R.gamma = gammas ? gammas[g] : kparams(params, d).gamma64;
        R.cost = costs ? costs[g] : params->cost;
        R.iterations = iters[g];
        R.converged = conv[g];
        double msum = 0, psum = 0;
        int used = 0, pused = 0;
        for (int f = 0; f < nfold; ++f) {
            if (fold_failed[f]) { ++R.failed; continue; }
            std::vector<double> truth, pred;
            int64_t hit = 0, cnt = 0;
            for (int64_t i = 0; i < n; ++i) {
                if (fh[i] != f) continue;
                const double* fv = &dec[((size_t)g * n + i) * k];
                ++cnt;
                if (mode == 0) { truth.push_back(yh[i]); pred.push_back(fv[0]); continue; }
                double lab;
                if (mode == 1) lab = fv[0] > 0 ? labels[0] : (fv[0] < 0 ? labels[1] : first);
                else {
                    int best = 0;
                    for (int c = 1; c < k; ++c) if (fv[c] > fv[best]) best = c;   // ties -> lowest
                    lab = labels[best];
                }
                hit += lab == (double)yh[i] ? 1 : 0;
            }
            if (mode == 0) {
                double se = 0;
                for (size_t i = 0; i < truth.size(); ++i) se += (pred[i] - truth[i]) * (pred[i] - truth[i]);
                msum += se / (double)truth.size();
                const double pc = pearson(truth, pred);
                if (std::isfinite(pc)) { psum += pc; ++pused; }
            } else {
                msum += (double)hit / (double)cnt;
            }
            ++used;
        }
        R.metric = used ? msum / used : NAN;
        R.pearson = mode == 0 ? (pused ? psum / pused : NAN) : 0.0;
    }
    if (cv_decision) {
        if (is_device_ptr(cv_decision))
            CK(cudaMemcpy(cv_decision, dec.data(), sizeof(double) * dec.size(), cudaMemcpyHostToDevice));
        else
            memcpy(cv_decision, dec.data(), sizeof(double) * dec.size());
    }
    return SVM_OK;
}

// ================================================================ batched solver (8(f) #1)
// Stepwise access to the batched one-vs-rest machinery: P binary problems on one dense X, each
// iteration = one k_ovr_solve (selection, subproblem) + one k_ovr_pass (tcgen05 X X_U^T, G update,
// candidates) for all problems (parity tests of the batched pass; drivers).
struct svm_batch {
    Data D;
    std::vector<Problem> probs;
    svm_params prm;
    cudaStream_t st = nullptr;
};

extern "C" int svm_batch_create(const float* X, const float* Y, int32_t nprob, int64_t n,
                                int64_t d, const svm_params* params, svm_batch** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    TRY(check_params(params, n, d));
    if (!X || !Y) return fail(SVM_EINVAL, "X or Y is NULL");
    if (params->type != SVM_C_CLASSIFICATION) return fail(SVM_EINVAL, "batched problems are C-SVC");
    if (nprob < 2 || nprob > OVR_MAXP) return fail(SVM_EINVAL, "nprob must be in [2, %d]", OVR_MAXP);
    svm_batch* B = new (std::nothrow) svm_batch();
    if (!B) return fail(SVM_ENOMEM, "batch allocation failed");
    B->prm = *params;
    B->st = (cudaStream_t)params->stream;
    int rc = build_dense(B->D, X, n, d, params->layout, pick_nblk(n), B->st);
    if (rc == SVM_OK) rc = own_inputs(B->D, B->st);
    std::vector<float> yh;
    if (rc == SVM_OK) rc = to_host(yh, Y, (int64_t)nprob * n, B->st);
    if (rc == SVM_OK) {
        for (int64_t i = 0; i < (int64_t)nprob * n; ++i)
            if (yh[i] != 1.0f && yh[i] != -1.0f) { rc = fail(SVM_EINVAL, "Y must hold +-1 labels"); break; }
    }
    {
        std::vector<Problem> tmp(nprob);   // (Problem owns device buffers: not copyable)
        B->probs.swap(tmp);
    }
    for (int p = 0; p < nprob && rc == SVM_OK; ++p)
        rc = problem_init(B->probs[p], B->D, yh.data() + (size_t)p * n, params, B->st);
    if (rc == SVM_OK && cudaStreamSynchronize(B->st) != cudaSuccess) rc = fail(SVM_ECUDA, "setup failed");
    if (rc != SVM_OK) { delete B; return rc; }
    *out = B;
    return SVM_OK;
}

extern "C" int svm_batch_set_state(svm_batch* B, int32_t p, const double* alpha, const float* G)
{
    if (!B || !alpha || !G || p < 0 || p >= (int)B->probs.size()) return fail(SVM_EINVAL, "bad argument");
    Problem& P = B->probs[p];
    const int64_t n = B->D.n;
    std::vector<double> ah;
    TRY(to_host(ah, alpha, n, B->st));
    for (int64_t i = 0; i < n; ++i)
        if (!(ah[i] >= 0.0 && ah[i] <= P.C)) return fail(SVM_EINVAL, "alpha[%lld] outside [0, C]", (long long)i);
    DBuf da, dg;
    TRY(to_device(da, alpha, n, B->st));
    TRY(to_device(dg, G, n, B->st));
    CK(lay_unpack_state(da.as<double>(), dg.as<float>(), n, B->D.n_pad, 1, P.alpha.as<double>(),
                        P.G.as<float>(), B->st));
    CK(lay_status_from_alpha(P.alpha.as<double>(), n, B->D.n_pad, 1, P.C, P.status.as<uint8_t>(), B->st));
    CK(cudaStreamSynchronize(B->st));
    return SVM_OK;
}

extern "C" int svm_batch_get_state(const svm_batch* B, int32_t p, double* alpha, float* G)
{
    if (!B || p < 0 || p >= (int)B->probs.size()) return fail(SVM_EINVAL, "bad argument");
    const Problem& P = B->probs[p];
    const int64_t n = B->D.n;
    DBuf da, dg;
    TRY(da.alloc(sizeof(double) * n));
    TRY(dg.alloc(sizeof(float) * n));
    CK(lay_pack_state(P.alpha.as<double>(), P.G.as<float>(), n, B->D.n_pad, 1, da.as<double>(),
                      dg.as<float>(), B->st));
    if (alpha) CK(cudaMemcpyAsync(alpha, da.p, sizeof(double) * n,
                                  is_device_ptr(alpha) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, B->st));
    if (G) CK(cudaMemcpyAsync(G, dg.p, sizeof(float) * n,
                              is_device_ptr(G) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, B->st));
    CK(cudaStreamSynchronize(B->st));
    return SVM_OK;
}

extern "C" int svm_batch_run(svm_batch* B, int64_t max_iter, int64_t* iterations)
{
    if (!B || max_iter < 1) return fail(SVM_EINVAL, "NULL batch or max_iter < 1");
    for (size_t p = 0; p < B->probs.size(); ++p) B->probs[p].max_iter = max_iter;
    bool handled = false;
    TRY(solve_batched(B->D, B->probs, &B->prm, B->st, &handled));
    if (!handled) return fail(SVM_EINVAL, "configuration not covered by the batched pass");
    if (iterations)
        for (size_t p = 0; p < B->probs.size(); ++p) iterations[p] = B->probs[p].iterations;   // (this run's)
    return SVM_OK;
}

extern "C" void svm_batch_free(svm_batch* B) { delete B; }

// ================================================================ solver-state API
struct svm_solver {
    Data D;
    Problem P;
    Exchange E;
    svm_params prm;
    cudaStream_t st = nullptr;
    int vranks = 1;   // svm_solver_set_ranks
};

static int solver_create_common(svm_solver* S, const float* y, const svm_params* params)
{
    std::vector<float> yh;
    TRY(to_host(yh, y, S->D.n, S->st));
    std::vector<std::vector<float>> ys;
    std::vector<double> labels;
    int mode = 0;
    double first = 0;
    TRY(label_problems(params, yh, ys, labels, &mode, &first));
    if (mode == 2) return fail(SVM_EINVAL, "solver API takes binary or regression problems only");
    TRY(S->E.alloc(S->D.nblk));
    TRY(problem_init(S->P, S->D, ys[0].data(), params, S->st));
    CK(cudaStreamSynchronize(S->st));
    return SVM_OK;
}

extern "C" int svm_solver_create(const float* X, const float* y, int64_t n, int64_t d,
                                 const svm_params* params, svm_solver** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    TRY(check_params(params, n, d));
    if (!X || !y) return fail(SVM_EINVAL, "X or y is NULL");
    svm_solver* S = new (std::nothrow) svm_solver();
    if (!S) return fail(SVM_ENOMEM, "solver allocation failed");
    S->prm = *params;
    S->st = (cudaStream_t)params->stream;
    int rc = build_dense(S->D, X, n, d, params->layout, pick_nblk(n), S->st);
    if (rc == SVM_OK) rc = own_inputs(S->D, S->st);
    if (rc == SVM_OK) rc = solver_create_common(S, y, params);
    if (rc != SVM_OK) { delete S; return rc; }
    *out = S;
    return SVM_OK;
}

extern "C" int svm_solver_create_csr(const int64_t* indptr, const int32_t* indices,
                                     const float* data, const float* y, int64_t n, int64_t d,
                                     const svm_params* params, svm_solver** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    TRY(check_params(params, n, d));
    if (!y) return fail(SVM_EINVAL, "y is NULL");
    svm_solver* S = new (std::nothrow) svm_solver();
    if (!S) return fail(SVM_ENOMEM, "solver allocation failed");
    S->prm = *params;
    S->st = (cudaStream_t)params->stream;
    int rc = build_csr(S->D, indptr, indices, data, n, d, pick_nblk(n), S->st);
    if (rc == SVM_OK) rc = own_inputs(S->D, S->st);
    if (rc == SVM_OK) rc = solver_create_common(S, y, params);
    if (rc != SVM_OK) { delete S; return rc; }
    *out = S;
    return SVM_OK;
}

extern "C" int svm_solver_size(const svm_solver* s, int64_t* m)
{
    if (!s || !m) return fail(SVM_EINVAL, "NULL solver or m");
    *m = s->D.n * s->P.ncopy;
    return SVM_OK;
}

extern "C" int svm_solver_set_state(svm_solver* s, const double* alpha, const float* G)
{
    if (!s || !alpha || !G) return fail(SVM_EINVAL, "NULL argument");
    int64_t m = s->D.n * s->P.ncopy;
    std::vector<double> ah;
    TRY(to_host(ah, alpha, m, s->st));
    for (int64_t i = 0; i < m; ++i)
        if (!(ah[i] >= 0.0 && ah[i] <= s->P.C))
            return fail(SVM_EINVAL, "alpha[%lld] = %g outside [0, C]", (long long)i, ah[i]);
    DBuf da, dg;
    TRY(to_device(da, alpha, m, s->st));
    TRY(to_device(dg, G, m, s->st));
    CK(lay_unpack_state(da.as<double>(), dg.as<float>(), s->D.n, s->D.n_pad, s->P.ncopy,
                        s->P.alpha.as<double>(), s->P.G.as<float>(), s->st));
    CK(lay_status_from_alpha(s->P.alpha.as<double>(), s->D.n, s->D.n_pad, s->P.ncopy, s->P.C,
                             s->P.status.as<uint8_t>(), s->st));
    CK(cudaStreamSynchronize(s->st));
    return SVM_OK;
}

extern "C" int svm_solver_get_state(const svm_solver* s, double* alpha, float* G)
{
    if (!s) return fail(SVM_EINVAL, "NULL solver");
    int64_t m = s->D.n * s->P.ncopy;
    DBuf da, dg;
    TRY(da.alloc(sizeof(double) * m));
    TRY(dg.alloc(sizeof(float) * m));
    CK(lay_pack_state(s->P.alpha.as<double>(), s->P.G.as<float>(), s->D.n, s->D.n_pad, s->P.ncopy,
                      da.as<double>(), dg.as<float>(), s->st));
    if (alpha) CK(cudaMemcpyAsync(alpha, da.p, sizeof(double) * m,
                                  is_device_ptr(alpha) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->st));
    if (G) CK(cudaMemcpyAsync(G, dg.p, sizeof(float) * m,
                              is_device_ptr(G) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return SVM_OK;
}

extern "C" int svm_solver_run(svm_solver* s, int64_t max_iter, svm_solver_stats* stats)
{
    if (!s) return fail(SVM_EINVAL, "NULL solver");
    if (max_iter < 0) return fail(SVM_EINVAL, "max_iter < 0");
    s->P.loop_ms = 0;
    int64_t before = s->P.iterations;
    SmoInfo info;
    LoopMode mode;
    mode.vranks = s->vranks;
    TRY(run_loop(s->D, s->P, s->E, max_iter, s->st, &info, nullptr, &mode));
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->iterations = s->P.iterations - before;
        stats->m_up = info.m_up;
        stats->M_low = info.M_low;
        stats->converged = info.converged;
        stats->last_nw = info.iterations > 0 ? info.last_nw : 0;
        for (int i = 0; i < stats->last_nw; ++i) {
            stats->last_w[i] = info.last_w[i];
            stats->last_dalpha[i] = info.last_dalpha[i];
        }
        stats->last_inner = info.last_inner;
        stats->loop_ms = s->P.loop_ms;
        stats->cache_passes = info.cache_allhit;
    }
    return SVM_OK;
}

extern "C" int svm_solver_kernel_rows(svm_solver* s, const int64_t* rows, int32_t nr, float* K)
{
    if (!s || !rows || !K) return fail(SVM_EINVAL, "NULL argument");
    if (nr < 1 || nr > SVM_WS) return fail(SVM_EINVAL, "nr must be in [1, 16]");
    std::vector<int64_t> rh;
    TRY(to_host(rh, rows, nr, s->st));
    for (int i = 0; i < nr; ++i)
        if (rh[i] < 0 || rh[i] >= s->D.n) return fail(SVM_EINVAL, "row index out of range");
    DBuf drows, dK;
    TRY(to_device(drows, rh.data(), nr, s->st));
    TRY(dK.alloc(sizeof(float) * s->D.n * nr));
    SmoArgs a = make_args(s->D, s->P, s->E);
    CK(launch_kernel_rows(a, drows.as<int64_t>(), nr, dK.as<float>(), s->st));
    CK(cudaMemcpyAsync(K, dK.p, sizeof(float) * s->D.n * nr,
                       is_device_ptr(K) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return SVM_OK;
}

extern "C" int svm_solver_set_ranks(svm_solver* s, int32_t vranks)
{
    if (!s) return fail(SVM_EINVAL, "NULL solver");
    if (vranks < 1 || vranks > SVM_MAX_RANKS || (vranks > 1 && s->D.nblk % vranks != 0))
        return fail(SVM_EINVAL, "vranks = %d must be in [1, %d] and divide the %d CTAs", vranks,
                    SVM_MAX_RANKS, s->D.nblk);
    s->vranks = vranks;
    return SVM_OK;
}

extern "C" int svm_solver_geometry(const svm_solver* s, int32_t* nblk, int64_t* rows_per_cta)
{
    if (!s) return fail(SVM_EINVAL, "NULL solver");
    if (nblk) *nblk = s->D.nblk;
    if (rows_per_cta) *rows_per_cta = s->D.rows_per_cta;
    return SVM_OK;
}

extern "C" int svm_solver_pass_bench(svm_solver* s, const int64_t* rows, int32_t nr,
                                     const float* coef, int64_t passes, double* ms)
{
    if (!s || !rows || !coef || !ms) return fail(SVM_EINVAL, "NULL argument");
    if (nr < 1 || nr > SVM_WS) return fail(SVM_EINVAL, "nr must be in [1, 16]");
    if (passes < 1) return fail(SVM_EINVAL, "passes must be >= 1");
    std::vector<int64_t> rh;
    std::vector<float> ch;
    TRY(to_host(rh, rows, nr, s->st));
    TRY(to_host(ch, coef, nr, s->st));
    for (int i = 0; i < nr; ++i) {
        if (rh[i] < 0 || rh[i] >= s->D.n) return fail(SVM_EINVAL, "row index out of range");
        for (int j = 0; j < i; ++j)
            if (rh[j] == rh[i]) return fail(SVM_EINVAL, "rows must be distinct");
    }
    DBuf drows, dc;
    TRY(to_device(drows, rh.data(), nr, s->st));
    TRY(to_device(dc, ch.data(), nr, s->st));
    LoopMode mode;
    mode.pass_rows = drows.as<int64_t>();
    mode.pass_c = dc.as<float>();
    mode.pass_nr = nr;
    mode.pass_ms = ms;
    SmoInfo info;
    return run_loop(s->D, s->P, s->E, passes, s->st, &info, nullptr, &mode);
}

extern "C" void svm_solver_free(svm_solver* s) { delete s; }

// ================================================================ row-sharded training
// Rank r owns rows [row0, row0 + n_local).  Exported (cudaIpc) buffers per rank: the candidate
// receive buffers (keys, payloads, flags), the scalar exchange buffer, its rows (dense row-major
// or CSR) and norms, and the per-row coefficient / SV-index export used to gather the model.
namespace {
constexpr uint32_t SHARD_MAGIC = 0x53564D42u;  // "SVMB"
enum { H_XW, H_XBUF, H_XFLAGS, H_XR, H_NORMS, H_INDPTR, H_INDICES, H_VALS, H_SVIDX, H_COEFX,
       H_COUNT };
struct ShardHandle {
    uint32_t magic;
    int32_t rank, world, nblk, csr, nprob, ncopy, pad;
    int64_t n_local, row0, n_global, d, rows_per_cta;
    cudaIpcMemHandle_t h[H_COUNT];
};
static_assert(sizeof(ShardHandle) <= SVM_SHARD_HANDLE_BYTES, "shard handle too large");
}  // namespace

struct svm_shard {
    Data D;
    svm_params prm;
    cudaStream_t st = nullptr;
    int rank = 0, world = 1;
    int64_t row0 = 0, n_global = 0;
    std::vector<std::vector<float>> ys;  // per problem, local rows
    std::vector<double> labels;
    int mode = 0, nprob = 1;
    double first = 0;
    Exchange E;
    DBuf xbuf, xflags, xvals, xout, xerr, svidx, coefx;
    uint32_t xepoch = 0;
    ShardCtx sc;
    XchgPeers xp;
    SvPeers svp;
    std::vector<void*> opened;
    bool connected = false;
    ~svm_shard()
    {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
    }
};

// device-side all-gather of K doubles across ranks (also a barrier)
static int shard_xchg(svm_shard* S, const std::vector<double>& vals, std::vector<double>& all,
                      double timeout_s = 60.0)
{
    int K = (int)vals.size();
    CK(cudaMemcpyAsync(S->xvals.p, vals.data(), sizeof(double) * K, cudaMemcpyHostToDevice, S->st));
    CK(cudaMemsetAsync(S->xerr.p, 0, sizeof(int), S->st));
    uint32_t tag = ++S->xepoch;
    CK(lay_xchg(S->xvals.as<double>(), K, S->rank, S->world, S->xp, tag, S->xout.as<double>(),
                (uint64_t)(timeout_s * 1e9), S->xerr.as<int>(), S->st));
    all.resize((size_t)S->world * K);
    int err = 0;
    CK(cudaMemcpyAsync(all.data(), S->xout.p, sizeof(double) * S->world * K, cudaMemcpyDeviceToHost, S->st));
    CK(cudaMemcpyAsync(&err, S->xerr.p, sizeof(int), cudaMemcpyDeviceToHost, S->st));
    CK(cudaStreamSynchronize(S->st));
    if (err) return fail(SVM_ETIMEOUT, "rank exchange timed out (a peer stopped)");
    return SVM_OK;
}

static int shard_create_common(svm_shard* S, const float* y_global, const svm_params* params)
{
    std::vector<float> yg;
    TRY(to_host(yg, y_global, S->n_global, S->st));
    std::vector<std::vector<float>> ys;
    TRY(label_problems(params, yg, ys, S->labels, &S->mode, &S->first));
    S->nprob = (int)ys.size();
    S->ys.resize(ys.size());
    for (size_t p = 0; p < ys.size(); ++p)
        S->ys[p].assign(ys[p].begin() + S->row0, ys[p].begin() + S->row0 + S->D.n);
    TRY(S->E.alloc(S->D.nblk));   // local level: this rank's CTAs; rank level: <= SVM_MAX_RANKS
    TRY(S->xbuf.alloc(sizeof(double) * 2 * S->world * XCH_K));
    TRY(S->xflags.alloc(sizeof(uint32_t) * S->world));
    CK(cudaMemset(S->xflags.p, 0, S->xflags.bytes));
    TRY(S->xvals.alloc(sizeof(double) * XCH_K));
    TRY(S->xout.alloc(sizeof(double) * S->world * XCH_K));
    TRY(S->xerr.alloc(sizeof(int)));
    TRY(S->svidx.alloc(sizeof(int64_t) * std::max<int64_t>(S->D.n, 1)));
    TRY(S->coefx.alloc(sizeof(double) * std::max<int64_t>(S->D.n, 1) * S->nprob));
    if (!S->D.csr && !S->D.XR_own.p) {  // exported rows must be a cudaMalloc base: own a copy
        TRY(S->D.XR_own.alloc(sizeof(float) * S->D.n * S->D.d));
        CK(cudaMemcpyAsync(S->D.XR_own.p, S->D.XR, sizeof(float) * S->D.n * S->D.d,
                           cudaMemcpyDeviceToDevice, S->st));
        S->D.XR = S->D.XR_own.as<float>();
    }
    if (S->D.csr) {
        if (!S->D.indptr_own.p) { TRY(to_device(S->D.indptr_own, S->D.indptr, S->D.n + 1, S->st)); S->D.indptr = S->D.indptr_own.as<int64_t>(); }
        if (!S->D.indices_own.p) { TRY(to_device(S->D.indices_own, S->D.indices, S->D.nnz, S->st)); S->D.indices = S->D.indices_own.as<int32_t>(); }
        if (!S->D.vals_own.p) { TRY(to_device(S->D.vals_own, S->D.vals, S->D.nnz, S->st)); S->D.vals = S->D.vals_own.as<float>(); }
    }
    CK(cudaStreamSynchronize(S->st));
    // everything a peer maps must be a cudaMalloc base (IPC cannot export pool memory)
    DBuf* exported[] = {&S->E.xw, &S->xbuf, &S->xflags, &S->D.XR_own, &S->D.norms,
                        &S->D.indptr_own, &S->D.indices_own, &S->D.vals_own, &S->svidx, &S->coefx};
    for (DBuf* b : exported) TRY(b->make_plain());
    if (!S->D.csr) S->D.XR = S->D.XR_own.as<float>();
    else {
        S->D.indptr = S->D.indptr_own.as<int64_t>();
        S->D.indices = S->D.indices_own.as<int32_t>();
        S->D.vals = S->D.vals_own.as<float>();
    }
    return SVM_OK;
}

static int shard_check_args(int64_t n_local, int64_t row0, int64_t n_global, int32_t rank,
                            int32_t world)
{
    if (world < 1 || world > SVM_MAX_RANKS) return fail(SVM_EINVAL, "world must be in [1, 8]");
    if (rank < 0 || rank >= world) return fail(SVM_EINVAL, "rank out of range");
    if (n_local < 1 || row0 < 0 || row0 + n_local > n_global)
        return fail(SVM_EINVAL, "local rows [row0, row0 + n_local) outside [0, n_global)");
    return SVM_OK;
}

extern "C" int svm_shard_create(const float* X_local, int64_t n_local, int64_t d, int64_t row0,
                                const float* y_global, int64_t n_global, int32_t rank,
                                int32_t world, const svm_params* params, svm_shard** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    TRY(check_params(params, n_global, d));
    TRY(shard_check_args(n_local, row0, n_global, rank, world));
    if (!X_local || !y_global) return fail(SVM_EINVAL, "X_local or y_global is NULL");
    svm_shard* S = new (std::nothrow) svm_shard();
    if (!S) return fail(SVM_ENOMEM, "shard allocation failed");
    S->prm = *params;
    S->st = (cudaStream_t)params->stream;
    S->rank = rank;
    S->world = world;
    S->row0 = row0;
    S->n_global = n_global;
    int nblk = pick_nblk((n_global + world - 1) / world);
    int rc = build_dense(S->D, X_local, n_local, d, params->layout, nblk, S->st);
    if (rc == SVM_OK) rc = shard_create_common(S, y_global, params);
    if (rc != SVM_OK) { delete S; return rc; }
    *out = S;
    return SVM_OK;
}

extern "C" int svm_shard_create_csr(const int64_t* indptr, const int32_t* indices,
                                    const float* data, int64_t n_local, int64_t d, int64_t row0,
                                    const float* y_global, int64_t n_global, int32_t rank,
                                    int32_t world, const svm_params* params, svm_shard** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    TRY(check_params(params, n_global, d));
    TRY(shard_check_args(n_local, row0, n_global, rank, world));
    if (!y_global) return fail(SVM_EINVAL, "y_global is NULL");
    svm_shard* S = new (std::nothrow) svm_shard();
    if (!S) return fail(SVM_ENOMEM, "shard allocation failed");
    S->prm = *params;
    S->st = (cudaStream_t)params->stream;
    S->rank = rank;
    S->world = world;
    S->row0 = row0;
    S->n_global = n_global;
    int nblk = pick_nblk((n_global + world - 1) / world);
    int rc = build_csr(S->D, indptr, indices, data, n_local, d, nblk, S->st);
    if (rc == SVM_OK) rc = shard_create_common(S, y_global, params);
    if (rc != SVM_OK) { delete S; return rc; }
    *out = S;
    return SVM_OK;
}

extern "C" int svm_shard_handle(const svm_shard* S, void* handle)
{
    if (!S || !handle) return fail(SVM_EINVAL, "NULL argument");
    ShardHandle H;
    memset(&H, 0, sizeof H);
    H.magic = SHARD_MAGIC;
    H.rank = S->rank;
    H.world = S->world;
    H.nblk = S->D.nblk;
    H.csr = S->D.csr ? 1 : 0;
    H.nprob = S->nprob;
    H.ncopy = S->prm.type == SVM_EPS_REGRESSION ? 2 : 1;
    H.n_local = S->D.n;
    H.row0 = S->row0;
    H.n_global = S->n_global;
    H.d = S->D.d;
    H.rows_per_cta = S->D.rows_per_cta;
    const void* ptrs[H_COUNT] = {S->E.xw.p, S->xbuf.p, S->xflags.p,
                                 S->D.csr ? nullptr : S->D.XR, S->D.norms.p,
                                 S->D.csr ? S->D.indptr : nullptr, S->D.csr ? S->D.indices : nullptr,
                                 S->D.csr ? S->D.vals : nullptr, S->svidx.p, S->coefx.p};
    for (int i = 0; i < H_COUNT; ++i)
        if (ptrs[i]) CK(cudaIpcGetMemHandle(&H.h[i], const_cast<void*>(ptrs[i])));
    memset(handle, 0, SVM_SHARD_HANDLE_BYTES);
    memcpy(handle, &H, sizeof H);
    return SVM_OK;
}

extern "C" int svm_shard_connect(svm_shard* S, const void* all_handles)
{
    if (!S || !all_handles) return fail(SVM_EINVAL, "NULL argument");
    if (S->connected) return fail(SVM_EINVAL, "shard already connected");
    const unsigned char* base = static_cast<const unsigned char*>(all_handles);
    ShardCtx& c = S->sc;
    c.rank = S->rank;
    c.world = S->world;
    c.row0 = S->row0;
    c.n_global = S->n_global;
    memset(&S->xp, 0, sizeof S->xp);
    memset(&S->svp, 0, sizeof S->svp);
    S->svp.world = S->world;
    int64_t expect_row0 = 0;
    for (int r = 0; r < S->world; ++r) {
        ShardHandle H;
        memcpy(&H, base + (size_t)r * SVM_SHARD_HANDLE_BYTES, sizeof H);
        if (H.magic != SHARD_MAGIC || H.rank != r || H.world != S->world || H.nblk != S->D.nblk ||
            H.csr != (S->D.csr ? 1 : 0) || H.nprob != S->nprob || H.n_global != S->n_global ||
            H.d != S->D.d)
            return fail(SVM_EPEER, "shard handle of rank %d does not match this run", r);
        if (H.row0 != expect_row0)
            return fail(SVM_EPEER, "ranks must hold contiguous row blocks in rank order");
        expect_row0 += H.n_local;
        c.rank_row0[r] = H.row0;
        S->svp.n_local[r] = H.n_local;
        S->svp.row0[r] = H.row0;
        void* p[H_COUNT] = {};
        if (r == S->rank) {
            void* mine[H_COUNT] = {S->E.xw.p, S->xbuf.p, S->xflags.p,
                                   S->D.csr ? nullptr : (void*)S->D.XR, S->D.norms.p,
                                   S->D.csr ? (void*)S->D.indptr : nullptr,
                                   S->D.csr ? (void*)S->D.indices : nullptr,
                                   S->D.csr ? (void*)S->D.vals : nullptr, S->svidx.p, S->coefx.p};
            memcpy(p, mine, sizeof p);
        } else {
            for (int i = 0; i < H_COUNT; ++i) {
                bool present = false;
                for (size_t b = 0; b < sizeof(cudaIpcMemHandle_t); ++b)
                    present |= H.h[i].reserved[b] != 0;
                if (!present) continue;
                cudaError_t e = cudaIpcOpenMemHandle(&p[i], H.h[i], cudaIpcMemLazyEnablePeerAccess);
                if (e != cudaSuccess)
                    return fail(SVM_EPEER, "cudaIpcOpenMemHandle(rank %d, buffer %d): %s", r, i,
                                cudaGetErrorString(e));
                S->opened.push_back(p[i]);
            }
        }
        c.xw[r] = (uint64_t*)p[H_XW];
        c.rpc[r] = H.rows_per_cta;
        c.XR[r] = (const float*)p[H_XR];
        c.norms[r] = (const float*)p[H_NORMS];
        c.indptr[r] = (const int64_t*)p[H_INDPTR];
        c.indices[r] = (const int32_t*)p[H_INDICES];
        c.vals[r] = (const float*)p[H_VALS];
        S->xp.buf[r] = (double*)p[H_XBUF];
        S->xp.flags[r] = (uint32_t*)p[H_XFLAGS];
        S->svp.XR[r] = c.XR[r];
        S->svp.indptr[r] = c.indptr[r];
        S->svp.indices[r] = c.indices[r];
        S->svp.vals[r] = c.vals[r];
        S->svp.norms[r] = c.norms[r];
        S->svp.svidx[r] = (const int64_t*)p[H_SVIDX];
        S->svp.coefx[r] = (const double*)p[H_COEFX];
    }
    if (expect_row0 != S->n_global) return fail(SVM_EPEER, "row blocks do not cover n_global");
    c.rank_row0[S->world] = S->n_global;
    S->connected = true;
    return SVM_OK;
}

// Global SV set of the per-row coefficients currently in every rank's coefx export (problems
// [0, nprob_used)): compaction locally, counts exchanged, rows gathered from their owners.
static int shard_global_sv(svm_shard* S, int nprob_used, const DBuf& flag, DBuf& SVT, DBuf& svn,
                           DBuf& coef, int64_t* nsv_out, int64_t* nsv_pad_out, DBuf* grow)
{
    const Data& D = S->D;
    DBuf idx;
    int64_t nloc = 0;
    TRY(compact(flag, D.n, idx, &nloc, S->st));
    if (nloc) CK(cudaMemcpyAsync(S->svidx.p, idx.p, sizeof(int64_t) * nloc, cudaMemcpyDeviceToDevice, S->st));
    CK(cudaStreamSynchronize(S->st));
    std::vector<double> all;
    TRY(shard_xchg(S, {(double)nloc}, all));       // also: every export is complete
    S->svp.off[0] = 0;
    for (int r = 0; r < S->world; ++r) S->svp.off[r + 1] = S->svp.off[r] + (int64_t)all[r];
    int64_t nsv = S->svp.off[S->world];
    int64_t nsv_pad = std::max<int64_t>(64, (nsv + 63) / 64 * 64);
    TRY(SVT.alloc(sizeof(float) * D.d * nsv_pad));
    TRY(svn.alloc(sizeof(float) * nsv_pad));
    TRY(coef.alloc(sizeof(double) * nsv_pad * nprob_used));
    if (D.csr) CK(cudaMemsetAsync(SVT.p, 0, SVT.bytes, S->st));
    if (grow) TRY(grow->alloc(sizeof(int64_t) * nsv_pad));
    CK(lay_gather_global_sv(S->svp, nsv, nsv_pad, D.d, nprob_used, SVT.as<float>(), svn.as<float>(),
                            coef.as<double>(), grow ? grow->as<int64_t>() : nullptr, S->st));
    CK(cudaStreamSynchronize(S->st));
    std::vector<double> none;
    TRY(shard_xchg(S, {0.0}, none));               // nobody rewrites exports before all gathered
    *nsv_out = nsv;
    *nsv_pad_out = nsv_pad;
    return SVM_OK;
}

static int shard_reduce(svm_shard* S, const Problem& P, Reduced* g)
{
    Reduced r;
    TRY(reduce_state(S->D, P, &r, S->st));
    std::vector<double> all;
    TRY(shard_xchg(S, {r.m_up, r.M_low, r.free_sum, r.free_cnt, r.dual}, all));
    Reduced t = {-INFINITY, INFINITY, 0, 0, 0};
    for (int k = 0; k < S->world; ++k) {  // fixed rank order: identical on every rank
        t.m_up = std::max(t.m_up, all[k * 5 + 0]);
        t.M_low = std::min(t.M_low, all[k * 5 + 1]);
        t.free_sum += all[k * 5 + 2];
        t.free_cnt += all[k * 5 + 3];
        t.dual += all[k * 5 + 4];
    }
    *g = t;
    return SVM_OK;
}

// As certify(): the global SVs (every rank's, over NVLink) against this rank's rows; with a valid
// CertState only the rows (of every rank) whose coefficient changed since the previous
// certification enter, with their coefficient change.
static int shard_certify(svm_shard* S, Problem& P, double* viol, CertState* cs = nullptr)
{
    double t0 = now_ms();
    const Data& D = S->D;
    DBuf flag, coefrow, SVT, svn, coef, F, dcoef;
    TRY(flag.alloc(D.n));
    CK(cudaMemsetAsync(flag.p, 0, D.n, S->st));
    TRY(problem_coef(D, P, coefrow, flag, S->st));
    const bool delta = cs && cs->valid && !getenv("SVMB200_FULL_RECERT");
    if (delta) {
        TRY(dcoef.alloc(sizeof(double) * D.n));
        CK(lay_coef_delta(coefrow.as<double>(), cs->coef.as<double>(), D.n, dcoef.as<double>(),
                          flag.as<uint8_t>(), S->st));
    }
    CK(cudaMemcpyAsync(S->coefx.p, delta ? dcoef.p : coefrow.p, sizeof(double) * D.n,
                       cudaMemcpyDeviceToDevice, S->st));
    int64_t nsv = 0, nsv_pad = 0;   // global count: the same decision on every rank
    TRY(shard_global_sv(S, 1, flag, SVT, svn, coef, &nsv, &nsv_pad, nullptr));
    if (nsv > 0 || !delta) TRY(training_decision(D, SVT, svn, nsv, nsv_pad, coef, P.kp, F, S->st));
    if (delta) {
        if (nsv > 0) CK(lay_add_f64(cs->F.as<double>(), F.as<double>(), D.n, S->st));
    } else if (cs) {
        std::swap(cs->F.p, F.p);
        std::swap(cs->F.bytes, F.bytes);
        std::swap(cs->F.plain, F.plain);
        std::swap(cs->coef.p, coefrow.p);
        std::swap(cs->coef.bytes, coefrow.bytes);
        std::swap(cs->coef.plain, coefrow.plain);
        cs->valid = true;
    }
    CK(pred_refresh_G(cs ? cs->F.as<double>() : F.as<double>(), P.yv.as<float>(),
                      P.status.as<uint8_t>(), D.n, D.n_pad, P.ncopy, P.eps, P.G.as<float>(), S->st));
    Reduced g;
    TRY(shard_reduce(S, P, &g));
    P.m_up = g.m_up;
    P.M_low = g.M_low;
    *viol = g.m_up - g.M_low;
    P.certified = true;
    P.cert_ms += now_ms() - t0;
    ++P.n_cert;
    return SVM_OK;
}

extern "C" int svm_shard_train(svm_shard* S, svm_model** out)
{
    if (!out) return fail(SVM_EINVAL, "out is NULL");
    *out = nullptr;
    if (!S) return fail(SVM_EINVAL, "shard is NULL");
    if (!S->connected) return fail(SVM_EINVAL, "svm_shard_connect has not been called");
    double t_start = now_ms();
    const Data& D = S->D;
    const svm_params* prm = &S->prm;
    std::vector<double> none;
    TRY(shard_xchg(S, {0.0}, none, 300.0));        // start barrier
    std::vector<Problem> probs(S->nprob);
    std::vector<double> bs(S->nprob);
    int32_t n_cert = 0;
    double dual = 0, worst = -INFINITY, loop_ms = 0, cert_ms = 0, exch_ms = 0;
    double xh[SMO_EXCH_BINS] = {}, upc = 0;
    int64_t cache_passes = 0;
    int64_t iters = 0;
    bool conv = true, cert = true;
    for (int p = 0; p < S->nprob; ++p) {
        Problem& P = probs[p];
        TRY(problem_init(P, D, S->ys[p].data(), prm, S->st));
        P.max_iter = prm->max_iter > 0 ? prm->max_iter
                                       : std::max<int64_t>(10 * S->n_global * P.ncopy, 10000);
        TRY(run_loop(D, P, S->E, P.max_iter, S->st, nullptr, &S->sc));
        CertState cs;
        for (int round = 0; P.converged && prm->certify != 0; ++round) {
            if (prm->certify < 0 && round == 0) {   // auto rule of svm_train, on the global SV count
                DBuf cf, fl, ix;
                TRY(fl.alloc(D.n));
                CK(cudaMemsetAsync(fl.p, 0, D.n, S->st));
                TRY(problem_coef(D, P, cf, fl, S->st));
                int64_t nloc = 0;
                TRY(compact(fl, D.n, ix, &nloc, S->st));
                std::vector<double> all;
                TRY(shard_xchg(S, {(double)nloc}, all));
                double nsv_g = 0;
                for (double v : all) nsv_g += v;
                if (!want_certify(prm, S->n_global, (int64_t)nsv_g, D.d)) break;
            }
            double viol = 0;
            TRY(shard_certify(S, P, &viol, &cs));
            const double target = SVM_CERT_MARGIN * P.tol;
            if (viol <= target) { P.converged = true; break; }
            P.converged = viol <= P.tol;
            if (round == SVM_MAX_RESUMES) break;
            P.tol_loop = std::min(P.tol_loop - 0.01 * P.tol, target - resume_factor() * (viol - target));
            int64_t left = P.max_iter - P.iterations;
            if (left <= 0) break;
            TRY(run_loop(D, P, S->E, left, S->st, nullptr, &S->sc));
        }
        Reduced g;
        TRY(shard_reduce(S, P, &g));
        bs[p] = g.free_cnt > 0 ? g.free_sum / g.free_cnt : 0.5 * (g.m_up + g.M_low);
        if (!std::isfinite(bs[p])) bs[p] = 0.0;
        dual += g.dual;
        worst = std::max(worst, g.m_up - g.M_low);
        iters += P.iterations;
        conv = conv && P.converged;
        cert = cert && P.certified;
        loop_ms += P.loop_ms;
        exch_ms += P.exch_ms;
        cache_passes += P.cache_allhit;
        for (int b = 0; b < SMO_EXCH_BINS; ++b) xh[b] += P.exch_hist[b];
        if (P.us_per_cycle > 0) upc = P.us_per_cycle;
        n_cert += P.n_cert;
        cert_ms += P.cert_ms;
    }
    // model: union of SVs over problems, coefficients of every problem, rows gathered
    DBuf flag;
    TRY(flag.alloc(D.n));
    CK(cudaMemsetAsync(flag.p, 0, D.n, S->st));
    for (int p = 0; p < S->nprob; ++p) {
        DBuf coefrow;
        TRY(problem_coef(D, probs[p], coefrow, flag, S->st));
        CK(cudaMemcpyAsync(S->coefx.as<double>() + (int64_t)p * D.n, coefrow.p, sizeof(double) * D.n,
                           cudaMemcpyDeviceToDevice, S->st));
    }
    svm_model* M = new (std::nothrow) svm_model();
    if (!M) return fail(SVM_ENOMEM, "model allocation failed");
    DBuf grow;
    int64_t nsv = 0, nsv_pad = 0;
    int rc = shard_global_sv(S, S->nprob, flag, M->SVT, M->svnorm, M->coef, &nsv, &nsv_pad, &grow);
    if (rc != SVM_OK) { delete M; return rc; }
    M->nsv = nsv;
    M->nsv_pad = nsv_pad;
    M->d = D.d;
    M->mode = S->mode;
    M->n_out = S->nprob;
    rc = build_sv_tiles(M, S->st);
    if (rc != SVM_OK) { delete M; return rc; }
    M->kp = probs[0].kp;
    M->first_label = S->first;
    rc = to_device(M->b, bs.data(), S->nprob, S->st);
    std::vector<double> lab = S->labels;
    if (lab.empty()) lab.push_back(0.0);
    if (rc == SVM_OK) rc = to_device(M->labels, lab.data(), (int64_t)lab.size(), S->st);
    if (rc != SVM_OK) { delete M; return rc; }
    M->sv_index.resize(nsv);
    M->coef_host.resize((size_t)nsv * S->nprob);
    if (nsv) {
        cudaMemcpyAsync(M->sv_index.data(), grow.p, sizeof(int64_t) * nsv, cudaMemcpyDeviceToHost, S->st);
        for (int p = 0; p < S->nprob; ++p)
            cudaMemcpyAsync(M->coef_host.data() + (size_t)p * nsv, M->coef.as<double>() + (int64_t)p * nsv_pad,
                            sizeof(double) * nsv, cudaMemcpyDeviceToHost, S->st);
    }
    cudaError_t e = cudaStreamSynchronize(S->st);
    if (e != cudaSuccess) { delete M; return fail(SVM_ECUDA, "%s", cudaGetErrorString(e)); }
    svm_model_info& I = M->info;
    memset(&I, 0, sizeof I);
    I.type = prm->type;
    I.kernel = prm->kernel;
    I.degree = prm->degree;
    I.gamma = M->kp.gamma64;
    I.coef0 = prm->coef0;
    I.n_features = D.d;
    I.n_train = S->n_global;
    I.n_sv = nsv;
    I.n_class = S->mode == 0 ? 0 : (int32_t)S->labels.size();
    I.n_problem = S->nprob;
    for (size_t i = 0; i < S->labels.size() && i < 64; ++i) I.labels[i] = S->labels[i];
    for (size_t i = 0; i < bs.size() && i < 64; ++i) I.b[i] = bs[i];
    I.iterations = iters;
    I.violation = worst;
    I.converged = conv ? 1 : 0;
    I.certified = cert ? 1 : 0;
    I.dual_objective = dual;
    I.loop_ms = loop_ms;
    I.exchange_ms = exch_ms;
    I.exchange_p50_us = exch_percentile(xh, 0.50) * upc;
    I.exchange_p99_us = exch_percentile(xh, 0.99) * upc;
    I.certifications = n_cert;
    I.cache_passes = cache_passes;
    I.certify_ms = cert_ms;
    I.passes = iters;
    I.pass_ms = loop_ms;
    I.train_ms = now_ms() - t_start;
    *out = M;
    return SVM_OK;
}

extern "C" void svm_shard_free(svm_shard* S) { delete S; }

// ---- one-call sharded training over an NCCL communicator (SURVEY 8(b) svm_train_sharded) -----
// NCCL is loaded on first use (dlopen of libnccl.so.2: the one the host framework already loaded
// when there is one), so the library has no link-time NCCL dependency.  The communicator carries
// the one setup exchange (the peer-mapping handles); the per-iteration exchange stays inside the
// persistent kernel over NVLink peer memory.
namespace {
struct NcclApi {
    typedef int (*GetUniqueId)(void*);
    typedef int (*CommInitRank)(void**, int, const void* /* ncclUniqueId by value, 128 B */, int);
    typedef int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t);
    typedef int (*CommDestroy)(void*);
    typedef const char* (*GetErrorString)(int);
    bool ok = false;
    GetUniqueId get_unique_id = nullptr;
    void* comm_init_rank = nullptr;   // called through a by-value 128-byte struct signature
    AllGather all_gather = nullptr;
    CommDestroy comm_destroy = nullptr;
    GetErrorString err = nullptr;
};
struct NcclId { char internal[128]; };
typedef int (*CommInitRankFn)(void**, int, NcclId, int);
const NcclApi& nccl_api()
{
    static std::once_flag once;
    static NcclApi api;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.get_unique_id = (NcclApi::GetUniqueId)dlsym(h, "ncclGetUniqueId");
        api.comm_init_rank = dlsym(h, "ncclCommInitRank");
        api.all_gather = (NcclApi::AllGather)dlsym(h, "ncclAllGather");
        api.comm_destroy = (NcclApi::CommDestroy)dlsym(h, "ncclCommDestroy");
        api.err = (NcclApi::GetErrorString)dlsym(h, "ncclGetErrorString");
        api.ok = api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy && api.err;
    });
    return api;
}
constexpr int NCCL_INT8 = 0;   // ncclDataType_t ncclInt8 / ncclChar
}  // namespace

extern "C" int svm_nccl_unique_id(void* id)
{
    if (!id) return fail(SVM_EINVAL, "id is NULL");
    const NcclApi& A = nccl_api();
    if (!A.ok) return fail(SVM_ENCCL, "libnccl.so.2 could not be loaded");
    int r = A.get_unique_id(id);
    if (r != 0) return fail(SVM_ENCCL, "ncclGetUniqueId: %s", A.err(r));
    return SVM_OK;
}

// All-gather of the SVM_SHARD_HANDLE_BYTES handle blobs over a fresh communicator, then
// connect + train; the communicator is destroyed before returning.
static int shard_run_nccl(svm_shard* S, const void* nccl_unique_id, svm_model** out)
{
    const NcclApi& A = nccl_api();
    if (!A.ok) return fail(SVM_ENCCL, "libnccl.so.2 could not be loaded");
    std::vector<char> mine(SVM_SHARD_HANDLE_BYTES), all((size_t)SVM_SHARD_HANDLE_BYTES * S->world);
    TRY(svm_shard_handle(S, mine.data()));
    NcclId id;
    memcpy(id.internal, nccl_unique_id, sizeof id.internal);
    void* comm = nullptr;
    int r = reinterpret_cast<CommInitRankFn>(A.comm_init_rank)(&comm, S->world, id, S->rank);
    if (r != 0) return fail(SVM_ENCCL, "ncclCommInitRank(rank %d of %d): %s", S->rank, S->world, A.err(r));
    DBuf dsend, drecv;
    int rc = SVM_OK;
    if ((rc = dsend.alloc(mine.size())) == SVM_OK && (rc = drecv.alloc(all.size())) == SVM_OK) {
        cudaMemcpyAsync(dsend.p, mine.data(), mine.size(), cudaMemcpyHostToDevice, S->st);
        r = A.all_gather(dsend.p, drecv.p, mine.size(), NCCL_INT8, comm, S->st);
        if (r != 0) rc = fail(SVM_ENCCL, "ncclAllGather: %s", A.err(r));
        else {
            cudaMemcpyAsync(all.data(), drecv.p, all.size(), cudaMemcpyDeviceToHost, S->st);
            if (cudaStreamSynchronize(S->st) != cudaSuccess) rc = fail(SVM_ECUDA, "handle exchange failed");
        }
    }
    A.comm_destroy(comm);
    if (rc != SVM_OK) return rc;
    TRY(svm_shard_connect(S, all.data()));
    return svm_shard_train(S, out);
}

extern "C" int svm_train_sharded(const float* X_local, int64_t n_local, int64_t d, int64_t row0,
                                 const float* y_global, int64_t n_global, int32_t rank,
                                 int32_t world, const void* nccl_unique_id,
                                 const svm_params* params, svm_model** out)
{
    if (!out || !nccl_unique_id) return fail(SVM_EINVAL, "out or nccl_unique_id is NULL");
    *out = nullptr;
    svm_shard* S = nullptr;
    TRY(svm_shard_create(X_local, n_local, d, row0, y_global, n_global, rank, world, params, &S));
    const int rc = shard_run_nccl(S, nccl_unique_id, out);
    svm_shard_free(S);
    return rc;
}

extern "C" int svm_train_sharded_csr(const int64_t* indptr, const int32_t* indices,
                                     const float* data, int64_t n_local, int64_t d, int64_t row0,
                                     const float* y_global, int64_t n_global, int32_t rank,
                                     int32_t world, const void* nccl_unique_id,
                                     const svm_params* params, svm_model** out)
{
    if (!out || !nccl_unique_id) return fail(SVM_EINVAL, "out or nccl_unique_id is NULL");
    *out = nullptr;
    svm_shard* S = nullptr;
    TRY(svm_shard_create_csr(indptr, indices, data, n_local, d, row0, y_global, n_global, rank,
                             world, params, &S));
    const int rc = shard_run_nccl(S, nccl_unique_id, out);
    svm_shard_free(S);
    return rc;
}
