/*
 * oracle/svm_oracle.c -- plain, slow, fp64 CPU oracle for the Rgtsvm working-set SMO path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path (paper_1706_05544_b200/) never
 * links, imports or calls it, and it shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n):
 *   - the dual of Eq. 2            min 1/2 a'Qa + p'a  s.t. y'a = 0, 0 <= a_i <= C
 *   - its SVC specialisation           p = -1 ("a linear term of an all-one vector")
 *   - its eps-SVR specialisation (Eq. 1)  m = 2l, y = [+1..; -1..],
 *                                             p = [eps - z; eps + z], map(i) = i mod l
 *   - the working-set loop of P:53 step by step, in the order SURVEY.md section 8(c) writes it:
 *       3. violation m_up - M_low and stop test           ("until ... converges")
 *       4. working set: |W|/2 largest s in I_up, |W|/2 smallest s in I_low
 *       5. subproblem: max-violating-pair SMO steps inside W          ("optimized based on the
 *                                                                       local gradient")
 *       6. gradient of ALL m coefficients: G_i += y_i sum_w y_w dA_w K(x_map(i), x_map(w))
 *       7. bias b (sign corrected)
 *       8. model coefficients and decision values
 *       9. dual objective diagnostic D = 1/2 a'(G + p)
 *   All arithmetic is fp64; inputs are the fp32 arrays the GPU path reads, promoted to fp64.
 *   Kernels are evaluated directly from their definitions: rbf uses sum (u_k - v_k)^2.
 *
 * Parity pins (tests/test_oracle_*.py): closed-form 2/3-point problems, XOR, constant-target SVR
 * (S:204-206), brute-force active-set QP for m <= 8, libsvm via
 * scikit-learn, finite differences and the invariants of S:172-174.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* e1071 / libsvm kernel numbering (P:77 names the four kernels; S:116 gives the formulas). */
enum { ORA_LINEAR = 0, ORA_POLY = 1, ORA_RBF = 2, ORA_SIGMOID = 3 };

typedef struct {
    int32_t kernel;
    int32_t degree;
    double gamma;
    double coef0;
} ora_kspec;

/* ---- step 2: the kernel function, directly from its definition ------------- */
double ora_kernel(const float* u, const float* v, int64_t d, const ora_kspec* ks)
{
    double s = 0.0;
    int64_t k;
    if (ks->kernel == ORA_RBF) {
        for (k = 0; k < d; ++k) {
            double t = (double)u[k] - (double)v[k];
            s += t * t;
        }
        return exp(-ks->gamma * s);
    }
    for (k = 0; k < d; ++k) s += (double)u[k] * (double)v[k];
    if (ks->kernel == ORA_LINEAR) return s;
    if (ks->kernel == ORA_POLY) {
        double base = ks->gamma * s + ks->coef0, r = 1.0;
        int32_t e;
        for (e = 0; e < ks->degree; ++e) r *= base; /* integer power by repeated product */
        return r;
    }
    return tanh(ks->gamma * s + ks->coef0); /* sigmoid */
}

/* ---- step 1: the Eq. 2 instance --------------------------------------
 * type 0 = C-classification: yz holds +-1 labels; m = n, y = yz, p = -1, map = identity.
 * type 3 = eps-regression:   yz holds z; m = 2n; positive copy (alpha*) first with y = +1,
 *                            p = eps - z; negative copy (alpha) second with y = -1, p = eps + z.
 * Returns m. */
int64_t ora_build_problem(int32_t type, const float* yz, int64_t n, double eps,
                          int8_t* y, double* p, int64_t* map)
{
    int64_t i;
    if (type == 0) {
        for (i = 0; i < n; ++i) {
            y[i] = yz[i] > 0.0f ? 1 : -1;
            p[i] = -1.0;
            map[i] = i;
        }
        return n;
    }
    for (i = 0; i < n; ++i) {
        y[i] = 1;
        p[i] = eps - (double)yz[i];
        map[i] = i;
        y[n + i] = -1;
        p[n + i] = eps + (double)yz[i];
        map[n + i] = i;
    }
    return 2 * n;
}

/* I_up / I_low of S:191. */
static int in_up(int8_t y, double a, double C) { return (y > 0 && a < C) || (y < 0 && a > 0.0); }
static int in_low(int8_t y, double a, double C) { return (y > 0 && a > 0.0) || (y < 0 && a < C); }

/* ---- step 3: maximal violation.  m_up = max_{I_up} s, M_low = min_{I_low} s with
 * s_i = -y_i G_i; -inf / +inf on empty sets. */
void ora_violation(int64_t m, const int8_t* y, const double* alpha, const double* G, double C,
                   double* m_up, double* M_low)
{
    double up = -INFINITY, low = INFINITY;
    int64_t i;
    for (i = 0; i < m; ++i) {
        double s = -(double)y[i] * G[i];
        if (in_up(y[i], alpha[i], C) && s > up) up = s;
        if (in_low(y[i], alpha[i], C) && s < low) low = s;
    }
    *m_up = up;
    *M_low = low;
}

/* "a before b" in the up list: larger s first, ties to the lower index. */
static int up_before(double sa, int64_t ia, double sb, int64_t ib)
{
    return sa > sb || (sa == sb && ia < ib);
}
/* "a before b" in the low list: smaller s first, ties to the lower index. */
static int low_before(double sa, int64_t ia, double sb, int64_t ib)
{
    return sa < sb || (sa == sb && ia < ib);
}

static int cmp_i64(const void* a, const void* b)
{
    int64_t x = *(const int64_t*)a, z = *(const int64_t*)b;
    return (x > z) - (x < z);
}

/* ---- step 4: working set ("picking 16 dual space coefficients based on which partial
 * derivatives ... are the largest, subject to dual space constraints").
 * q/2 largest s in I_up and q/2 smallest s in I_low, ordered by (s, index) with ties to the
 * lower index; the union, deduplicated without backfill, sorted ascending.  Returns |W|. */
int32_t ora_select(int64_t m, const int8_t* y, const double* alpha, const double* G, double C,
                   int32_t q, int64_t* W)
{
    int32_t half = q / 2, nu = 0, nl = 0, nw = 0, a, b;
    int64_t* ui = (int64_t*)malloc(sizeof(int64_t) * (size_t)half);
    int64_t* li = (int64_t*)malloc(sizeof(int64_t) * (size_t)half);
    double* us = (double*)malloc(sizeof(double) * (size_t)half);
    double* ls = (double*)malloc(sizeof(double) * (size_t)half);
    int64_t i;
    for (i = 0; i < m; ++i) {
        double s = -(double)y[i] * G[i];
        if (in_up(y[i], alpha[i], C)) { /* insertion into the sorted up list */
            if (nu < half || up_before(s, i, us[nu - 1], ui[nu - 1])) {
                int32_t pos = nu < half ? nu++ : half - 1;
                while (pos > 0 && up_before(s, i, us[pos - 1], ui[pos - 1])) {
                    us[pos] = us[pos - 1];
                    ui[pos] = ui[pos - 1];
                    --pos;
                }
                us[pos] = s;
                ui[pos] = i;
            }
        }
        if (in_low(y[i], alpha[i], C)) { /* insertion into the sorted low list */
            if (nl < half || low_before(s, i, ls[nl - 1], li[nl - 1])) {
                int32_t pos = nl < half ? nl++ : half - 1;
                while (pos > 0 && low_before(s, i, ls[pos - 1], li[pos - 1])) {
                    ls[pos] = ls[pos - 1];
                    li[pos] = li[pos - 1];
                    --pos;
                }
                ls[pos] = s;
                li[pos] = i;
            }
        }
    }
    for (a = 0; a < nu; ++a) W[nw++] = ui[a];
    for (b = 0; b < nl; ++b) {
        int dup = 0;
        for (a = 0; a < nu; ++a) dup |= (ui[a] == li[b]);
        if (!dup) W[nw++] = li[b];
    }
    qsort(W, (size_t)nw, sizeof(int64_t), cmp_i64);
    free(ui);
    free(li);
    free(us);
    free(ls);
    return nw;
}

/* ---- step 5: the |W|-variable subproblem ("The 16 dual space coefficients are then
 * optimized based on the local gradient"; "alpha and alpha* increments are optimized under
 * the constraints").  Alpha outside W is fixed; aW, GW are local copies updated in
 * place.  QW is |W| x |W| row-major with QW[a*nw+b] = y_a y_b K(x_map(a), x_map(b)).
 * Each step: i = argmax_{W and I_up} s, j = argmin_{W and I_low} s (ties to the lower position);
 * stop when s_i - s_j <= inner_tol; eta = max(Q_ii + Q_jj - 2 y_i y_j Q_ij, tau), tau = 1e-12
 * (S:201); t = (s_i - s_j)/eta clipped to the box; a_i += y_i t, a_j -= y_j t, with a
 * variable clipped to a bound set to exactly 0 or C; GW += Q[:,i] y_i t - Q[:,j] y_j t.
 * Returns the number of pair steps taken. */
int32_t ora_subproblem(int32_t nw, const int8_t* yW, double* aW, double* GW, const double* QW,
                       double C, double inner_tol, int32_t max_steps)
{
    const double tau = 1e-12;
    int32_t step;
    for (step = 0; step < max_steps; ++step) {
        int32_t i = -1, j = -1, a;
        double si = -INFINITY, sj = INFINITY, eta, t, lim_i, lim_j;
        for (a = 0; a < nw; ++a) {
            double s = -(double)yW[a] * GW[a];
            if (in_up(yW[a], aW[a], C) && s > si) { si = s; i = a; }
            if (in_low(yW[a], aW[a], C) && s < sj) { sj = s; j = a; }
        }
        if (i < 0 || j < 0 || si - sj <= inner_tol) break;
        eta = QW[i * nw + i] + QW[j * nw + j] - 2.0 * (double)yW[i] * (double)yW[j] * QW[i * nw + j];
        if (eta < tau) eta = tau;
        t = (si - sj) / eta;
        lim_i = yW[i] > 0 ? C - aW[i] : aW[i];
        lim_j = yW[j] > 0 ? aW[j] : C - aW[j];
        {
            int clip_i = 0, clip_j = 0;
            if (t >= lim_i) { t = lim_i; clip_i = 1; }
            if (t >= lim_j) { t = lim_j; clip_j = 1; clip_i = clip_i && (lim_i == lim_j); }
            aW[i] += (double)yW[i] * t;
            aW[j] -= (double)yW[j] * t;
            if (clip_i) aW[i] = yW[i] > 0 ? C : 0.0;
            if (clip_j) aW[j] = yW[j] > 0 ? 0.0 : C;
        }
        for (a = 0; a < nw; ++a)
            GW[a] += QW[a * nw + i] * ((double)yW[i] * t) - QW[a * nw + j] * ((double)yW[j] * t);
    }
    return step;
}

/* ---- step 6: gradient of all m coefficients ("calculating the gradient for all dual space
 * coefficients"; "the responses terms are updated"):
 *   G_i += y_i * sum_{w in W} y_w dA_w K(x_map(i), x_map(w))   for every i.
 * X is row-major n x d fp32. */
void ora_gradient_update(const float* X, int64_t d, int64_t m, const int8_t* y, const int64_t* map,
                         int32_t nw, const int64_t* W, const double* dalpha, const ora_kspec* ks,
                         double* G)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < m; ++i) {
        double acc = 0.0;
        int32_t a;
        for (a = 0; a < nw; ++a) {
            if (dalpha[a] == 0.0) continue;
            acc += (double)y[W[a]] * dalpha[a] *
                   ora_kernel(X + map[i] * d, X + map[W[a]] * d, d, ks);
        }
        G[i] += (double)y[i] * acc;
    }
}

/* ---- step 7: bias (S:231 with the sign of the no-free case corrected):
 * b = mean of s_i over free i (0 < a_i < C), else the midpoint (m_up + M_low)/2. */
double ora_bias(int64_t m, const int8_t* y, const double* alpha, const double* G, double C)
{
    double sum = 0.0, up, low;
    int64_t cnt = 0, i;
    for (i = 0; i < m; ++i) {
        if (alpha[i] > 0.0 && alpha[i] < C) {
            sum += -(double)y[i] * G[i];
            ++cnt;
        }
    }
    if (cnt > 0) return sum / (double)cnt;
    ora_violation(m, y, alpha, G, C, &up, &low);
    return 0.5 * (up + low);
}

/* ---- step 9: dual objective D = 1/2 a'(G + p) (min form, so D <= 0). */
double ora_dual_objective(int64_t m, const double* alpha, const double* G, const double* p)
{
    double s = 0.0;
    int64_t i;
    for (i = 0; i < m; ++i) s += alpha[i] * (G[i] + p[i]);
    return 0.5 * s;
}

/* ---- the loop of P:53.  alpha and G are outputs (length m); on entry they are
 * overwritten with alpha = 0, G = p.  Stops when m_up - M_low <= tol (the KKT reading of
 * "until the primal and dual objective converges") or after max_iter iterations.
 * info[0] = iterations, info[1] = m_up, info[2] = M_low, info[3] = converged (1/0),
 * info[4] = total inner pair steps.  Returns the iteration count. */
int64_t ora_train(const float* X, int64_t n, int64_t d, const ora_kspec* ks, int64_t m,
                  const int8_t* y, const double* p, const int64_t* map, double C, double tol,
                  int32_t q, int64_t max_iter, double inner_tol, int32_t inner_max,
                  double* alpha, double* G, double* info)
{
    int64_t* W = (int64_t*)malloc(sizeof(int64_t) * (size_t)q);
    int8_t* yW = (int8_t*)malloc((size_t)q);
    double* aW = (double*)malloc(sizeof(double) * (size_t)q);
    double* a0 = (double*)malloc(sizeof(double) * (size_t)q);
    double* GW = (double*)malloc(sizeof(double) * (size_t)q);
    double* dA = (double*)malloc(sizeof(double) * (size_t)q);
    double* QW = (double*)malloc(sizeof(double) * (size_t)q * (size_t)q);
    int64_t it = 0, i;
    double up = 0, low = 0, inner_total = 0;
    int converged = 0;
    (void)n;
    for (i = 0; i < m; ++i) {
        alpha[i] = 0.0;
        G[i] = p[i];
    }
    for (;;) {
        int32_t nw, a, b;
        ora_violation(m, y, alpha, G, C, &up, &low);
        if (up - low <= tol) { converged = 1; break; }
        if (it >= max_iter) break;
        nw = ora_select(m, y, alpha, G, C, q, W);
        for (a = 0; a < nw; ++a) {
            yW[a] = y[W[a]];
            aW[a] = a0[a] = alpha[W[a]];
            GW[a] = G[W[a]];
        }
        for (a = 0; a < nw; ++a)
            for (b = 0; b < nw; ++b)
                QW[a * nw + b] = (double)yW[a] * (double)yW[b] *
                                 ora_kernel(X + map[W[a]] * d, X + map[W[b]] * d, d, ks);
        inner_total += ora_subproblem(nw, yW, aW, GW, QW, C, inner_tol, inner_max);
        for (a = 0; a < nw; ++a) dA[a] = aW[a] - a0[a];
        ora_gradient_update(X, d, m, y, map, nw, W, dA, ks, G);
        for (a = 0; a < nw; ++a) alpha[W[a]] = aW[a];
        ++it;
    }
    info[0] = (double)it;
    info[1] = up;
    info[2] = low;
    info[3] = (double)converged;
    info[4] = inner_total;
    free(W); free(yW); free(aW); free(a0); free(GW); free(dA); free(QW);
    return it;
}

/* One outer iteration from a given state (steps 4-6), for one-step parity tests.
 * Writes W (ascending) and returns |W|; alpha and G are updated in place; dalpha[a] is the
 * change of alpha[W[a]].  *steps receives the inner pair-step count. */
int32_t ora_step(const float* X, int64_t d, const ora_kspec* ks, int64_t m, const int8_t* y,
                 const int64_t* map, double C, int32_t q, double inner_tol, int32_t inner_max,
                 double* alpha, double* G, int64_t* W, double* dalpha, int32_t* steps)
{
    int8_t* yW = (int8_t*)malloc((size_t)q);
    double* aW = (double*)malloc(sizeof(double) * (size_t)q);
    double* GW = (double*)malloc(sizeof(double) * (size_t)q);
    double* QW = (double*)malloc(sizeof(double) * (size_t)q * (size_t)q);
    int32_t nw = ora_select(m, y, alpha, G, C, q, W), a, b;
    for (a = 0; a < nw; ++a) {
        yW[a] = y[W[a]];
        aW[a] = alpha[W[a]];
        GW[a] = G[W[a]];
    }
    for (a = 0; a < nw; ++a)
        for (b = 0; b < nw; ++b)
            QW[a * nw + b] = (double)yW[a] * (double)yW[b] *
                             ora_kernel(X + map[W[a]] * d, X + map[W[b]] * d, d, ks);
    *steps = ora_subproblem(nw, yW, aW, GW, QW, C, inner_tol, inner_max);
    for (a = 0; a < nw; ++a) dalpha[a] = aW[a] - alpha[W[a]];
    ora_gradient_update(X, d, m, y, map, nw, W, dalpha, ks, G);
    for (a = 0; a < nw; ++a) alpha[W[a]] = aW[a];
    free(yW); free(aW); free(GW); free(QW);
    return nw;
}

/* ---- step 8: per-training-row coefficients: SVC coef_i = y_i a_i;
 * SVR beta_r = a_r - a_{r+n} (positive copy alpha* minus negative copy alpha).  Entries with
 * |coef| <= 1e-12 C are pruned to exactly 0. */
void ora_coef(int32_t type, int64_t n, const int8_t* y, const double* alpha, double C, double* coef)
{
    int64_t i;
    for (i = 0; i < n; ++i) {
        double c = type == 0 ? (double)y[i] * alpha[i] : alpha[i] - alpha[n + i];
        coef[i] = fabs(c) <= 1e-12 * C ? 0.0 : c;
    }
}

/* Decision values f(x_q) = sum_s coef_s K(sv_s, x_q) + b.  SV rows with coef == 0
 * contribute nothing and are skipped.  SV and Xq are row-major fp32. */
void ora_decision(const float* SV, int64_t nsv, int64_t d, const double* coef, double b,
                  const ora_kspec* ks, const float* Xq, int64_t nq, double* f)
{
    int64_t q;
#pragma omp parallel for schedule(static)
    for (q = 0; q < nq; ++q) {
        double acc = 0.0;
        int64_t s;
        for (s = 0; s < nsv; ++s)
            if (coef[s] != 0.0) acc += coef[s] * ora_kernel(SV + s * d, Xq + q * d, d, ks);
        f[q] = acc + b;
    }
}

/* G = Q alpha + p recomputed from scratch, for invariant checks. */
void ora_gradient_full(const float* X, int64_t d, const ora_kspec* ks, int64_t m, const int8_t* y,
                       const int64_t* map, const double* alpha, const double* p, double* G)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < m; ++i) {
        double acc = 0.0;
        int64_t j;
        for (j = 0; j < m; ++j)
            if (alpha[j] != 0.0)
                acc += (double)y[i] * (double)y[j] * alpha[j] *
                       ora_kernel(X + map[i] * d, X + map[j] * d, d, ks);
        G[i] = acc + p[i];
    }
}

int32_t ora_num_threads(void)
{
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}
