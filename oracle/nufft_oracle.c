/* TEST INFRASTRUCTURE ONLY (oracle, "port").
 *
 * Plain-C restatement of the reference's low-rank NUFFT path, used as the
 * CHECKER by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
 * It is never the thing measured or shipped: the product library
 * (paper_1701_04492_b200/libnufft_b200.so) never links or calls it.
 *
 * Every function follows the reference operation for operation (same order
 * of floating-point operations, long double where the reference uses it), so
 * that — given the same FFT backend (oracle/fft_shim.c) — the port is
 * bit-identical to the reference headers compiled unmodified (oracle/_ref);
 * tests/test_oracle.py pins that, and pins both against the reference's own
 * known answers.  Build with -ffp-contract=off (oracle/Makefile): the
 * reference relies on the FMA-exact split at transforms.hpp:60-64 and on
 * uncontracted complex products.
 *
 * Reference file:line anchors are relative to /root/reference/proj/include/nufft.
 * Error codes: 0 ok, 1 invalid_argument, 2 domain_error, 3 other. */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fftw3.h"

typedef struct {
    double re, im;
} cplx;

static _Thread_local const char* g_err = "";
const char* orc_last_error(void) { return g_err; }
#define FAIL(code, msg) \
    do {                \
        g_err = (msg);  \
        return (code);  \
    } while (0)

/* std::complex<double> products as libstdc++/__muldc3 evaluate them for
 * finite operands: (ac - bd, ad + bc), each product rounded. */
static inline cplx cmul(cplx a, cplx b) {
    cplx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}
static inline cplx cadd(cplx a, cplx b) {
    cplx r = {a.re + b.re, a.im + b.im};
    return r;
}
static inline cplx cscale(cplx a, double d) {
    cplx r = {a.re * d, a.im * d};
    return r;
}
static inline cplx cconj(cplx a) {
    cplx r = {a.re, -a.im};
    return r;
}

/* ------------------------------------------------------------------ FFT */
/* fft.hpp:46-123 — one forward/backward plan pair per size, cached. */
typedef struct {
    int n;
    fftw_plan fwd, bwd;
} fft_pair;
static fft_pair* g_fft = NULL;
static int g_fft_n = 0, g_fft_cap = 0;
static uint64_t* g_exec_counts_n = NULL; /* parallel arrays: size, count */
static uint64_t* g_exec_counts_c = NULL;
static int g_counts_len = 0, g_counts_cap = 0;
static pthread_mutex_t g_fft_mu = PTHREAD_MUTEX_INITIALIZER;

static fft_pair orc_fft_plan_for(int n) {
    pthread_mutex_lock(&g_fft_mu);
    for (int i = 0; i < g_fft_n; ++i)
        if (g_fft[i].n == n) {
            fft_pair p = g_fft[i];
            pthread_mutex_unlock(&g_fft_mu);
            return p;
        }
    if (g_fft_n == g_fft_cap) {
        g_fft_cap = g_fft_cap ? 2 * g_fft_cap : 16;
        g_fft = (fft_pair*)realloc(g_fft, sizeof(fft_pair) * g_fft_cap);
    }
    fft_pair p;
    p.n = n;
    p.fwd = fftw_plan_dft_1d(n, NULL, NULL, FFTW_FORWARD, FFTW_ESTIMATE | FFTW_UNALIGNED);
    p.bwd = fftw_plan_dft_1d(n, NULL, NULL, FFTW_BACKWARD, FFTW_ESTIMATE | FFTW_UNALIGNED);
    g_fft[g_fft_n++] = p;
    pthread_mutex_unlock(&g_fft_mu);
    return p;
}

/* fft.hpp:91-95 test hook */
static void count_exec(int n) {
    pthread_mutex_lock(&g_fft_mu);
    int i = 0;
    for (; i < g_counts_len; ++i)
        if (g_exec_counts_n[i] == (uint64_t)n) break;
    if (i == g_counts_len) {
        if (g_counts_len == g_counts_cap) {
            g_counts_cap = g_counts_cap ? 2 * g_counts_cap : 16;
            g_exec_counts_n = (uint64_t*)realloc(g_exec_counts_n, 8 * g_counts_cap);
            g_exec_counts_c = (uint64_t*)realloc(g_exec_counts_c, 8 * g_counts_cap);
        }
        g_exec_counts_n[i] = (uint64_t)n;
        g_exec_counts_c[i] = 0;
        ++g_counts_len;
    }
    ++g_exec_counts_c[i];
    pthread_mutex_unlock(&g_fft_mu);
}
uint64_t orc_fft_exec_count(size_t n) {
    uint64_t c = 0;
    pthread_mutex_lock(&g_fft_mu);
    for (int i = 0; i < g_counts_len; ++i)
        if (g_exec_counts_n[i] == (uint64_t)n) c = g_exec_counts_c[i];
    pthread_mutex_unlock(&g_fft_mu);
    return c;
}
void orc_fft_reset_exec_counts(void) {
    pthread_mutex_lock(&g_fft_mu);
    g_counts_len = 0;
    pthread_mutex_unlock(&g_fft_mu);
}

static void fft_fwd(int n, const cplx* in, cplx* out) { /* FftPlan::forward fft.hpp:97-102 */
    fft_pair p = orc_fft_plan_for(n);
    fftw_execute_dft(p.fwd, (fftw_complex*)in, (fftw_complex*)out);
    count_exec(n);
}
static void fft_bwd_raw(int n, const cplx* in, cplx* out) { /* fft.hpp:104-109 */
    fft_pair p = orc_fft_plan_for(n);
    fftw_execute_dft(p.bwd, (fftw_complex*)in, (fftw_complex*)out);
    count_exec(n);
}

int orc_fft_forward(const double* in, double* out, size_t n) { /* fft.hpp:140-145 */
    if (n == 0) FAIL(1, "fft_forward: empty input");
    fft_fwd((int)n, (const cplx*)in, (cplx*)out);
    return 0;
}
int orc_fft_inverse(const double* in, double* out, size_t n) { /* fft.hpp:148-156 */
    if (n == 0) FAIL(1, "fft_inverse: empty input");
    cplx* o = (cplx*)out;
    fft_bwd_raw((int)n, (const cplx*)in, o);
    const double scale = 1.0 / (double)n;
    for (size_t i = 0; i < n; ++i) o[i] = cscale(o[i], scale);
    return 0;
}
/* fft.hpp:161-178: rows in place; columns through gather/scatter scratch */
static void fft_rows_forward(cplx* m, size_t rows, size_t cols) {
    for (size_t r = 0; r < rows; ++r) fft_fwd((int)cols, m + r * cols, m + r * cols);
}
static void fft_cols_forward(cplx* m, size_t rows, size_t cols) {
    cplx* in = (cplx*)malloc(sizeof(cplx) * rows);
    cplx* out = (cplx*)malloc(sizeof(cplx) * rows);
    for (size_t c = 0; c < cols; ++c) {
        for (size_t r = 0; r < rows; ++r) in[r] = m[r * cols + c];
        fft_fwd((int)rows, in, out);
        for (size_t r = 0; r < rows; ++r) m[r * cols + c] = out[r];
    }
    free(in);
    free(out);
}
int orc_fft_2d_forward(const double* in, double* out, size_t rows, size_t cols) { /* :185-193 */
    if (rows * cols == 0) FAIL(1, "fft_2d_forward: empty input");
    memcpy(out, in, sizeof(cplx) * rows * cols);
    fft_cols_forward((cplx*)out, rows, cols);
    fft_rows_forward((cplx*)out, rows, cols);
    return 0;
}

/* ------------------------------------------------------ special.hpp */
int orc_lambert_w(double x, double* out) { /* special.hpp:15-31 */
    if (isnan(x) || x < 0.0) FAIL(2, "lambert_w: argument must be nonnegative");
    if (x == 0.0) {
        *out = 0.0;
        return 0;
    }
    double w = log1p(x);
    if (w < 0.0) w = 0.0;
    for (int iter = 0; iter < 50; ++iter) {
        const double ew = exp(w);
        const double f = w * ew - x;
        const double denom = ew * (w + 1.0) - (w + 2.0) * f / (2.0 * w + 2.0);
        const double step = f / denom;
        w -= step;
        if (fabs(f) <= 1e-14 * fabs(x) || fabs(step) <= 1e-16 * fabs(w)) break;
    }
    *out = w;
    return 0;
}

static long double bessel_j_series(int order, long double z) { /* special.hpp:37-49 */
    const long double h = 0.5L * z;
    long double term = 1.0L;
    for (int k = 1; k <= order; ++k) term *= h / (long double)k;
    long double sum = term;
    const long double h2 = -h * h;
    for (int m = 1; m <= 64; ++m) {
        term *= h2 / ((long double)m * (long double)(m + order));
        sum += term;
        if (fabs((double)term) < 1e-22) break;
    }
    return sum;
}

int orc_bessel_j_int(int order, double z, double* out) { /* special.hpp:56-61 */
    if (order < 0) FAIL(2, "bessel_j_int: order must be >= 0");
    if (!(fabs(z) <= 2.0)) FAIL(2, "bessel_j_int: |z| must be <= 2");
    *out = (double)bessel_j_series(order, z);
    return 0;
}

/* ------------------------------------------------------ lowrank.hpp */
/* a[p*K + r] = i^r * (double)(4 J_{(p+r)/2}(z) J_{(r-p)/2}(z)),  z = -gamma*pi/2  (:36-65) */
int orc_cheb_coefficients(double gamma, size_t K, double* a_out) {
    if (!(gamma > 0.0)) FAIL(1, "cheb_coefficients: gamma must be positive");
    if (gamma > 0.5) FAIL(1, "cheb_coefficients: gamma must be <= 1/2");
    if (K < 1) FAIL(1, "cheb_coefficients: K must be >= 1");
    static const double ipow[4][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    const long double kPiExt = 3.14159265358979323846264338327950288L;
    const long double z = -(long double)gamma * kPiExt / 2.0L;
    cplx* a = (cplx*)a_out;
    for (size_t i = 0; i < K * K; ++i) a[i].re = a[i].im = 0.0;
    for (size_t p = 0; p < K; ++p)
        for (size_t r = 0; r < K; ++r) {
            const long diff = (long)r - (long)p;
            if (diff % 2 != 0) continue;
            const int half_sum = (int)((p + r) / 2);
            const int half_diff = (int)(diff / 2);
            long double jj = bessel_j_series(half_sum, z) * bessel_j_series(abs(half_diff), z);
            if (half_diff < 0 && (-half_diff) % 2 != 0) jj = -jj;
            const double d = (double)(4.0L * jj);
            a[p * K + r].re = ipow[r % 4][0] * d;
            a[p * K + r].im = ipow[r % 4][1] * d;
        }
    return 0;
}

static double log_tail_bound(double gamma, size_t K) { /* :70-73 */
    const double km1 = (double)(K - 1);
    return log(140.0) + km1 * (log(5.0 * gamma) - log(km1));
}

/* :95-119 — Table 1 within a factor 2 of a row's epsilon, else Lambert-W plus the nudge */
int orc_select_rank(double gamma, double epsilon, size_t* out) {
    static const double brackets[5] = {1.0 / 32, 1.0 / 16, 1.0 / 8, 1.0 / 4, 1.0 / 2};
    static const double row_eps[3] = {2.2e-16, 1.2e-7, 9.8e-4};
    static const size_t row_k[3][5] = {{8, 9, 11, 13, 16}, {5, 6, 7, 8, 10}, {3, 3, 4, 5, 7}};
    if (!(epsilon > 0.0) || !(epsilon < 1.0)) FAIL(2, "select_rank: epsilon must be in (0, 1)");
    if (!(gamma >= 0.0) || gamma > 0.5) FAIL(2, "select_rank: gamma must be in [0, 1/2]");
    if (gamma == 0.0) {
        *out = 1;
        return 0;
    }
    for (int row = 0; row < 3; ++row) {
        const double ratio = epsilon / row_eps[row];
        if (ratio >= 0.5 && ratio <= 2.0)
            for (int i = 0; i < 5; ++i)
                if (gamma <= brackets[i]) {
                    *out = row_k[row][i];
                    return 0;
                }
    }
    double w;
    orc_lambert_w(log(140.0 / epsilon) / (5.0 * gamma), &w);
    const double raw = 5.0 * gamma * exp(w);
    size_t k = (size_t)ceil(raw);
    if (k < 3) k = 3;
    const double log_eps = log(epsilon);
    while (k <= 64 && log_tail_bound(gamma, k) > log_eps) ++k;
    if (k > 64) FAIL(2, "select_rank: epsilon below attainable precision (rank cap 64)");
    *out = k;
    return 0;
}

/* :126-143 — T_0..T_{K-1} by a long-double three-term recurrence, row-major n x K */
int orc_cheb_eval_matrix(const double* pts, size_t n, size_t K, double* t) {
    if (K < 1) FAIL(1, "cheb_eval_matrix: K must be >= 1");
    long double* row = (long double*)malloc(sizeof(long double) * K);
    for (size_t j = 0; j < n; ++j) {
        double xd = pts[j];
        if (fabs(xd) > 1.0 + 1e-12) {
            free(row);
            FAIL(2, "cheb_eval_matrix: point outside [-1, 1]");
        }
        xd = xd < -1.0 ? -1.0 : (xd > 1.0 ? 1.0 : xd);
        const long double x = xd;
        row[0] = 1.0L;
        if (K > 1) row[1] = x;
        for (size_t p = 2; p < K; ++p) row[p] = 2.0L * x * row[p - 1] - row[p - 2];
        for (size_t p = 0; p < K; ++p) t[j * K + p] = (double)row[p];
    }
    free(row);
    return 0;
}

/* :161-210 — rank-K factors for A_jk = exp(-2 pi i delta_j omega_k).
 * u (rank x n) and v (rank x m) are complex row blocks; pass NULL to query rank. */
int orc_build_factors(const double* delta, size_t n, double gamma, const double* omega_scaled,
                      size_t m, double epsilon, size_t* rank, double* u_out, double* v_out) {
    cplx* u = (cplx*)u_out;
    cplx* v = (cplx*)v_out;
    if (gamma == 0.0) {
        *rank = 1;
        if (u)
            for (size_t j = 0; j < n; ++j) u[j].re = 1.0, u[j].im = 0.0;
        if (v)
            for (size_t k = 0; k < m; ++k) v[k].re = 1.0, v[k].im = 0.0;
        return 0;
    }
    size_t K;
    int rc = orc_select_rank(gamma, epsilon, &K);
    if (rc) return rc;
    *rank = K;
    if (!u && !v) return 0;
    const size_t P = K + 4; /* kCoefficientPadding :156 */
    cplx* coeffs = (cplx*)malloc(sizeof(cplx) * P * P);
    rc = orc_cheb_coefficients(gamma, P, (double*)coeffs);
    if (rc) {
        free(coeffs);
        return rc;
    }
    if (u) {
        double* scaled = (double*)malloc(sizeof(double) * n);
        for (size_t j = 0; j < n; ++j) scaled[j] = delta[j] / gamma;
        double* tp = (double*)malloc(sizeof(double) * n * P);
        rc = orc_cheb_eval_matrix(scaled, n, P, tp);
        free(scaled);
        if (rc) {
            free(tp);
            free(coeffs);
            return rc;
        }
        for (size_t j = 0; j < n; ++j) {
            const double th = -M_PI * delta[j];
            const cplx pre = {cos(th), sin(th)}; /* std::polar(1.0, th) */
            for (size_t r = 0; r < K; ++r) {
                long double ar = 0.5L * (long double)coeffs[r].re;
                long double ai = 0.5L * (long double)coeffs[r].im;
                for (size_t p = 1; p < P; ++p) {
                    const long double tv = (long double)tp[j * P + p];
                    ar += (long double)coeffs[p * P + r].re * tv;
                    ai += (long double)coeffs[p * P + r].im * tv;
                }
                const cplx acc = {(double)ar, (double)ai};
                u[r * n + j] = cmul(pre, acc);
            }
        }
        free(tp);
    }
    if (v) {
        double* w = (double*)malloc(sizeof(double) * m);
        for (size_t k = 0; k < m; ++k) w[k] = 2.0 * omega_scaled[k] - 1.0;
        double* tr = (double*)malloc(sizeof(double) * m * K);
        rc = orc_cheb_eval_matrix(w, m, K, tr);
        free(w);
        if (rc) {
            free(tr);
            free(coeffs);
            return rc;
        }
        for (size_t r = 0; r < K; ++r) {
            const double weight = (r == 0) ? 0.5 : 1.0;
            for (size_t k = 0; k < m; ++k) {
                v[r * m + k].re = weight * tr[k * K + r];
                v[r * m + k].im = 0.0;
            }
        }
        free(tr);
    }
    free(coeffs);
    return 0;
}

/* --------------------------------------------------- transforms.hpp */
int orc_normalize_samples(const double* raw, size_t n, double* out) { /* :35-45 */
    for (size_t j = 0; j < n; ++j) {
        if (!isfinite(raw[j])) FAIL(1, "normalize_samples: sample is not finite");
        double v = raw[j] - floor(raw[j]);
        if (v >= 1.0) v = 0.0;
        out[j] = v;
    }
    return 0;
}

static double exact_perturbation(double grid, double x, double s) { /* :60-64 */
    const double p = grid * x;
    const double err = fma(grid, x, -p);
    return (p - s) + err;
}
static double snap_gamma(double gamma, double grid) { /* :70-73 */
    return gamma <= grid * 0x1p-54 ? 0.0 : gamma;
}

int orc_grid_assign(const double* x, size_t n, size_t grid, long* s, size_t* t, double* gamma) {
    if (grid < 1) FAIL(1, "grid_assign: grid size must be >= 1"); /* :77-92 */
    const double dn = (double)grid;
    double g = 0.0;
    for (size_t j = 0; j < n; ++j) {
        const long sj = (long)round(dn * x[j]);
        s[j] = sj;
        t[j] = (size_t)(sj % (long)grid);
        const double d = fabs(exact_perturbation(dn, x[j], (double)sj));
        if (g < d) g = d;
    }
    *gamma = snap_gamma(g, dn);
    return 0;
}

/* Plan2 (:105-114) */
typedef struct {
    size_t n;
    double eps;
    double* x;
    long* s;
    size_t* t;
    double gamma;
    size_t K;
    cplx* u; /* K x n */
    cplx* v; /* K x n */
} orc_plan2;

static void plan2_free(orc_plan2* p) {
    if (!p) return;
    free(p->x);
    free(p->s);
    free(p->t);
    free(p->u);
    free(p->v);
    free(p);
}
void orc_plan2_destroy(void* p) { plan2_free((orc_plan2*)p); }

/* builds the factors of a plan whose samples (x, s, t, gamma) are filled */
static int plan2_factors(orc_plan2* P, const double* delta, double gamma_for_factors,
                         const double* omega_scaled) {
    size_t K;
    int rc = orc_build_factors(delta, P->n, gamma_for_factors, omega_scaled, P->n, P->eps, &K,
                               NULL, NULL);
    if (rc) return rc;
    P->K = K;
    P->u = (cplx*)malloc(sizeof(cplx) * K * P->n);
    P->v = (cplx*)malloc(sizeof(cplx) * K * P->n);
    return orc_build_factors(delta, P->n, gamma_for_factors, omega_scaled, P->n, P->eps, &K,
                             (double*)P->u, (double*)P->v);
}

int orc_plan2_create(const double* x_raw, size_t n, double eps, void** out) { /* :133-147 */
    if (n == 0) FAIL(1, "plan_nufft2: no samples");
    if (!(eps > 0.0) || !(eps < 1.0)) FAIL(2, "epsilon must be in (0, 1)");
    orc_plan2* P = (orc_plan2*)calloc(1, sizeof(orc_plan2));
    P->n = n;
    P->eps = eps;
    P->x = (double*)malloc(sizeof(double) * n);
    P->s = (long*)malloc(sizeof(long) * n);
    P->t = (size_t*)malloc(sizeof(size_t) * n);
    int rc = orc_normalize_samples(x_raw, n, P->x);
    if (!rc) rc = orc_grid_assign(P->x, n, n, P->s, P->t, &P->gamma);
    if (rc) {
        plan2_free(P);
        return rc;
    }
    double* omega = (double*)malloc(sizeof(double) * n);
    double* delta = (double*)malloc(sizeof(double) * n);
    const double dn = (double)n;
    for (size_t k = 0; k < n; ++k) omega[k] = (double)k / (double)n;
    for (size_t j = 0; j < n; ++j) delta[j] = exact_perturbation(dn, P->x[j], (double)P->s[j]);
    rc = plan2_factors(P, delta, P->gamma, omega);
    free(omega);
    free(delta);
    if (rc) {
        plan2_free(P);
        return rc;
    }
    orc_fft_plan_for((int)n);
    *out = P;
    return 0;
}

size_t orc_plan2_rank(void* p) { return ((orc_plan2*)p)->K; }
double orc_plan2_gamma(void* p) { return ((orc_plan2*)p)->gamma; }
int orc_plan2_samples(void* p, double* x, long* s, size_t* t) {
    orc_plan2* P = (orc_plan2*)p;
    memcpy(x, P->x, sizeof(double) * P->n);
    memcpy(s, P->s, sizeof(long) * P->n);
    memcpy(t, P->t, sizeof(size_t) * P->n);
    return 0;
}
int orc_plan2_factors(void* p, double* u, double* v) {
    orc_plan2* P = (orc_plan2*)p;
    memcpy(u, P->u, sizeof(cplx) * P->K * P->n);
    memcpy(v, P->v, sizeof(cplx) * P->K * P->n);
    return 0;
}

/* accumulate_term :152-161 — f += u_r .* gather_t(F(v_r .* c)) */
static void accumulate_term(const orc_plan2* P, const cplx* c, size_t r, cplx* win, cplx* wout,
                            cplx* f) {
    const size_t n = P->n;
    const cplx* vr = P->v + r * n;
    const cplx* ur = P->u + r * n;
    for (size_t k = 0; k < n; ++k) win[k] = cmul(vr[k], c[k]);
    fft_fwd((int)n, win, wout);
    for (size_t j = 0; j < n; ++j) f[j] = cadd(f[j], cmul(ur[j], wout[P->t[j]]));
}

typedef struct {
    const orc_plan2* P;
    const cplx* c;
    size_t lo, hi;
    cplx* partial;
} term_job;

static void* term_worker(void* arg) {
    term_job* job = (term_job*)arg;
    const size_t n = job->P->n;
    cplx* win = (cplx*)malloc(sizeof(cplx) * n);
    cplx* wout = (cplx*)malloc(sizeof(cplx) * n);
    for (size_t r = job->lo; r < job->hi; ++r)
        accumulate_term(job->P, job->c, r, win, wout, job->partial);
    free(win);
    free(wout);
    return NULL;
}

/* exec_nufft2 :168-199 (threads > 1: contiguous r ranges, merged in worker order) */
int orc_plan2_exec(void* p, const double* c_in, double* f_out, unsigned threads) {
    const orc_plan2* P = (const orc_plan2*)p;
    const size_t n = P->n, k = P->K;
    const cplx* c = (const cplx*)c_in;
    cplx* f = (cplx*)f_out;
    if (threads <= 1 || k == 1) {
        memset(f, 0, sizeof(cplx) * n);
        term_job job = {P, c, 0, k, f};
        term_worker(&job);
        return 0;
    }
    const unsigned workers = threads < k ? threads : (unsigned)k;
    term_job* jobs = (term_job*)malloc(sizeof(term_job) * workers);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
    for (unsigned w = 0; w < workers; ++w) {
        jobs[w].P = P;
        jobs[w].c = c;
        jobs[w].lo = k * w / workers;
        jobs[w].hi = k * (w + 1) / workers;
        jobs[w].partial = (cplx*)calloc(n, sizeof(cplx));
        pthread_create(&th[w], NULL, term_worker, &jobs[w]);
    }
    for (unsigned w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    memcpy(f, jobs[0].partial, sizeof(cplx) * n);
    for (unsigned w = 1; w < workers; ++w)
        for (size_t j = 0; j < n; ++j) f[j] = cadd(f[j], jobs[w].partial[j]);
    for (unsigned w = 0; w < workers; ++w) free(jobs[w].partial);
    free(jobs);
    free(th);
    return 0;
}

/* exec_transpose_core :206-221 */
static void transpose_core(const orc_plan2* P, const cplx* g, cplx* f) {
    const size_t n = P->n;
    cplx* scatter = (cplx*)malloc(sizeof(cplx) * n);
    cplx* work = (cplx*)malloc(sizeof(cplx) * n);
    memset(f, 0, sizeof(cplx) * n);
    for (size_t r = 0; r < P->K; ++r) {
        const cplx* ur = P->u + r * n;
        memset(scatter, 0, sizeof(cplx) * n);
        for (size_t j = 0; j < n; ++j) scatter[P->t[j]] = cadd(scatter[P->t[j]], cmul(ur[j], g[j]));
        for (size_t i = 0; i < n; ++i) scatter[i] = cconj(scatter[i]);
        fft_bwd_raw((int)n, scatter, work);
        const cplx* vr = P->v + r * n;
        for (size_t i = 0; i < n; ++i) f[i] = cadd(f[i], cmul(vr[i], cconj(work[i])));
    }
    free(scatter);
    free(work);
}

int orc_plan2_adjoint(void* p, const double* f_in, double* out) { /* :226-232 */
    const orc_plan2* P = (const orc_plan2*)p;
    const size_t n = P->n;
    cplx* g = (cplx*)malloc(sizeof(cplx) * n);
    for (size_t j = 0; j < n; ++j) g[j] = cconj(((const cplx*)f_in)[j]);
    transpose_core(P, g, (cplx*)out);
    for (size_t j = 0; j < n; ++j) ((cplx*)out)[j] = cconj(((cplx*)out)[j]);
    free(g);
    return 0;
}

/* Plan1 / plan_nufft1 :237-285 — inner type-II plan on omega/N with delta = omega - round(omega) */
typedef struct {
    size_t n;
    double* freqs;
    orc_plan2* inner;
} orc_plan1;

void orc_plan1_destroy(void* p) {
    orc_plan1* P = (orc_plan1*)p;
    if (!P) return;
    free(P->freqs);
    plan2_free(P->inner);
    free(P);
}

static int plan1_build(const double* omega, size_t n, double eps, orc_plan1** out) {
    if (n == 0) FAIL(1, "plan_nufft1: no frequencies");
    if (!(eps > 0.0) || !(eps < 1.0)) FAIL(2, "epsilon must be in (0, 1)");
    const double dn = (double)n;
    double* scaled = (double*)malloc(sizeof(double) * n);
    for (size_t k = 0; k < n; ++k) {
        if (!isfinite(omega[k]) || omega[k] < 0.0 || omega[k] > dn) {
            free(scaled);
            FAIL(1, "plan_nufft1: frequency outside [0, N]");
        }
        scaled[k] = omega[k] / dn;
    }
    orc_plan1* P = (orc_plan1*)calloc(1, sizeof(orc_plan1));
    P->n = n;
    P->freqs = (double*)malloc(sizeof(double) * n);
    memcpy(P->freqs, omega, sizeof(double) * n);
    orc_plan2* in = (orc_plan2*)calloc(1, sizeof(orc_plan2));
    P->inner = in;
    in->n = n;
    in->eps = eps;
    in->x = (double*)malloc(sizeof(double) * n);
    in->s = (long*)malloc(sizeof(long) * n);
    in->t = (size_t*)malloc(sizeof(size_t) * n);
    orc_normalize_samples(scaled, n, in->x);
    free(scaled);
    double* delta = (double*)malloc(sizeof(double) * n);
    double gamma = 0.0;
    for (size_t k = 0; k < n; ++k) {
        const long s = (long)round(omega[k]);
        in->s[k] = s;
        in->t[k] = (size_t)(s % (long)n);
        delta[k] = omega[k] - (double)s;
        const double d = fabs(delta[k]);
        if (gamma < d) gamma = d;
    }
    in->gamma = snap_gamma(gamma, dn);
    double* omega_scaled = (double*)malloc(sizeof(double) * n);
    for (size_t k = 0; k < n; ++k) omega_scaled[k] = (double)k / dn;
    int rc = plan2_factors(in, delta, gamma, omega_scaled); /* un-snapped gamma, :282 */
    free(delta);
    free(omega_scaled);
    if (rc) {
        orc_plan1_destroy(P);
        return rc;
    }
    orc_fft_plan_for((int)n);
    *out = P;
    return 0;
}
int orc_plan1_create(const double* omega, size_t n, double eps, void** out) {
    orc_plan1* P = NULL;
    int rc = plan1_build(omega, n, eps, &P);
    if (!rc) *out = P;
    return rc;
}
size_t orc_plan1_rank(void* p) { return ((orc_plan1*)p)->inner->K; }
double orc_plan1_gamma(void* p) { return ((orc_plan1*)p)->inner->gamma; }
int orc_plan1_exec(void* p, const double* c, double* f) { /* :287-289 */
    transpose_core(((orc_plan1*)p)->inner, (const cplx*)c, (cplx*)f);
    return 0;
}

/* -------------------------------------------------------- oracle.hpp */
static const long double kTwoPiExt = 6.28318530717958647692528676655900577L;
static cplx unit_phase_turns(long double turns) { /* oracle.hpp:51-55 */
    turns -= floorl(turns);
    const long double phase = -kTwoPiExt * turns;
    cplx r = {(double)cosl(phase), (double)sinl(phase)};
    return r;
}
static cplx unit_phase_product(double x, double w) { /* oracle.hpp:59-65 */
    const double p = x * w;
    const double err = fma(x, w, -p);
    const long double turns = (long double)(p - floor(p)) + (long double)err;
    return unit_phase_turns(turns);
}
int orc_unit_phase_product(double x, double w, double* out) {
    cplx z = unit_phase_product(x, w);
    out[0] = z.re;
    out[1] = z.im;
    return 0;
}

/* Plan3 / plan_nufft3 :308-380 */
typedef struct {
    size_t n;
    double* x;
    long* s;
    size_t* t;
    double gamma;
    size_t KA;
    int btrivial;
    size_t kc;
    cplx* cu; /* kc x n */
    cplx* cv; /* kc x n */
    orc_plan1* inner;
} orc_plan3;

void orc_plan3_destroy(void* p) {
    orc_plan3* P = (orc_plan3*)p;
    if (!P) return;
    free(P->x);
    free(P->s);
    free(P->t);
    free(P->cu);
    free(P->cv);
    orc_plan1_destroy(P->inner);
    free(P);
}

int orc_plan3_create(const double* x_raw, const double* omega, size_t n, double eps, void** out) {
    if (n == 0) FAIL(1, "plan_nufft3: no samples");
    if (!(eps > 0.0) || !(eps < 1.0)) FAIL(2, "epsilon must be in (0, 1)");
    const double dn = (double)n;
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(omega[i]) || omega[i] < 0.0 || !(omega[i] < dn))
            FAIL(1, "plan_nufft3: frequency outside [0, N)");
    orc_plan3* P = (orc_plan3*)calloc(1, sizeof(orc_plan3));
    P->n = n;
    P->x = (double*)malloc(sizeof(double) * n);
    P->s = (long*)malloc(sizeof(long) * n);
    P->t = (size_t*)malloc(sizeof(size_t) * n);
    int rc = orc_normalize_samples(x_raw, n, P->x);
    if (!rc) rc = orc_grid_assign(P->x, n, n, P->s, P->t, &P->gamma);
    if (rc) {
        orc_plan3_destroy(P);
        return rc;
    }
    double* omega_scaled = (double*)malloc(sizeof(double) * n);
    double* delta = (double*)malloc(sizeof(double) * n);
    for (size_t k = 0; k < n; ++k) omega_scaled[k] = omega[k] / dn;
    for (size_t j = 0; j < n; ++j) delta[j] = exact_perturbation(dn, P->x[j], (double)P->s[j]);
    size_t K;
    rc = orc_build_factors(delta, n, P->gamma, omega_scaled, n, eps, &K, NULL, NULL);
    if (rc) {
        free(omega_scaled);
        free(delta);
        orc_plan3_destroy(P);
        return rc;
    }
    cplx* ua = (cplx*)malloc(sizeof(cplx) * K * n);
    cplx* va = (cplx*)malloc(sizeof(cplx) * K * n);
    orc_build_factors(delta, n, P->gamma, omega_scaled, n, eps, &K, (double*)ua, (double*)va);
    free(omega_scaled);
    free(delta);
    P->KA = K;
    double* beta = (double*)malloc(sizeof(double) * n);
    int trivial = 1;
    for (size_t j = 0; j < n; ++j) {
        beta[j] = (double)(P->s[j] - (long)P->t[j]) / dn;
        trivial = trivial && beta[j] == 0.0;
    }
    P->btrivial = trivial;
    if (trivial) {
        P->kc = K;
        P->cu = ua;
        P->cv = va;
    } else {
        P->kc = 2 * K;
        P->cu = (cplx*)malloc(sizeof(cplx) * 2 * K * n);
        P->cv = (cplx*)malloc(sizeof(cplx) * 2 * K * n);
        cplx* e = (cplx*)malloc(sizeof(cplx) * n);
        for (size_t i = 0; i < n; ++i) e[i] = unit_phase_product(omega[i], 1.0);
        for (size_t r = 0; r < K; ++r)
            for (size_t j = 0; j < n; ++j) {
                P->cu[r * n + j] = cscale(ua[r * n + j], 1.0 - beta[j]);
                P->cv[r * n + j] = va[r * n + j];
            }
        for (size_t r = 0; r < K; ++r)
            for (size_t j = 0; j < n; ++j) {
                P->cu[(K + r) * n + j] = cscale(ua[r * n + j], beta[j]);
                P->cv[(K + r) * n + j] = cmul(va[r * n + j], e[j]);
            }
        free(e);
        free(ua);
        free(va);
    }
    free(beta);
    rc = plan1_build(omega, n, eps, &P->inner);
    if (rc) {
        orc_plan3_destroy(P);
        return rc;
    }
    *out = P;
    return 0;
}
int orc_plan3_info(void* p, int* btrivial, size_t* rank_a, size_t* effective, size_t* rank_inner) {
    orc_plan3* P = (orc_plan3*)p;
    *btrivial = P->btrivial;
    *rank_a = P->KA;
    *effective = P->kc;
    *rank_inner = P->inner->inner->K;
    return 0;
}
int orc_plan3_exec(void* p, const double* c_in, double* f_out) { /* :382-394 */
    const orc_plan3* P = (const orc_plan3*)p;
    const size_t n = P->n;
    const cplx* c = (const cplx*)c_in;
    cplx* f = (cplx*)f_out;
    cplx* scaled = (cplx*)malloc(sizeof(cplx) * n);
    cplx* y = (cplx*)malloc(sizeof(cplx) * n);
    memset(f, 0, sizeof(cplx) * n);
    for (size_t q = 0; q < P->kc; ++q) {
        const cplx* u = P->cu + q * n;
        const cplx* v = P->cv + q * n;
        for (size_t i = 0; i < n; ++i) scaled[i] = cmul(v[i], c[i]);
        transpose_core(P->inner->inner, scaled, y);
        for (size_t j = 0; j < n; ++j) f[j] = cadd(f[j], cmul(u[j], y[P->t[j]]));
    }
    free(scaled);
    free(y);
    return 0;
}

/* ----------------------------------------------------- transform2d.hpp */
typedef struct {
    size_t m, n, count;
    double *x, *y;
    long *sx, *sy;
    size_t *tx, *ty;
    double gx, gy;
    size_t kx, ky;
    cplx *ux, *vx, *uy, *vy;
    size_t* flat;
} orc_plan2d;

void orc_plan2d2_destroy(void* p) {
    orc_plan2d* P = (orc_plan2d*)p;
    if (!P) return;
    free(P->x);
    free(P->y);
    free(P->sx);
    free(P->sy);
    free(P->tx);
    free(P->ty);
    free(P->ux);
    free(P->vx);
    free(P->uy);
    free(P->vy);
    free(P->flat);
    free(P);
}

int orc_plan2d2_create(const double* x_raw, const double* y_raw, size_t count, size_t m,
                       size_t n, double eps, void** out) { /* transform2d.hpp:65-100 */
    if (count == 0) FAIL(1, "plan_nufft2d2: no samples");
    if (m < 1 || n < 1) FAIL(1, "plan_nufft2d2: grid sizes must be >= 1");
    if (!(eps > 0.0) || !(eps < 1.0)) FAIL(2, "epsilon must be in (0, 1)");
    orc_plan2d* P = (orc_plan2d*)calloc(1, sizeof(orc_plan2d));
    P->m = m;
    P->n = n;
    P->count = count;
    P->x = (double*)malloc(8 * count);
    P->y = (double*)malloc(8 * count);
    P->sx = (long*)malloc(8 * count);
    P->sy = (long*)malloc(8 * count);
    P->tx = (size_t*)malloc(8 * count);
    P->ty = (size_t*)malloc(8 * count);
    int rc = orc_normalize_samples(x_raw, count, P->x);
    if (!rc) rc = orc_normalize_samples(y_raw, count, P->y);
    if (!rc) rc = orc_grid_assign(P->x, count, n, P->sx, P->tx, &P->gx);
    if (!rc) rc = orc_grid_assign(P->y, count, m, P->sy, P->ty, &P->gy);
    if (rc) {
        orc_plan2d2_destroy(P);
        return rc;
    }
    double* dx = (double*)malloc(8 * count);
    double* dy = (double*)malloc(8 * count);
    for (size_t j = 0; j < count; ++j) {
        dx[j] = exact_perturbation((double)n, P->x[j], (double)P->sx[j]);
        dy[j] = exact_perturbation((double)m, P->y[j], (double)P->sy[j]);
    }
    double* wx = (double*)malloc(8 * n);
    double* wy = (double*)malloc(8 * m);
    for (size_t k = 0; k < n; ++k) wx[k] = (double)k / (double)n;
    for (size_t k = 0; k < m; ++k) wy[k] = (double)k / (double)m;
    rc = orc_build_factors(dx, count, P->gx, wx, n, eps, &P->kx, NULL, NULL);
    if (!rc) rc = orc_build_factors(dy, count, P->gy, wy, m, eps, &P->ky, NULL, NULL);
    if (!rc) {
        P->ux = (cplx*)malloc(sizeof(cplx) * P->kx * count);
        P->vx = (cplx*)malloc(sizeof(cplx) * P->kx * n);
        P->uy = (cplx*)malloc(sizeof(cplx) * P->ky * count);
        P->vy = (cplx*)malloc(sizeof(cplx) * P->ky * m);
        orc_build_factors(dx, count, P->gx, wx, n, eps, &P->kx, (double*)P->ux, (double*)P->vx);
        orc_build_factors(dy, count, P->gy, wy, m, eps, &P->ky, (double*)P->uy, (double*)P->vy);
    }
    free(dx);
    free(dy);
    free(wx);
    free(wy);
    if (rc) {
        orc_plan2d2_destroy(P);
        return rc;
    }
    P->flat = (size_t*)malloc(8 * count);
    for (size_t j = 0; j < count; ++j) P->flat[j] = m * P->tx[j] + P->ty[j];
    orc_fft_plan_for((int)m);
    orc_fft_plan_for((int)n);
    *out = P;
    return 0;
}
int orc_plan2d2_info(void* p, size_t* rank_x, size_t* rank_y, double* gx, double* gy) {
    orc_plan2d* P = (orc_plan2d*)p;
    *rank_x = P->kx;
    *rank_y = P->ky;
    *gx = P->gx;
    *gy = P->gy;
    return 0;
}
int orc_plan2d2_flat_index(void* p, size_t* out) {
    orc_plan2d* P = (orc_plan2d*)p;
    memcpy(out, P->flat, 8 * P->count);
    return 0;
}
/* exec_nufft2d2_impl :107-140 (row stage reused across r2) */
int orc_plan2d2_exec(void* p, const double* C_in, double* f_out) {
    const orc_plan2d* P = (const orc_plan2d*)p;
    const size_t m = P->m, n = P->n, count = P->count;
    const cplx* C = (const cplx*)C_in;
    cplx* f = (cplx*)f_out;
    cplx* row_stage = (cplx*)malloc(sizeof(cplx) * m * n);
    cplx* full = (cplx*)malloc(sizeof(cplx) * m * n);
    memset(f, 0, sizeof(cplx) * count);
    for (size_t r1 = 0; r1 < P->kx; ++r1) {
        const cplx* vx = P->vx + r1 * n;
        const cplx* ux = P->ux + r1 * count;
        for (size_t r = 0; r < m; ++r)
            for (size_t c = 0; c < n; ++c) row_stage[r * n + c] = cmul(C[r * n + c], vx[c]);
        fft_rows_forward(row_stage, m, n);
        for (size_t r2 = 0; r2 < P->ky; ++r2) {
            memcpy(full, row_stage, sizeof(cplx) * m * n);
            const cplx* vy = P->vy + r2 * m;
            for (size_t r = 0; r < m; ++r)
                for (size_t c = 0; c < n; ++c) full[r * n + c] = cmul(full[r * n + c], vy[r]);
            fft_cols_forward(full, m, n);
            const cplx* uy = P->uy + r2 * count;
            for (size_t j = 0; j < count; ++j)
                f[j] = cadd(f[j], cmul(cmul(ux[j], uy[j]), full[P->ty[j] * n + P->tx[j]]));
        }
    }
    free(row_stage);
    free(full);
    return 0;
}

/* ---------------------------------------------- direct sums (oracle.hpp) */
typedef struct {
    double sum, comp;
} csum;
static void csum_add(csum* s, double value) { /* oracle.hpp:20-34 Neumaier */
    const double t = s->sum + value;
    if (fabs(s->sum) >= fabs(value))
        s->comp += (s->sum - t) + value;
    else
        s->comp += (value - t) + s->sum;
    s->sum = t;
}

int orc_nudft_direct(const double* x, const double* omega, const double* c_in, size_t n,
                     double* f_out) { /* oracle.hpp:70-84 */
    const cplx* c = (const cplx*)c_in;
    cplx* f = (cplx*)f_out;
    for (size_t j = 0; j < n; ++j) {
        csum re = {0, 0}, im = {0, 0};
        for (size_t k = 0; k < n; ++k) {
            const cplx z = cmul(c[k], unit_phase_product(x[j], omega[k]));
            csum_add(&re, z.re);
            csum_add(&im, z.im);
        }
        f[j].re = re.sum + re.comp;
        f[j].im = im.sum + im.comp;
    }
    return 0;
}

int orc_nudft2d_direct(const double* x, const double* y, size_t count, const double* C_in,
                       size_t m, size_t n, double* f_out) { /* oracle.hpp:88-107 */
    if (m * n == 0) FAIL(1, "nudft2d_direct: inconsistent matrix dimensions");
    const cplx* C = (const cplx*)C_in;
    cplx* f = (cplx*)f_out;
    for (size_t j = 0; j < count; ++j) {
        const long double xj = x[j], yj = y[j];
        csum re = {0, 0}, im = {0, 0};
        for (size_t r = 0; r < m; ++r)
            for (size_t c = 0; c < n; ++c) {
                const cplx z =
                    cmul(C[r * n + c], unit_phase_turns((long double)r * yj + (long double)c * xj));
                csum_add(&re, z.re);
                csum_add(&im, z.im);
            }
        f[j].re = re.sum + re.comp;
        f[j].im = im.sum + im.comp;
    }
    return 0;
}

int orc_worst_grid(size_t n, double gamma, double* x) { /* oracle.hpp:113-127 */
    if (n < 1) FAIL(1, "worst_grid: N must be >= 1");
    if (!(gamma >= 0.0) || gamma > 0.5) FAIL(1, "worst_grid: gamma must be in [0, 1/2]");
    const double dn = (double)n;
    for (size_t j = 0; j < n; ++j) {
        const double shifted = (j <= n / 2) ? ((double)j + gamma) : ((double)j - gamma);
        double v = shifted / dn;
        v -= floor(v);
        x[j] = v;
    }
    return 0;
}

/* ----------------------------------------- random.hpp (mt19937_64 + Box-Muller) */
typedef struct {
    uint64_t mt[312];
    int idx;
    double spare;
    int have_spare;
} orc_sampler;

void* orc_sampler_new(unsigned long long seed) {
    orc_sampler* s = (orc_sampler*)calloc(1, sizeof(orc_sampler));
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
    return s;
}
void orc_sampler_free(void* s) { free(s); }

static uint64_t mt_next(orc_sampler* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) |
                               (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
static double uniform01(orc_sampler* s) { return ldexp((double)(mt_next(s) >> 11), -53); }
double orc_sampler_normal(void* sp) {
    orc_sampler* s = (orc_sampler*)sp;
    if (s->have_spare) {
        s->have_spare = 0;
        return s->spare;
    }
    double u1;
    do {
        u1 = uniform01(s);
    } while (u1 <= 0.0);
    const double u2 = uniform01(s);
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * M_PI * u2;
    s->spare = radius * sin(angle);
    s->have_spare = 1;
    return radius * cos(angle);
}
void orc_sampler_uniform_vector(void* s, size_t n, double lo, double hi, double* out) {
    for (size_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * uniform01((orc_sampler*)s);
}
void orc_sampler_complex_vector(void* s, size_t n, double* out) {
    for (size_t i = 0; i < n; ++i) {
        out[2 * i] = orc_sampler_normal(s);
        out[2 * i + 1] = orc_sampler_normal(s);
    }
}

/* -------------------------------------------------------- inverse.hpp */
/* F1~* g = conj(F2~ conj(g)) on the inner plan (transforms.hpp:294-300) */
int orc_plan1_adjoint(void* p, const double* g_in, double* out) {
    const orc_plan1* P = (const orc_plan1*)p;
    const size_t n = P->n;
    cplx* tmp = (cplx*)malloc(sizeof(cplx) * n);
    for (size_t j = 0; j < n; ++j) tmp[j] = cconj(((const cplx*)g_in)[j]);
    orc_plan2_exec(P->inner, (const double*)tmp, out, 1);
    for (size_t j = 0; j < n; ++j) ((cplx*)out)[j] = cconj(((cplx*)out)[j]);
    free(tmp);
    return 0;
}

typedef struct {
    size_t n;
    cplx* spectrum;  /* 2n, imaginary parts truncated */
    cplx* first_col; /* n */
} orc_toeplitz;

void orc_toeplitz_destroy(void* p) {
    orc_toeplitz* T = (orc_toeplitz*)p;
    if (!T) return;
    free(T->spectrum);
    free(T->first_col);
    free(T);
}

/* detail::toeplitz_from_first_column inverse.hpp:37-50 */
int orc_toeplitz_column(const double* col_in, size_t n, void** out) {
    const cplx* col = (const cplx*)col_in;
    const size_t n2 = 2 * n;
    orc_toeplitz* T = (orc_toeplitz*)calloc(1, sizeof(orc_toeplitz));
    T->n = n;
    T->first_col = (cplx*)malloc(sizeof(cplx) * n);
    memcpy(T->first_col, col, sizeof(cplx) * n);
    cplx* symbol = (cplx*)calloc(n2, sizeof(cplx));
    for (size_t j = 0; j < n; ++j) symbol[j] = col[j];
    for (size_t j = 1; j < n; ++j) symbol[n2 - j] = cconj(col[j]);
    T->spectrum = (cplx*)malloc(sizeof(cplx) * n2);
    fft_fwd((int)n2, symbol, T->spectrum);
    for (size_t j = 0; j < n2; ++j) T->spectrum[j].im = 0.0;
    free(symbol);
    orc_fft_plan_for((int)n2);
    *out = T;
    return 0;
}

/* toeplitz_from_normal inverse.hpp:54-58: first column F2~* F2~ e_0 */
int orc_toeplitz_normal(void* plan2, void** out) {
    const orc_plan2* P = (const orc_plan2*)plan2;
    const size_t n = P->n;
    cplx* e0 = (cplx*)calloc(n, sizeof(cplx));
    cplx* f = (cplx*)malloc(sizeof(cplx) * n);
    cplx* col = (cplx*)malloc(sizeof(cplx) * n);
    e0[0].re = 1.0;
    orc_plan2_exec(plan2, (const double*)e0, (double*)f, 1);
    orc_plan2_adjoint(plan2, (const double*)f, (double*)col);
    int rc = orc_toeplitz_column((const double*)col, n, out);
    free(e0);
    free(f);
    free(col);
    return rc;
}

/* toeplitz_from_gram inverse.hpp:61-66: first column F1~ F1~* e_0 */
int orc_toeplitz_gram(void* plan1, void** out) {
    const orc_plan1* P = (const orc_plan1*)plan1;
    const size_t n = P->n;
    cplx* e0 = (cplx*)calloc(n, sizeof(cplx));
    cplx* g = (cplx*)malloc(sizeof(cplx) * n);
    cplx* col = (cplx*)malloc(sizeof(cplx) * n);
    e0[0].re = 1.0;
    orc_plan1_adjoint(plan1, (const double*)e0, (double*)g);
    orc_plan1_exec(plan1, (const double*)g, (double*)col);
    int rc = orc_toeplitz_column((const double*)col, n, out);
    free(e0);
    free(g);
    free(col);
    return rc;
}

int orc_toeplitz_members(void* p, double* spectrum, double* first_col) {
    const orc_toeplitz* T = (const orc_toeplitz*)p;
    if (spectrum) memcpy(spectrum, T->spectrum, sizeof(cplx) * 2 * T->n);
    if (first_col) memcpy(first_col, T->first_col, sizeof(cplx) * T->n);
    return 0;
}

/* toeplitz_matvec inverse.hpp:70-85 */
static void toeplitz_apply(const orc_toeplitz* T, const cplx* v, cplx* out) {
    const size_t n = T->n, n2 = 2 * n;
    cplx* padded = (cplx*)calloc(n2, sizeof(cplx));
    cplx* spec = (cplx*)malloc(sizeof(cplx) * n2);
    cplx* back = (cplx*)malloc(sizeof(cplx) * n2);
    for (size_t j = 0; j < n; ++j) padded[j] = v[j];
    fft_fwd((int)n2, padded, spec);
    for (size_t j = 0; j < n2; ++j) spec[j] = cscale(spec[j], T->spectrum[j].re);
    fft_bwd_raw((int)n2, spec, back);
    const double scale = 1.0 / (double)n2;
    for (size_t j = 0; j < n; ++j) out[j] = cscale(back[j], scale);
    free(padded);
    free(spec);
    free(back);
}
int orc_toeplitz_matvec(void* p, const double* v, size_t len, double* out) {
    const orc_toeplitz* T = (const orc_toeplitz*)p;
    if (len != T->n) FAIL(1, "toeplitz_matvec: length mismatch");
    toeplitz_apply(T, (const cplx*)v, (cplx*)out);
    return 0;
}

size_t orc_default_cg_max_iter(size_t n) { /* inverse.hpp:161-164 */
    const size_t sqrt_n = (size_t)ceil(sqrt((double)n));
    return 4 * sqrt_n > 100 ? 4 * sqrt_n : 100;
}

static double dot_real(const cplx* a, const cplx* b, size_t n) { /* inverse.hpp:105-111 */
    double s = 0.0;
    for (size_t j = 0; j < n; ++j) s += a[j].re * b[j].re + a[j].im * b[j].im;
    return s;
}
static double norm2(const cplx* v, size_t n) { /* inverse.hpp:99-103 (std::norm = re^2 + im^2) */
    double s = 0.0;
    for (size_t j = 0; j < n; ++j) s += v[j].re * v[j].re + v[j].im * v[j].im;
    return sqrt(s);
}

/* cg_solve inverse.hpp:118-157 with the Toeplitz matvec */
int orc_cg_toeplitz(void* op, const double* rhs_in, size_t n, double tol, size_t max_iter, double* sol_out,
                    size_t* iters, double* relres, int* converged, double* history, size_t* hist_len) {
    const orc_toeplitz* T = (const orc_toeplitz*)op;
    if (!(tol > 0.0)) FAIL(2, "cg_solve: tol must be positive");
    const cplx* rhs = (const cplx*)rhs_in;
    cplx* x = (cplx*)sol_out;
    memset(x, 0, sizeof(cplx) * n);
    *iters = 0;
    *relres = 0.0;
    *converged = 0;
    *hist_len = 0;
    const double rhs_norm = norm2(rhs, n);
    if (rhs_norm == 0.0) {
        *converged = 1;
        return 0;
    }
    cplx* r = (cplx*)malloc(sizeof(cplx) * n);
    cplx* p = (cplx*)malloc(sizeof(cplx) * n);
    cplx* ap = (cplx*)malloc(sizeof(cplx) * n);
    memcpy(r, rhs, sizeof(cplx) * n);
    memcpy(p, r, sizeof(cplx) * n);
    double rho = dot_real(r, r, n);
    int done = 0;
    for (size_t it = 1; it <= max_iter; ++it) {
        toeplitz_apply(T, p, ap);
        const double denom = dot_real(p, ap, n);
        if (denom <= 0.0) break;
        const double alpha = rho / denom;
        for (size_t j = 0; j < n; ++j) {
            x[j] = cadd(x[j], cscale(p[j], alpha));
            r[j].re -= alpha * ap[j].re;
            r[j].im -= alpha * ap[j].im;
        }
        const double rho_next = dot_real(r, r, n);
        *iters = it;
        *relres = sqrt(rho_next) / rhs_norm;
        if (history) history[*hist_len] = *relres;
        ++*hist_len;
        if (*relres <= tol) {
            *converged = 1;
            done = 1;
            break;
        }
        const double beta = rho_next / rho;
        for (size_t j = 0; j < n; ++j) p[j] = cadd(r[j], cscale(p[j], beta));
        rho = rho_next;
    }
    if (!done) *relres = sqrt(rho) / rhs_norm;
    free(r);
    free(p);
    free(ap);
    return 0;
}

/* inufft2 inverse.hpp:171-183 (op NULL: built from the plan) */
int orc_inufft2(void* plan2, void* op, const double* f, double tol, double* sol, size_t* iters, double* relres,
                int* converged, double* history, size_t* hist_len) {
    const orc_plan2* P = (const orc_plan2*)plan2;
    void* own = NULL;
    if (!op) {
        orc_toeplitz_normal(plan2, &own);
        op = own;
    }
    if (!(P->gamma < 0.5)) {
        orc_toeplitz_destroy(own);
        FAIL(2, "inufft2: gamma >= 1/2, samples may not be distinct");
    }
    cplx* rhs = (cplx*)malloc(sizeof(cplx) * P->n);
    orc_plan2_adjoint(plan2, f, (double*)rhs);
    int rc = orc_cg_toeplitz(op, (const double*)rhs, P->n, tol, orc_default_cg_max_iter(P->n), sol, iters, relres,
                             converged, history, hist_len);
    free(rhs);
    orc_toeplitz_destroy(own);
    return rc;
}

/* inufft1 inverse.hpp:187-200 */
int orc_inufft1(void* plan1, void* op, const double* f, double tol, double* sol, size_t* iters, double* relres,
                int* converged, double* history, size_t* hist_len) {
    const orc_plan1* P = (const orc_plan1*)plan1;
    void* own = NULL;
    if (!op) {
        orc_toeplitz_gram(plan1, &own);
        op = own;
    }
    if (!(P->inner->gamma < 0.5)) {
        orc_toeplitz_destroy(own);
        FAIL(2, "inufft1: gamma >= 1/2, frequencies may not be distinct");
    }
    cplx* y = (cplx*)malloc(sizeof(cplx) * P->n);
    int rc = orc_cg_toeplitz(op, f, P->n, tol, orc_default_cg_max_iter(P->n), (double*)y, iters, relres, converged,
                             history, hist_len);
    if (!rc) orc_plan1_adjoint(plan1, (const double*)y, sol);
    free(y);
    orc_toeplitz_destroy(own);
    return rc;
}
