// TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// A C-ABI over the UNMODIFIED reference headers, compiled in place from
// /root/reference/proj/include by oracle/Makefile (output: oracle/_ref/,
// git-ignored).  It lets tests/ and bench.py's CPU baseline call the
// reference's own plan/exec functions through ctypes.  Nothing here is part
// of the product; the product library never links it.
//
// Entry points mirror, one to one:
//   plan_nufft2 / exec_nufft2 / exec_nufft2_adjoint  transforms.hpp:133,168,226
//   plan_nufft1 / exec_nufft1                        transforms.hpp:246,287
//   plan_nufft3 / exec_nufft3                        transforms.hpp:321,382
//   plan_nufft2d2 / exec_nufft2d2                    transform2d.hpp:65,145
//   nudft_direct / nudft2d_direct / worst_grid       oracle.hpp:70,88,113
//   select_rank / cheb_coefficients / build_factors  lowrank.hpp:95,36,161
//   fft_forward / fft_inverse / fft_2d_forward       fft.hpp:140,148,185
//   GaussianSampler                                  random.hpp:14-60
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "nufft/nufft.hpp"
#include "nufft/random.hpp"

using namespace nufft;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

std::vector<double> vec(const double* p, size_t n) { return std::vector<double>(p, p + n); }
ComplexVector cvec(const double* p, size_t n) {
    ComplexVector v(n);
    if (n) std::memcpy(v.data(), p, n * sizeof(Complex));
    return v;
}
void put(const ComplexVector& v, double* out) {
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(Complex));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- special / lowrank -------------------------------------------------
int ref_lambert_w(double x, double* out) {
    return guard([&] { *out = lambert_w(x); });
}
int ref_bessel_j_int(int order, double z, double* out) {
    return guard([&] { *out = bessel_j_int(order, z); });
}
int ref_select_rank(double gamma, double eps, size_t* k) {
    return guard([&] { *k = select_rank(gamma, eps); });
}
int ref_cheb_coefficients(double gamma, size_t K, double* a) {
    return guard([&] {
        auto c = cheb_coefficients(gamma, K);
        std::memcpy(a, c.a.data(), c.a.size() * sizeof(Complex));
    });
}
int ref_cheb_eval_matrix(const double* pts, size_t n, size_t K, double* out) {
    return guard([&] {
        auto t = cheb_eval_matrix(vec(pts, n), K);
        std::memcpy(out, t.data(), t.size() * sizeof(double));
    });
}
// u: rank*n complex, v: rank*m complex (caller sizes by the returned rank;
// pass u = v = nullptr to query the rank only).
int ref_build_factors(const double* delta, size_t n, double gamma, const double* omega_scaled,
                      size_t m, double eps, size_t* rank, double* u, double* v) {
    return guard([&] {
        auto f = build_factors(vec(delta, n), gamma, vec(omega_scaled, m), eps);
        *rank = f.rank;
        if (u)
            for (size_t r = 0; r < f.rank; ++r) put(f.u[r], u + 2 * r * n);
        if (v)
            for (size_t r = 0; r < f.rank; ++r) put(f.v[r], v + 2 * r * m);
    });
}

// ---- fft ---------------------------------------------------------------
int ref_fft_forward(const double* in, double* out, size_t n) {
    return guard([&] { put(fft_forward(cvec(in, n)), out); });
}
int ref_fft_inverse(const double* in, double* out, size_t n) {
    return guard([&] { put(fft_inverse(cvec(in, n)), out); });
}
int ref_fft_2d_forward(const double* in, double* out, size_t rows, size_t cols) {
    return guard([&] {
        ComplexMatrix m(rows, cols);
        m.data = cvec(in, rows * cols);
        put(fft_2d_forward(m).data, out);
    });
}

// ---- samples -----------------------------------------------------------
int ref_normalize_samples(const double* raw, size_t n, double* out) {
    return guard([&] {
        auto v = normalize_samples(vec(raw, n));
        std::memcpy(out, v.data(), n * sizeof(double));
    });
}
int ref_grid_assign(const double* x, size_t n, size_t grid, long* s, size_t* t, double* gamma) {
    return guard([&] {
        auto g = grid_assign(vec(x, n), grid);
        std::memcpy(s, g.s.data(), n * sizeof(long));
        std::memcpy(t, g.t.data(), n * sizeof(size_t));
        *gamma = g.gamma;
    });
}

// ---- type II -----------------------------------------------------------
int ref_plan2_create(const double* x, size_t n, double eps, void** out) {
    return guard([&] { *out = new Plan2(plan_nufft2(vec(x, n), eps)); });
}
void ref_plan2_destroy(void* p) { delete static_cast<Plan2*>(p); }
size_t ref_plan2_rank(void* p) { return static_cast<Plan2*>(p)->rank(); }
double ref_plan2_gamma(void* p) { return static_cast<Plan2*>(p)->gamma(); }
int ref_plan2_samples(void* p, double* x, long* s, size_t* t) {
    return guard([&] {
        const auto& S = static_cast<Plan2*>(p)->samples;
        std::memcpy(x, S.x.data(), S.size() * sizeof(double));
        std::memcpy(s, S.s.data(), S.size() * sizeof(long));
        std::memcpy(t, S.t.data(), S.size() * sizeof(size_t));
    });
}
int ref_plan2_factors(void* p, double* u, double* v) {
    return guard([&] {
        const auto& F = static_cast<Plan2*>(p)->factors;
        for (size_t r = 0; r < F.rank; ++r) {
            put(F.u[r], u + 2 * r * F.u[r].size());
            put(F.v[r], v + 2 * r * F.v[r].size());
        }
    });
}
int ref_plan2_exec(void* p, const double* c, double* f, unsigned threads) {
    return guard([&] {
        auto* P = static_cast<Plan2*>(p);
        put(exec_nufft2(*P, cvec(c, P->size()), threads), f);
    });
}
int ref_plan2_adjoint(void* p, const double* f, double* out) {
    return guard([&] {
        auto* P = static_cast<Plan2*>(p);
        put(exec_nufft2_adjoint(*P, cvec(f, P->size())), out);
    });
}

// ---- type I ------------------------------------------------------------
int ref_plan1_create(const double* omega, size_t n, double eps, void** out) {
    return guard([&] { *out = new Plan1(plan_nufft1(vec(omega, n), eps)); });
}
void ref_plan1_destroy(void* p) { delete static_cast<Plan1*>(p); }
size_t ref_plan1_rank(void* p) { return static_cast<Plan1*>(p)->rank(); }
double ref_plan1_gamma(void* p) { return static_cast<Plan1*>(p)->gamma(); }
int ref_plan1_exec(void* p, const double* c, double* f) {
    return guard([&] {
        auto* P = static_cast<Plan1*>(p);
        put(exec_nufft1(*P, cvec(c, P->size())), f);
    });
}

int ref_plan1_adjoint(void* p, const double* g, double* out) {
    return guard([&] {
        auto* P = static_cast<Plan1*>(p);
        put(detail::exec_nufft1_adjoint(*P, cvec(g, P->size())), out);
    });
}

// ---- inverse (inverse.hpp) ---------------------------------------------
int ref_toeplitz_column(const double* col, size_t n, void** out) {
    return guard([&] { *out = new ToeplitzOperator(detail::toeplitz_from_first_column(cvec(col, n))); });
}
int ref_toeplitz_normal(void* plan2, void** out) {
    return guard([&] { *out = new ToeplitzOperator(toeplitz_from_normal(*static_cast<Plan2*>(plan2))); });
}
int ref_toeplitz_gram(void* plan1, void** out) {
    return guard([&] { *out = new ToeplitzOperator(toeplitz_from_gram(*static_cast<Plan1*>(plan1))); });
}
void ref_toeplitz_destroy(void* p) { delete static_cast<ToeplitzOperator*>(p); }
int ref_toeplitz_members(void* p, double* spectrum, double* first_col) {
    return guard([&] {
        auto* T = static_cast<ToeplitzOperator*>(p);
        if (spectrum) put(T->spectrum, spectrum);
        if (first_col) put(T->firstColumn, first_col);
    });
}
int ref_toeplitz_matvec(void* p, const double* v, size_t len, double* out) {
    return guard([&] { put(toeplitz_matvec(*static_cast<ToeplitzOperator*>(p), cvec(v, len)), out); });
}
size_t ref_default_cg_max_iter(size_t n) { return detail::default_cg_max_iter(n); }
static void put_report(const CgReport& r, double* sol, size_t* iters, double* relres, int* conv, double* hist,
                       size_t* hist_len) {
    put(r.solution, sol);
    *iters = r.iterations;
    *relres = r.relativeResidual;
    *conv = r.converged ? 1 : 0;
    *hist_len = r.residualHistory.size();
    if (hist && !r.residualHistory.empty())
        std::memcpy(hist, r.residualHistory.data(), sizeof(double) * r.residualHistory.size());
}
int ref_cg_toeplitz(void* op, const double* rhs, size_t n, double tol, size_t max_iter, double* sol, size_t* iters,
                    double* relres, int* conv, double* hist, size_t* hist_len) {
    return guard([&] {
        auto* T = static_cast<ToeplitzOperator*>(op);
        const CgReport r = cg_solve([T](const ComplexVector& v) { return toeplitz_matvec(*T, v); }, cvec(rhs, n), tol,
                                    max_iter);
        put_report(r, sol, iters, relres, conv, hist, hist_len);
    });
}
int ref_inufft2(void* plan2, void* op, const double* f, double tol, double* sol, size_t* iters, double* relres,
                int* conv, double* hist, size_t* hist_len) {
    return guard([&] {
        auto* P = static_cast<Plan2*>(plan2);
        const CgReport r = op ? inufft2(*P, *static_cast<ToeplitzOperator*>(op), cvec(f, P->size()), tol)
                              : inufft2(*P, cvec(f, P->size()), tol);
        put_report(r, sol, iters, relres, conv, hist, hist_len);
    });
}
int ref_inufft1(void* plan1, void* op, const double* f, double tol, double* sol, size_t* iters, double* relres,
                int* conv, double* hist, size_t* hist_len) {
    return guard([&] {
        auto* P = static_cast<Plan1*>(plan1);
        const CgReport r = op ? inufft1(*P, *static_cast<ToeplitzOperator*>(op), cvec(f, P->size()), tol)
                              : inufft1(*P, cvec(f, P->size()), tol);
        put_report(r, sol, iters, relres, conv, hist, hist_len);
    });
}

// ---- type III ----------------------------------------------------------
int ref_plan3_create(const double* x, const double* omega, size_t n, double eps, void** out) {
    return guard([&] { *out = new Plan3(plan_nufft3(vec(x, n), vec(omega, n), eps)); });
}
void ref_plan3_destroy(void* p) { delete static_cast<Plan3*>(p); }
int ref_plan3_info(void* p, int* btrivial, size_t* rank_a, size_t* effective, size_t* rank_inner) {
    auto* P = static_cast<Plan3*>(p);
    *btrivial = P->bTrivial ? 1 : 0;
    *rank_a = P->factorsA.rank;
    *effective = P->effective_rank();
    *rank_inner = P->inner.rank();
    return 0;
}
int ref_plan3_exec(void* p, const double* c, double* f) {
    return guard([&] {
        auto* P = static_cast<Plan3*>(p);
        put(exec_nufft3(*P, cvec(c, P->size())), f);
    });
}

// ---- 2D type II --------------------------------------------------------
int ref_plan2d2_create(const double* x, const double* y, size_t count, size_t m, size_t n,
                       double eps, void** out) {
    return guard(
        [&] { *out = new Plan2D(plan_nufft2d2(vec(x, count), vec(y, count), m, n, eps)); });
}
void ref_plan2d2_destroy(void* p) { delete static_cast<Plan2D*>(p); }
int ref_plan2d2_info(void* p, size_t* rank_x, size_t* rank_y, double* gx, double* gy) {
    auto* P = static_cast<Plan2D*>(p);
    *rank_x = P->rank_x();
    *rank_y = P->rank_y();
    *gx = P->grid.gammaX;
    *gy = P->grid.gammaY;
    return 0;
}
int ref_plan2d2_flat_index(void* p, size_t* out) {
    auto* P = static_cast<Plan2D*>(p);
    std::memcpy(out, P->flatIndex.data(), P->flatIndex.size() * sizeof(size_t));
    return 0;
}
int ref_plan2d2_exec(void* p, const double* C, double* f) {
    return guard([&] {
        auto* P = static_cast<Plan2D*>(p);
        ComplexMatrix M(P->m, P->n);
        M.data = cvec(C, P->m * P->n);
        put(exec_nufft2d2(*P, M), f);
    });
}

// ---- oracle.hpp ----------------------------------------------------------
int ref_nudft_direct(const double* x, const double* omega, const double* c, size_t n, double* f) {
    return guard([&] { put(nudft_direct(vec(x, n), vec(omega, n), cvec(c, n)), f); });
}
int ref_nudft2d_direct(const double* x, const double* y, size_t count, const double* C, size_t m,
                       size_t n, double* f) {
    return guard([&] {
        ComplexMatrix M(m, n);
        M.data = cvec(C, m * n);
        put(nudft2d_direct(vec(x, count), vec(y, count), M), f);
    });
}
int ref_worst_grid(size_t n, double gamma, double* out) {
    return guard([&] {
        auto v = worst_grid(n, gamma);
        std::memcpy(out, v.data(), n * sizeof(double));
    });
}

// ---- random.hpp ----------------------------------------------------------
void* ref_sampler_new(unsigned long long seed) { return new GaussianSampler(seed); }
void ref_sampler_free(void* s) { delete static_cast<GaussianSampler*>(s); }
double ref_sampler_normal(void* s) { return (*static_cast<GaussianSampler*>(s))(); }
void ref_sampler_uniform_vector(void* s, size_t n, double lo, double hi, double* out) {
    auto v = static_cast<GaussianSampler*>(s)->uniform_vector(n, lo, hi);
    std::memcpy(out, v.data(), n * sizeof(double));
}
void ref_sampler_complex_vector(void* s, size_t n, double* out) {
    put(static_cast<GaussianSampler*>(s)->complex_vector(n), out);
}

}  // extern "C"
