#pragma once

// Drop-in for proj/include/nufft/inverse.hpp: the type-II normal matrix and
// the type-I Gram matrix as Hermitian Toeplitz operators in their 2N
// circulant embedding, and conjugate gradients.  The operator lives on the
// device (nufft_toeplitz); `spectrum` and `firstColumn` are host mirrors of
// the reference's members.  inufft1/inufft2 run the whole CG solve on the
// GPU (device-resident vectors, fixed-order reductions); cg_solve with an
// arbitrary host callable keeps the reference's host algorithm, since the
// operator is the caller's host code.

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <functional>
#include <memory>
#include <stdexcept>
#include <vector>

#include "nufft/fft.hpp"
#include "nufft/transforms.hpp"

namespace nufft {

/// Hermitian Toeplitz operator (inverse.hpp:22-27).
struct ToeplitzOperator {
    std::size_t n = 0;
    ComplexVector spectrum;     // length 2n, imaginary parts 0
    ComplexVector firstColumn;  // length n
    std::shared_ptr<detail::FftPlan> fft;
    std::shared_ptr<nufft_toeplitz> device;
};

namespace detail {

inline ToeplitzOperator wrap_toeplitz(nufft_toeplitz* raw) {
    ToeplitzOperator op;
    op.device = own<nufft_toeplitz, nufft_toeplitz_destroy>(raw);
    check(nufft_toeplitz_size(raw, &op.n));
    op.spectrum.resize(2 * op.n);
    op.firstColumn.resize(op.n);
    check(nufft_toeplitz_members(raw, dp(op.spectrum), dp(op.firstColumn)));
    op.fft = fft_plan_for(2 * op.n);
    return op;
}

/// inverse.hpp:37-50
inline ToeplitzOperator toeplitz_from_first_column(ComplexVector column) {
    nufft_toeplitz* raw = nullptr;
    check(nufft_toeplitz_from_first_column(dp(column), column.size(), -1, &raw));
    return wrap_toeplitz(raw);
}

}  // namespace detail

/// F2~* F2~ of a type-II plan (inverse.hpp:54-58)
inline ToeplitzOperator toeplitz_from_normal(const Plan2& plan) {
    nufft_toeplitz* raw = nullptr;
    detail::check(nufft_toeplitz_from_normal(plan.device.get(), &raw));
    return detail::wrap_toeplitz(raw);
}

/// F1~ F1~* of a type-I plan (inverse.hpp:61-66)
inline ToeplitzOperator toeplitz_from_gram(const Plan1& plan) {
    nufft_toeplitz* raw = nullptr;
    detail::check(nufft_toeplitz_from_gram(plan.device.get(), &raw));
    return detail::wrap_toeplitz(raw);
}

/// inverse.hpp:70-85 (on the device)
inline ComplexVector toeplitz_matvec(const ToeplitzOperator& op, const ComplexVector& v) {
    if (v.size() != op.n) throw std::invalid_argument("toeplitz_matvec: length mismatch");
    ComplexVector out(op.n);
    detail::check(nufft_toeplitz_matvec_host(op.device.get(), detail::dp(v), v.size(), detail::dp(out)));
    return out;
}

/// inverse.hpp:89-95
struct CgReport {
    ComplexVector solution;
    std::size_t iterations = 0;
    double relativeResidual = 0.0;
    bool converged = false;
    std::vector<double> residualHistory;
};

namespace detail {

/// Re <a, b> = sum_j Re(conj(a_j) b_j), summed in index order
inline double dot_real(const ComplexVector& a, const ComplexVector& b) {
    double acc = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) acc += a[i].real() * b[i].real() + a[i].imag() * b[i].imag();
    return acc;
}

inline double norm2(const ComplexVector& v) { return std::sqrt(dot_real(v, v)); }

inline std::size_t default_cg_max_iter(std::size_t n) { return nufft_default_cg_max_iter(n); }

inline CgReport cg_report(const nufft_cg_report& r, ComplexVector solution, std::vector<double> history) {
    CgReport out;
    out.solution = std::move(solution);
    out.iterations = r.iterations;
    out.relativeResidual = r.relative_residual;
    out.converged = r.converged != 0;
    history.resize(r.history_len);
    out.residualHistory = std::move(history);
    return out;
}

}  // namespace detail

/// Conjugate gradients on the host for a Hermitian positive (semi)definite
/// operator given as a callable (the reference's cg_solve, inverse.hpp:118-157):
/// x0 = 0, the real part of <p, A p> as the step denominator (a non-positive one
/// ends the iteration), relative residual |r_k| / |rhs| recorded after every
/// step and compared with tol, at most max_iter steps.  The device solvers
/// below (inufft1 / inufft2) run the same iteration on the GPU.
template <typename Operator>
CgReport cg_solve(Operator&& apply, const ComplexVector& rhs, double tol, std::size_t max_iter) {
    if (!(tol > 0.0)) throw std::domain_error("cg_solve: tol must be positive");
    CgReport out;
    ComplexVector& x = out.solution;
    x.assign(rhs.size(), Complex(0.0, 0.0));
    const double scale = detail::norm2(rhs);
    if (scale == 0.0) {  // A x = 0 is solved by x = 0
        out.converged = true;
        return out;
    }
    ComplexVector resid(rhs), dir(rhs);
    double rr = detail::dot_real(resid, resid);
    auto update = [](ComplexVector& y, double a, const ComplexVector& v) {
        for (std::size_t i = 0; i < y.size(); ++i) y[i] += a * v[i];
    };
    std::size_t k = 0;
    while (k < max_iter) {
        const ComplexVector q = apply(dir);
        const double curv = detail::dot_real(dir, q);
        if (!(curv > 0.0)) break;  // lost positive definiteness (or a zero direction)
        const double step = rr / curv;
        update(x, step, dir);
        update(resid, -step, q);
        const double rr_new = detail::dot_real(resid, resid);
        ++k;
        out.iterations = k;
        out.relativeResidual = std::sqrt(rr_new) / scale;
        out.residualHistory.push_back(out.relativeResidual);
        if (out.relativeResidual <= tol) {
            out.converged = true;
            return out;
        }
        const double ratio = rr_new / rr;
        for (std::size_t i = 0; i < dir.size(); ++i) dir[i] = resid[i] + ratio * dir[i];
        rr = rr_new;
    }
    out.relativeResidual = std::sqrt(rr) / scale;
    return out;
}

/// Inverse type II on the device (inverse.hpp:171-183).
inline CgReport inufft2(const Plan2& plan, const ToeplitzOperator& op, const ComplexVector& f, double tol) {
    if (f.size() != plan.size()) throw std::invalid_argument("inufft2: length mismatch");
    ComplexVector sol(f.size());
    const std::size_t cap = detail::default_cg_max_iter(plan.size());
    std::vector<double> hist(cap);
    nufft_cg_report rep{};
    detail::check(nufft_inufft2_host(plan.device.get(), op.device.get(), detail::dp(f), f.size(), tol,
                                     detail::dp(sol), &rep, hist.data(), cap));
    return detail::cg_report(rep, std::move(sol), std::move(hist));
}

inline CgReport inufft2(const Plan2& plan, const ComplexVector& f, double tol) {
    if (f.size() != plan.size()) throw std::invalid_argument("inufft2: length mismatch");
    if (!(plan.gamma() < 0.5)) throw std::domain_error("inufft2: gamma >= 1/2, samples may not be distinct");
    return inufft2(plan, toeplitz_from_normal(plan), f, tol);
}

/// Inverse type I on the device (inverse.hpp:187-200).
inline CgReport inufft1(const Plan1& plan, const ToeplitzOperator& op, const ComplexVector& f, double tol) {
    if (f.size() != plan.size()) throw std::invalid_argument("inufft1: length mismatch");
    ComplexVector sol(f.size());
    const std::size_t cap = detail::default_cg_max_iter(plan.size());
    std::vector<double> hist(cap);
    nufft_cg_report rep{};
    detail::check(nufft_inufft1_host(plan.device.get(), op.device.get(), detail::dp(f), f.size(), tol,
                                     detail::dp(sol), &rep, hist.data(), cap));
    return detail::cg_report(rep, std::move(sol), std::move(hist));
}

inline CgReport inufft1(const Plan1& plan, const ComplexVector& f, double tol) {
    if (f.size() != plan.size()) throw std::invalid_argument("inufft1: length mismatch");
    if (!(plan.gamma() < 0.5))
        throw std::domain_error("inufft1: gamma >= 1/2, frequencies may not be distinct");
    return inufft1(plan, toeplitz_from_gram(plan), f, tol);
}

}  // namespace nufft
