#pragma once

// Drop-in for proj/include/nufft/lowrank.hpp: Bessel-product coefficients,
// the rank rule, Chebyshev rows and the rank-K factors.  Per-point work
// (cheb_eval_matrix, build_factors) is evaluated on the GPU.

#include <cstddef>
#include <vector>

#include "fft.hpp"
#include "special.hpp"

namespace nufft {

/// a_pr for one gamma as a K x K row-major block (lowrank.hpp:28-34).
struct ChebCoefficients {
    std::size_t K = 0;
    double gamma = 0.0;
    std::vector<Complex> a;  // a[p * K + r]

    const Complex& at(std::size_t p, std::size_t r) const { return a[p * K + r]; }
};

inline ChebCoefficients cheb_coefficients(double gamma, std::size_t K) {
    ChebCoefficients out;
    out.K = K;
    out.gamma = gamma;
    out.a.assign(K * K, Complex(0, 0));
    detail::check(nufft_cheb_coefficients(gamma, K, reinterpret_cast<double*>(out.a.data())));
    return out;
}

inline std::size_t select_rank(double gamma, double epsilon) {
    std::size_t k = 0;
    detail::check(nufft_select_rank(gamma, epsilon, &k));
    return k;
}

/// Columns T_0 .. T_{K-1}(x) row-major N x K (lowrank.hpp:126-143).
inline std::vector<double> cheb_eval_matrix(const std::vector<double>& points, std::size_t K) {
    std::vector<double> t(points.size() * K);
    detail::check(nufft_cheb_eval_matrix(points.data(), points.size(), K, t.data()));
    return t;
}

/// K column pairs (u_r, v_r) with sum_r u_r v_r^T ~ A (lowrank.hpp:147-151).
struct LowRankFactors {
    std::size_t rank = 0;
    std::vector<ComplexVector> u;
    std::vector<ComplexVector> v;
};

namespace detail {
inline constexpr std::size_t kCoefficientPadding = 4;
}

inline LowRankFactors build_factors(const std::vector<double>& delta, double gamma,
                                    const std::vector<double>& omega_scaled, double epsilon) {
    const std::size_t n = delta.size(), m = omega_scaled.size();
    LowRankFactors out;
    detail::check(nufft_build_factors(delta.data(), n, gamma, omega_scaled.data(), m, epsilon,
                                      &out.rank, nullptr, nullptr));
    std::vector<Complex> u(out.rank * n), v(out.rank * m);
    detail::check(nufft_build_factors(delta.data(), n, gamma, omega_scaled.data(), m, epsilon,
                                      &out.rank, reinterpret_cast<double*>(u.data()),
                                      reinterpret_cast<double*>(v.data())));
    out.u.resize(out.rank);
    out.v.resize(out.rank);
    for (std::size_t r = 0; r < out.rank; ++r) {
        out.u[r].assign(u.begin() + r * n, u.begin() + (r + 1) * n);
        out.v[r].assign(v.begin() + r * m, v.begin() + (r + 1) * m);
    }
    return out;
}

}  // namespace nufft
