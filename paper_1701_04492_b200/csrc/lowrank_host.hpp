// Plan-time scalar math of the low-rank engine (host, long double where the
// reference uses it).  These are O(1) or O(K^2) per plan — the per-sample and
// per-frequency work (factor evaluation, Chebyshev rows) runs on the device.
#pragma once

#include <cstddef>
#include <vector>

namespace nb {

// special.hpp:15-31 — principal Lambert-W on [0, inf) by Halley iteration
double lambert_w(double x);
// special.hpp:37-49 — ascending Bessel series in long double
long double bessel_j_series(int order, long double z);
double bessel_j_int(int order, double z);     // special.hpp:56-61
double bessel_j_signed(int order, double z);  // special.hpp:64-68

// lowrank.hpp:95-119 — Table 1 within a factor 2 of a row, else Lambert-W + nudge
std::size_t select_rank(double gamma, double epsilon);
// lowrank.hpp:36-65 — a[p*K + r] as interleaved complex (2*K*K doubles)
std::vector<double> cheb_coefficients(double gamma, std::size_t K);
// lowrank.hpp:156 — the p-sum runs to P = K + 4
constexpr std::size_t kCoefficientPadding = 4;
constexpr std::size_t kRankCap = 64;

// Bessel-form evaluation of the same factors on the device:
//   u_r(delta) = 2 i^r exp(-i pi delta) J_r(-pi delta),  v_r(w) = (r==0 ? 1/2 : 1) T_r(2w-1)
// (Jacobi-Anger; identical to the reference's Chebyshev expansion
// sum'_p a_pr T_p(delta/gamma) up to its P = K+4 truncation, which is below
// 1e-25 at gamma <= 1/2).  J_r(x) = h^r g_r(h^2), h = x/2, with
//   g_r(w) = sum_m (-w)^m / (m! (m+r)!)
// evaluated by Horner on kSeriesTerms coefficients per r.
constexpr int kSeriesTerms = 16;  // m = 0..15
// coefficient table a[r][m] = (-1)^m/(m!(m+r)!), r < kRankCap (long double, rounded once)
const std::vector<double>& bessel_series_table();
// smallest Horner degree M_r (<= 15) per r so that the truncated tail of
// 2 |h|^r g_r stays below 2^-62 for |delta| <= gamma
std::vector<int> bessel_series_degrees(double gamma, std::size_t K);
// degree of g_r for full RELATIVE accuracy (truncation < 2^-56 of g_r) at |h| <= pi gamma / 2:
// the starting values of the backward Bessel recurrence
int bessel_series_degree_rel(double gamma, int r);

}  // namespace nb
