// Plan-time scalar math, restating the reference's host functions in the
// same operation order (so select_rank / cheb_coefficients are bit-identical
// to proj/include/nufft/lowrank.hpp and special.hpp).
#include "lowrank_host.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <mutex>

#include "common.cuh"

namespace nb {

double lambert_w(double x) {  // special.hpp:15-31
    if (std::isnan(x) || x < 0.0) throw_domain("lambert_w: argument must be nonnegative");
    if (x == 0.0) return 0.0;
    double w = std::max(0.0, std::log1p(x));
    for (int iter = 0; iter < 50; ++iter) {
        const double ew = std::exp(w);
        const double f = w * ew - x;
        const double denom = ew * (w + 1.0) - (w + 2.0) * f / (2.0 * w + 2.0);
        const double step = f / denom;
        w -= step;
        if (std::abs(f) <= 1e-14 * std::abs(x) || std::abs(step) <= 1e-16 * std::abs(w)) break;
    }
    return w;
}

long double bessel_j_series(int order, long double z) {  // special.hpp:37-49
    const long double h = 0.5L * z;
    long double term = 1.0L;
    for (int k = 1; k <= order; ++k) term *= h / static_cast<long double>(k);
    long double sum = term;
    const long double h2 = -h * h;
    for (int m = 1; m <= 64; ++m) {
        term *= h2 / (static_cast<long double>(m) * static_cast<long double>(m + order));
        sum += term;
        if (std::abs(static_cast<double>(term)) < 1e-22) break;
    }
    return sum;
}

double bessel_j_int(int order, double z) {  // special.hpp:56-61
    if (order < 0) throw_domain("bessel_j_int: order must be >= 0");
    if (!(std::abs(z) <= 2.0)) throw_domain("bessel_j_int: |z| must be <= 2");
    return static_cast<double>(bessel_j_series(order, z));
}

double bessel_j_signed(int order, double z) {  // special.hpp:64-68
    if (order >= 0) return bessel_j_int(order, z);
    const double v = bessel_j_int(-order, z);
    return (order % 2 == 0) ? v : -v;
}

namespace {
double log_tail_bound(double gamma, std::size_t K) {  // lowrank.hpp:70-73
    const double km1 = static_cast<double>(K - 1);
    return std::log(140.0) + km1 * (std::log(5.0 * gamma) - std::log(km1));
}
struct RankRow {
    double epsilon;
    std::array<std::size_t, 5> k;
};
constexpr std::array<double, 5> kBrackets = {1.0 / 32, 1.0 / 16, 1.0 / 8, 1.0 / 4, 1.0 / 2};
constexpr std::array<RankRow, 3> kTable = {{
    {2.2e-16, {8, 9, 11, 13, 16}},
    {1.2e-7, {5, 6, 7, 8, 10}},
    {9.8e-4, {3, 3, 4, 5, 7}},
}};  // Table 1, lowrank.hpp:75-87
}  // namespace

std::size_t select_rank(double gamma, double epsilon) {  // lowrank.hpp:95-119
    if (!(epsilon > 0.0) || !(epsilon < 1.0))
        throw_domain("select_rank: epsilon must be in (0, 1)");
    if (!(gamma >= 0.0) || gamma > 0.5) throw_domain("select_rank: gamma must be in [0, 1/2]");
    if (gamma == 0.0) return 1;
    for (const auto& row : kTable) {
        const double ratio = epsilon / row.epsilon;
        if (ratio >= 0.5 && ratio <= 2.0)
            for (std::size_t i = 0; i < kBrackets.size(); ++i)
                if (gamma <= kBrackets[i]) return row.k[i];
    }
    const double w = lambert_w(std::log(140.0 / epsilon) / (5.0 * gamma));
    const double raw = 5.0 * gamma * std::exp(w);
    std::size_t k = std::max<std::size_t>(3, static_cast<std::size_t>(std::ceil(raw)));
    const double log_eps = std::log(epsilon);
    while (k <= kRankCap && log_tail_bound(gamma, k) > log_eps) ++k;
    if (k > kRankCap)
        throw_domain("select_rank: epsilon below attainable precision (rank cap 64)");
    return k;
}

std::vector<double> cheb_coefficients(double gamma, std::size_t K) {  // lowrank.hpp:36-65
    if (!(gamma > 0.0)) throw_invalid("cheb_coefficients: gamma must be positive");
    if (gamma > 0.5) throw_invalid("cheb_coefficients: gamma must be <= 1/2");
    if (K < 1) throw_invalid("cheb_coefficients: K must be >= 1");
    static const double ipow[4][2] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    constexpr long double kPiExt = 3.14159265358979323846264338327950288L;
    const long double z = -static_cast<long double>(gamma) * kPiExt / 2.0L;
    std::vector<double> a(2 * K * K, 0.0);
    for (std::size_t p = 0; p < K; ++p)
        for (std::size_t r = 0; r < K; ++r) {
            const long diff = static_cast<long>(r) - static_cast<long>(p);
            if (diff % 2 != 0) continue;
            const int half_sum = static_cast<int>((p + r) / 2);
            const int half_diff = static_cast<int>(diff / 2);
            long double jj =
                bessel_j_series(half_sum, z) * bessel_j_series(std::abs(half_diff), z);
            if (half_diff < 0 && (-half_diff) % 2 != 0) jj = -jj;
            const double d = static_cast<double>(4.0L * jj);
            a[2 * (p * K + r)] = ipow[r % 4][0] * d;
            a[2 * (p * K + r) + 1] = ipow[r % 4][1] * d;
        }
    return a;
}

const std::vector<double>& bessel_series_table() {
    static std::vector<double> table;
    static std::once_flag once;
    std::call_once(once, [] {
        table.assign(kRankCap * kSeriesTerms, 0.0);
        std::vector<long double> fact(kRankCap + kSeriesTerms + 2, 1.0L);
        for (std::size_t i = 1; i < fact.size(); ++i)
            fact[i] = fact[i - 1] * static_cast<long double>(i);
        for (std::size_t r = 0; r < kRankCap; ++r)
            for (int m = 0; m < kSeriesTerms; ++m) {
                const long double v = 1.0L / (fact[m] * fact[m + r]);
                table[r * kSeriesTerms + m] = static_cast<double>((m % 2) ? -v : v);
            }
    });
    return table;
}

std::vector<int> bessel_series_degrees(double gamma, std::size_t K) {
    std::vector<int> deg(K, kSeriesTerms - 1);
    if (!(gamma > 0.0)) {
        std::fill(deg.begin(), deg.end(), 0);
        return deg;
    }
    // |h| <= pi*gamma/2 (with a sliver of slack for rounding of delta)
    const long double hmax = 3.14159265358979323846264338327950288L * gamma / 2.0L * (1.0L + 1e-12L);
    const long double w = hmax * hmax;
    const long double tol = std::ldexp(1.0L, -62);
    for (std::size_t r = 0; r < K; ++r) {
        // tail after degree M: first omitted term w^(M+1)/((M+1)!(M+1+r)!) times a
        // geometric safety factor; scaled by 2 |h|^r
        long double hr = 1.0L;
        for (std::size_t i = 0; i < r; ++i) hr *= hmax;
        for (int M = 0; M < kSeriesTerms; ++M) {
            long double term = 1.0L;  // w^(M+1) / ((M+1)! (M+1+r)!)
            for (int i = 1; i <= M + 1; ++i) term *= w / (static_cast<long double>(i) *
                                                           static_cast<long double>(i + r));
            for (std::size_t i = 1; i <= r; ++i) term /= static_cast<long double>(i);
            const long double ratio = w / ((M + 2.0L) * (M + 2.0L + r));
            const long double tail = term / (1.0L - std::min(ratio, 0.5L));
            if (2.0L * hr * tail <= tol) {
                deg[r] = M;
                break;
            }
        }
    }
    return deg;
}

int bessel_series_degree_rel(double gamma, int r) {
    const long double hmax = 3.14159265358979323846264338327950288L * gamma / 2.0L * (1.0L + 1e-12L);
    const long double w = hmax * hmax;
    const long double tol = std::ldexp(1.0L, -56);
    const long double lower = 1.0L - w / (r + 1.0L);  // g_r r! >= 1 - w/(r+1) (alternating, decreasing)
    if (!(lower > 0.0L)) return kSeriesTerms - 1;
    for (int M = 0; M < kSeriesTerms; ++M) {
        long double term = 1.0L;  // w^(M+1) r! / ((M+1)! (M+1+r)!)
        for (int i = 1; i <= M + 1; ++i) term *= w / (static_cast<long double>(i) * static_cast<long double>(i + r));
        if (term / lower <= tol) return M;
    }
    return kSeriesTerms - 1;
}

}  // namespace nb
