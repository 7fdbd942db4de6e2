// Drop-in usage example and GPU self-check for the C++ headers in include/nufft:
// the same calls a user of the reference makes (README "Library usage"),
// compiled against include/ and linked with libnufft_b200.so.
// Prints "OK" and exits 0 when the checks pass.
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>

#include "nufft/nufft.hpp"

using nufft::Complex;
using nufft::ComplexVector;

static double rel(const ComplexVector& a, const ComplexVector& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / den);
}

int main() {
    std::mt19937_64 eng(7);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> G(0.0, 1.0);
    const size_t n = 1 << 12;
    std::vector<double> x(n);
    ComplexVector c(n);
    for (auto& v : x) v = U(eng);
    for (auto& z : c) z = Complex(G(eng), G(eng));

    nufft::Plan2 plan = nufft::plan_nufft2(x, 1e-14);  // offline stage
    ComplexVector f = nufft::exec_nufft2(plan, c);     // online stage
    if (plan.rank() != 20) return std::printf("rank %zu\n", plan.rank()), 1;
    // direct sum at a few outputs
    double worst = 0;
    for (size_t j = 0; j < n; j += 511) {
        long double re = 0, im = 0;
        for (size_t k = 0; k < n; ++k) {
            const long double ph = -2.0L * 3.14159265358979323846264338327950288L *
                                   std::fmod((long double)x[j] * (long double)k, 1.0L);
            re += c[k].real() * std::cos(ph) - c[k].imag() * std::sin(ph);
            im += c[k].real() * std::sin(ph) + c[k].imag() * std::cos(ph);
        }
        worst = std::max(worst, std::abs(f[j] - Complex((double)re, (double)im)) / std::sqrt((double)n));
    }
    if (!(worst < 1e-12)) return std::printf("direct-sum deviation %g\n", worst), 1;
    // uniform samples -> exactly one FFT
    std::vector<double> eq(96);
    for (size_t j = 0; j < eq.size(); ++j) eq[j] = double(j) / 96.0;
    auto pu = nufft::plan_nufft2(eq, 2.2e-16);
    ComplexVector cu(96, Complex(1, 0));
    nufft::fft_reset_exec_counts();
    auto fu = nufft::exec_nufft2(pu, cu);
    if (nufft::fft_exec_count(96) != 1) return std::printf("fft count\n"), 1;
    if (rel(fu, nufft::fft_forward(cu)) > 1e-14) return std::printf("uniform != fft\n"), 1;
    // exceptions keep the reference's types
    try {
        nufft::plan_nufft2({}, 1e-12);
        return 1;
    } catch (const std::invalid_argument&) {
    }
    try {
        nufft::plan_nufft2({0.5}, 1.0);
        return 1;
    } catch (const std::domain_error&) {
    }
    // concurrent executions of one plan are bit-identical
    ComplexVector a, b;
    std::thread t1([&] { a = nufft::exec_nufft2(plan, c); });
    std::thread t2([&] { b = nufft::exec_nufft2(plan, c); });
    t1.join();
    t2.join();
    if (a != f || b != f) return std::printf("nondeterministic\n"), 1;
    // lazily materialized factors
    if (plan.factors.u.size() != 20 || plan.factors.u[3].size() != n) return 1;
    // type I / III / 2D
    std::vector<double> w(n);
    for (size_t k = 0; k < n; ++k) w[k] = std::min((double)n, std::max(0.0, k + U(eng) - 0.5));
    auto p1 = nufft::plan_nufft1(w, 1e-12);
    auto f1 = nufft::exec_nufft1(p1, c);
    auto p3 = nufft::plan_nufft3(x, std::vector<double>(w.begin(), w.end()), 1e-9);
    (void)p3;
    nufft::ComplexMatrix C(16, 16);
    for (auto& z : C.data) z = Complex(G(eng), G(eng));
    std::vector<double> y(300), xx(300);
    for (auto& v : y) v = U(eng);
    for (auto& v : xx) v = U(eng);
    auto pd = nufft::plan_nufft2d2(xx, y, 16, 16, 1e-9);
    auto fd = nufft::exec_nufft2d2(pd, C);
    if (fd.size() != 300 || f1.size() != n) return 1;
    // multi-GPU drop-in (include/nufft/multi_gpu.hpp) on a one-rank communicator: the
    // in-library r-split with its chunked NCCL reduce equals the single-GPU exec
    {
        nufft::Communicator comm(nufft::make_comm_id(), 1, 0, 0);
        if (comm.nranks() != 1 || comm.rank() != 0) return std::printf("comm info\n"), 1;
        const auto fm = nufft::exec_nufft2(plan, c, comm);
        if (fm != f) return std::printf("exec_multi != exec\n"), 1;
        const auto [r0, r1] = nufft::term_range(plan.rank(), 4, 1);
        if (r0 != 5 || r1 != 10) return std::printf("term_range\n"), 1;
    }
    std::printf("OK rank=%zu worst=%.3g\n", plan.rank(), worst);
    return 0;
}
