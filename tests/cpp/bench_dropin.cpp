// End-to-end timing of exactly what a C++ user of the reference writes
// (proj/include/nufft/transforms.hpp:133-147, 168-199; random.hpp:14-60):
//
//     nufft::GaussianSampler rng(seed);
//     auto x = rng.uniform_vector(n, 0, 1);  auto c = rng.complex_vector(n);
//     auto plan = nufft::plan_nufft2(x, eps);
//     nufft::ComplexVector f = nufft::exec_nufft2(plan, c);   // timed
//
// compiled against the drop-in headers in include/nufft and linked with
// libnufft_b200.so: pageable std::vector in, freshly allocated std::vector out,
// one vector per call.  bench.py runs it and reports the median as
// e2e.dropin_pageable.  Usage: bench_dropin <n> <eps> <seed> <steps> <warmup>
// Prints one JSON object.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "nufft/nufft.hpp"

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s n eps seed steps warmup\n", argv[0]);
        return 2;
    }
    const size_t n = std::strtoull(argv[1], nullptr, 10);
    const double eps = std::strtod(argv[2], nullptr);
    const unsigned long long seed = std::strtoull(argv[3], nullptr, 10);
    const int steps = std::atoi(argv[4]), warmup = std::atoi(argv[5]);
    using clk = std::chrono::steady_clock;
    try {
        nufft::GaussianSampler rng(seed);
        const std::vector<double> x = rng.uniform_vector(n, 0.0, 1.0);
        const nufft::ComplexVector c = rng.complex_vector(n);
        const auto t0 = clk::now();
        const nufft::Plan2 plan = nufft::plan_nufft2(x, eps);
        const double plan_s = std::chrono::duration<double>(clk::now() - t0).count();
        double checksum = 0.0;
        for (int i = 0; i < warmup; ++i) checksum += std::abs(nufft::exec_nufft2(plan, c)[n / 2]);
        std::vector<double> ms;
        for (int i = 0; i < steps; ++i) {
            const auto a = clk::now();
            const nufft::ComplexVector f = nufft::exec_nufft2(plan, c);
            ms.push_back(std::chrono::duration<double, std::milli>(clk::now() - a).count());
            checksum += std::abs(f[n / 2]);
        }
        std::vector<double> sorted = ms;
        std::sort(sorted.begin(), sorted.end());
        const double med = sorted[sorted.size() / 2];
        std::printf("{\"n\": %zu, \"eps\": %g, \"rank\": %zu, \"plan_s\": %.6f, \"median_ms\": %.6f, "
                    "\"min_ms\": %.6f, \"steps\": %d, \"checksum\": %.17g}\n",
                    n, eps, plan.rank(), plan_s, med, sorted.front(), steps, checksum);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bench_dropin: %s\n", e.what());
        return 1;
    }
    return 0;
}
