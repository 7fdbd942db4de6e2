// Device evaluation of the low-rank sample factor in Bessel form.
//
//   u_r(delta) = 2 i^r exp(-i pi delta) J_r(-pi delta)
//              = 2 exp(2 i h) (i h)^r g_r(h^2),  h = -pi*delta/2,
//   g_r(w)     = sum_m (-w)^m / (m! (m+r)!)    (Horner, degree deg[r] <= 15)
//
// which is the reference's sum'_p a_pr exp(-i pi delta) T_p(delta/gamma)
// (lowrank.hpp:186-199) without its P = K+4 Chebyshev truncation.  The
// coefficient table is universal (independent of gamma, epsilon) and lives
// in constant memory, one copy per translation unit that includes this
// header (ensure_bessel_constants uploads it per device).
#pragma once

#include <mutex>

#include "common.cuh"
#include "lowrank_host.hpp"

namespace nb {

static __constant__ double kBes[kRankCap * kSeriesTerms];

static inline void ensure_bessel_constants(int device) {
    static std::once_flag once[64];
    std::call_once(once[device & 63], [] {
        const auto& t = bessel_series_table();
        NB_CUDA(cudaMemcpyToSymbol(kBes, t.data(), sizeof(double) * t.size()));
    });
}

// g_r(w) by Horner of degree D (compile time), coefficients kBes[r][0..D]
template <int D>
__device__ __forceinline__ double bessel_g(int r, double w) {
    const double* a = kBes + r * kSeriesTerms;
    double p = a[D];
#pragma unroll
    for (int m = D - 1; m >= 0; --m) p = __fma_rn(p, w, a[m]);
    return p;
}

// runtime-degree variant (generic paths)
__device__ __forceinline__ double bessel_g_rt(int r, int deg, double w) {
    const double* a = kBes + r * kSeriesTerms;
    double p = a[deg];
    for (int m = deg - 1; m >= 0; --m) p = __fma_rn(p, w, a[m]);
    return p;
}

// g_r(w) for C samples at once, degree D fixed at compile time: one
// (uniform, constant-bank) coefficient load feeds C independent FMAs.
template <int C, int D>
__device__ __forceinline__ void series_fixed(double (&g)[C], const double (&w)[C], const double* a) {
#pragma unroll
    for (int c = 0; c < C; ++c) g[c] = a[D];
#pragma unroll
    for (int m = D - 1; m >= 0; --m) {
        const double am = a[m];
#pragma unroll
        for (int c = 0; c < C; ++c) g[c] = __fma_rn(g[c], w[c], am);
    }
}

// runtime degree (warp-uniform) -> unrolled straight-line Horner
template <int C>
__device__ __forceinline__ void series_deg(double (&g)[C], const double (&w)[C], const double* a, int deg) {
    switch (deg) {
        case 0: series_fixed<C, 0>(g, w, a); break;
        case 1: series_fixed<C, 1>(g, w, a); break;
        case 2: series_fixed<C, 2>(g, w, a); break;
        case 3: series_fixed<C, 3>(g, w, a); break;
        case 4: series_fixed<C, 4>(g, w, a); break;
        case 5: series_fixed<C, 5>(g, w, a); break;
        case 6: series_fixed<C, 6>(g, w, a); break;
        case 7: series_fixed<C, 7>(g, w, a); break;
        case 8: series_fixed<C, 8>(g, w, a); break;
        case 9: series_fixed<C, 9>(g, w, a); break;
        case 10: series_fixed<C, 10>(g, w, a); break;
        case 11: series_fixed<C, 11>(g, w, a); break;
        case 12: series_fixed<C, 12>(g, w, a); break;
        case 13: series_fixed<C, 13>(g, w, a); break;
        case 14: series_fixed<C, 14>(g, w, a); break;
        default: series_fixed<C, kSeriesTerms - 1>(g, w, a); break;
    }
}

// -pi/2 * delta
__device__ __forceinline__ double half_phase(double delta) {
    return delta * -1.5707963267948966192313216916397514;
}

// single u_r value (generic paths): 2 exp(2ih) (ih)^r g_r(h^2)
__device__ __forceinline__ double2 u_factor(double delta, int r, int deg) {
    const double h = half_phase(delta);
    const double g = bessel_g_rt(r, deg, h * h);
    double hr = 1.0;
    for (int i = 0; i < r; ++i) hr *= h;
    double s, c;
    sincos(2.0 * h, &s, &c);
    // i^r * (2 hr g) * (c + i s)
    const double m = 2.0 * hr * g;
    double2 z = make_double2(c * m, s * m);
    switch (r & 3) {
        case 1: z = make_double2(-z.y, z.x); break;
        case 2: z = make_double2(-z.x, -z.y); break;
        case 3: z = make_double2(z.y, -z.x); break;
        default: break;
    }
    return z;
}

// v_r(k) = (r==0 ? 1/2 : 1) T_r(2 k/n - 1) by the fp64 three-term recurrence
__device__ __forceinline__ double v_factor_from_s(double s, int r) {
    if (r == 0) return 0.5;
    double tm1 = 1.0, t = s;
    for (int i = 1; i < r; ++i) {
        const double tn = __fma_rn(2.0 * s, t, -tm1);
        tm1 = t;
        t = tn;
    }
    return t;
}
// s = 2*(k/n) - 1 formed as the reference does (lowrank.hpp:202, transforms.hpp:140-142)
__device__ __forceinline__ double grid_s(long long k, long long n) {
    const double w = (double)k / (double)n;
    return __dsub_rn(__dmul_rn(2.0, w), 1.0);
}

}  // namespace nb
