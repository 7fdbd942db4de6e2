#pragma once

// Drop-in for proj/include/nufft/special.hpp: principal Lambert-W and integer
// order Bessel J (plan-time scalars, evaluated by the library's host code in
// the reference's operation order).

#include "fft.hpp"

namespace nufft {

inline double lambert_w(double x) {
    double out = 0.0;
    detail::check(nufft_lambert_w(x, &out));
    return out;
}

inline double bessel_j_int(int order, double z) {
    double out = 0.0;
    detail::check(nufft_bessel_j_int(order, z, &out));
    return out;
}

inline double bessel_j_signed(int order, double z) {
    double out = 0.0;
    detail::check(nufft_bessel_j_signed(order, z, &out));
    return out;
}

}  // namespace nufft
