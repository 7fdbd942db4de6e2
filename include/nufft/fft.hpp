#pragma once

// Drop-in replacement for the reference's FFT adapter
// (proj/include/nufft/fft.hpp).  Same types, names and conventions —
// forward = sum_k v_k e^{-2 pi i j k/N} unnormalized, inverse carries 1/N —
// but every transform runs on the GPU through the C-ABI in nufft_b200.h
// (link with libnufft_b200.so).  Errors surface as the reference's exception
// types: std::invalid_argument and std::domain_error.

#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../nufft_b200.h"

namespace nufft {

using Complex = std::complex<double>;
using ComplexVector = std::vector<Complex>;

/// Row-major complex matrix (fft.hpp:26-36).
struct ComplexMatrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    ComplexVector data;

    ComplexMatrix() = default;
    ComplexMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c) {}

    Complex& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    const Complex& at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
};

namespace detail {

/// Re-throw a C-ABI status as the reference's exception type.
inline void check(int rc) {
    if (rc == NUFFT_OK) return;
    const std::string msg = nufft_last_error();
    if (rc == NUFFT_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == NUFFT_DOMAIN_ERROR) throw std::domain_error(msg);
    throw std::runtime_error("nufft_b200: " + msg);
}

inline void check_nonempty(std::size_t n, const char* what) {
    if (n == 0) throw std::invalid_argument(std::string(what) + ": empty input");
}

inline const double* dp(const ComplexVector& v) { return reinterpret_cast<const double*>(v.data()); }
inline double* dp(ComplexVector& v) { return reinterpret_cast<double*>(v.data()); }

/// Size handle kept for API compatibility (fft.hpp:46-78); the device engine
/// selects its own kernels per size.
class FftPlan {
  public:
    explicit FftPlan(std::size_t n) : n_(n) {}
    std::size_t size() const { return n_; }

  private:
    std::size_t n_;
};

// In-place forward DFT of every row / every column (fft.hpp:161-178).
inline void fft_rows_forward(ComplexMatrix& m) {
    check(nufft_fft_rows_forward_host(dp(m.data), m.rows, m.cols));
}
inline void fft_cols_forward(ComplexMatrix& m) {
    check(nufft_fft_cols_forward_host(dp(m.data), m.rows, m.cols));
}

}  // namespace detail

inline std::shared_ptr<detail::FftPlan> fft_plan_for(std::size_t n) {
    detail::check_nonempty(n, "fft_plan_for");
    return std::make_shared<detail::FftPlan>(n);
}

/// Number of logical 1D transforms of size n executed since the last reset.
inline std::uint64_t fft_exec_count(std::size_t n) { return nufft_fft_exec_count(n); }
inline void fft_reset_exec_counts() { nufft_fft_reset_exec_counts(); }

inline ComplexVector fft_forward(const ComplexVector& v) {
    detail::check_nonempty(v.size(), "fft_forward");
    ComplexVector out(v.size());
    detail::check(nufft_fft_forward_host(detail::dp(v), detail::dp(out), v.size()));
    return out;
}

inline ComplexVector fft_inverse(const ComplexVector& v) {
    detail::check_nonempty(v.size(), "fft_inverse");
    ComplexVector out(v.size());
    detail::check(nufft_fft_inverse_host(detail::dp(v), detail::dp(out), v.size()));
    return out;
}

inline ComplexMatrix fft_2d_forward(const ComplexMatrix& c) {
    detail::check_nonempty(c.rows * c.cols, "fft_2d_forward");
    if (c.data.size() != c.rows * c.cols)
        throw std::invalid_argument("fft_2d_forward: inconsistent dimensions");
    ComplexMatrix out(c.rows, c.cols);
    detail::check(nufft_fft_2d_forward_host(detail::dp(c.data), detail::dp(out.data), c.rows, c.cols));
    return out;
}

/// Column-major flattening: entry (r, c) lands at index rows*c + r (fft.hpp:196-201).
inline ComplexVector vec_column_major(const ComplexMatrix& m) {
    ComplexVector out(m.rows * m.cols);
    for (std::size_t c = 0; c < m.cols; ++c)
        for (std::size_t r = 0; r < m.rows; ++r) out[m.rows * c + r] = m.at(r, c);
    return out;
}

}  // namespace nufft
