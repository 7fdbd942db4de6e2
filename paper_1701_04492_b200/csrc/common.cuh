// Shared device/host helpers for the B200 low-rank NUFFT.
//
// Complex values are double2 (re, im) — byte-compatible with the reference's
// std::complex<double> (proj/include/nufft/fft.hpp:22-23), so host buffers
// cross the C-ABI without repacking.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace nb {

// ------------------------------------------------------------------ errors
// Status codes of the C-ABI (include/nufft_b200.h).
enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,
    kDomainError = 2,
    kCudaError = 3,
    kNcclError = 4,
    kOutOfMemory = 5,
    kInternal = 6,
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(kInvalidArgument, m); }
[[noreturn]] inline void throw_domain(const std::string& m) { throw Error(kDomainError, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    const int code = (e == cudaErrorMemoryAllocation) ? kOutOfMemory : kCudaError;
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")");
}
#define NB_CUDA(x) ::nb::cuda_check((x), #x, __FILE__, __LINE__)
// every kernel launch of the library goes through NB_LAUNCH(), which also
// counts it (nufft_kernel_launch_count) so benchmarks can report launches
void count_launch();
#define NB_LAUNCH()                                                              \
    do {                                                                         \
        ::nb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
        ::nb::count_launch();                                                    \
    } while (0)

// ------------------------------------------------------------------ complex
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
    return make_double2(a.x * s, a.y * s);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
#ifdef __CUDACC__
// a*b with two FMAs (more accurate than the rounded-product form)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__fma_rn(a.x, b.x, -a.y * b.y), __fma_rn(a.x, b.y, a.y * b.x));
}
// acc + a*b
__device__ __forceinline__ double2 cmla(double2 acc, double2 a, double2 b) {
    acc.x = __fma_rn(a.x, b.x, acc.x);
    acc.x = __fma_rn(-a.y, b.y, acc.x);
    acc.y = __fma_rn(a.x, b.y, acc.y);
    acc.y = __fma_rn(a.y, b.x, acc.y);
    return acc;
}
// exp(-2*pi*i * num/den) for integers 0 <= num < den with den a power of two or not;
// the argument num/den is formed once (exact when den is a power of two).
__device__ __forceinline__ double2 unit_root(long long num, long long den) {
    double s, c;
    sincospi(-2.0 * (double)num / (double)den, &s, &c);
    return make_double2(c, s);
}
#endif

// ------------------------------------------------------------------ misc
__host__ __device__ constexpr int ilog2_c(unsigned long long v) {
    int l = 0;
    while ((1ull << l) < v) ++l;
    return l;
}
inline bool is_pow2(size_t v) { return v && !(v & (v - 1)); }
inline int ilog2(size_t v) {
    int l = 0;
    while ((size_t(1) << l) < v) ++l;
    return l;
}
inline int sm_count(int device) {
    int n = 0;
    NB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    return n;
}

}  // namespace nb
