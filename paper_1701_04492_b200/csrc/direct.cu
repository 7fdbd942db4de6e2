// GPU direct-sum NUDFT: the O(N^2) ground truth of
// proj/include/nufft/oracle.hpp:70-107 on the device, for exact-error sweeps
// at sizes the CPU oracle cannot reach.
//
//   f_j = sum_k c_k exp(-2 pi i x_j w_k)          (nudft_direct, oracle.hpp:70-86)
//   f_j = sum_{r,c} C_rc exp(-2 pi i (r y_j + c x_j))   (nudft2d_direct, :90-107)
//
// Accuracy follows the reference's construction without long double: the
// product x*w is split exactly (p = x*w, e = fma(x, w, -p), oracle.hpp:59-65)
// and reduced mod 1 as the double-double (p - floor(p)) + e; the phase is
// sincospi of the high part times the first-order rotation by the low part
// (|e| <= ulp(p)/2, so the dropped terms are below 1e-17).  Each output is one
// thread summing all terms in ascending k with Neumaier compensation
// (oracle.hpp:20-44), i.e. in the reference's order; inputs are staged through
// shared memory in tiles.
#include <cmath>

#include "plans.hpp"

namespace nb {

namespace {

constexpr int kTile = 256;

struct Neumaier {
    double sum = 0.0, comp = 0.0;
    __device__ __forceinline__ void add(double v) {
        const double t = sum + v;
        if (fabs(sum) >= fabs(v))
            comp += (sum - t) + v;
        else
            comp += (v - t) + sum;
        sum = t;
    }
    __device__ __forceinline__ double value() const { return sum + comp; }
};

// exp(-2 pi i (hi + lo)) with hi in [0, 1) exact and |lo| tiny
__device__ __forceinline__ double2 unit_phase_dd(double hi, double lo) {
    double s, c;
    sincospi(-2.0 * hi, &s, &c);
    const double th = -6.283185307179586476925286766559 * lo;  // rotation by the low part
    const double c2 = __fma_rn(-0.5 * th, th, 1.0);            // cos th to second order
    return make_double2(__fma_rn(-s, th, c * c2), __fma_rn(c, th, s * c2));
}

__device__ __forceinline__ double2 unit_phase_product(double x, double w) {
    const double p = x * w;
    const double e = __fma_rn(x, w, -p);
    return unit_phase_dd(p - floor(p), e);
}

__global__ void __launch_bounds__(kTile) k_nudft_direct(const double* __restrict__ x, long long nx,
                                                        const double* __restrict__ w,
                                                        const double2* __restrict__ c, long long n,
                                                        double2* __restrict__ f) {
    __shared__ double sw[kTile];
    __shared__ double2 sc[kTile];
    const long long j = static_cast<long long>(blockIdx.x) * kTile + threadIdx.x;
    const double xj = j < nx ? x[j] : 0.0;
    Neumaier re, im;
    for (long long k0 = 0; k0 < n; k0 += kTile) {
        __syncthreads();
        if (k0 + threadIdx.x < n) {
            sw[threadIdx.x] = w[k0 + threadIdx.x];
            sc[threadIdx.x] = c[k0 + threadIdx.x];
        }
        __syncthreads();
        const int m = (int)((n - k0) < kTile ? (n - k0) : kTile);
        for (int k = 0; k < m; ++k) {
            const double2 e = unit_phase_product(xj, sw[k]);
            const double2 ck = sc[k];
            re.add(ck.x * e.x - ck.y * e.y);  // std::complex product (ac - bd, ad + bc)
            im.add(ck.x * e.y + ck.y * e.x);
        }
    }
    if (j < nx) f[j] = make_double2(re.value(), im.value());
}

// 2D: turns = r y + c x, each product split exactly, summed in double-double
__global__ void __launch_bounds__(kTile) k_nudft2d_direct(const double* __restrict__ x,
                                                          const double* __restrict__ y, long long cnt,
                                                          const double2* __restrict__ C, long long m,
                                                          long long n, double2* __restrict__ f) {
    __shared__ double2 sc[kTile];
    const long long j = static_cast<long long>(blockIdx.x) * kTile + threadIdx.x;
    const double xj = j < cnt ? x[j] : 0.0, yj = j < cnt ? y[j] : 0.0;
    Neumaier re, im;
    const long long total = m * n;
    for (long long t0 = 0; t0 < total; t0 += kTile) {
        __syncthreads();
        if (t0 + threadIdx.x < total) sc[threadIdx.x] = C[t0 + threadIdx.x];
        __syncthreads();
        const int cntk = (int)((total - t0) < kTile ? (total - t0) : kTile);
        for (int i = 0; i < cntk; ++i) {
            const long long idx = t0 + i;
            const double r = (double)(idx / n), cc = (double)(idx % n);
            const double py = r * yj, ey = __fma_rn(r, yj, -py);
            const double px = cc * xj, ex = __fma_rn(cc, xj, -px);
            const double fy = py - floor(py), fx = px - floor(px);
            const double s = fy + fx;
            const double es = (fy - (s - (s - fy))) + (fx - (s - fy));  // TwoSum error
            const double hi = s - floor(s);
            const double2 e = unit_phase_dd(hi, es + ey + ex);
            const double2 ck = sc[i];
            re.add(ck.x * e.x - ck.y * e.y);
            im.add(ck.x * e.y + ck.y * e.x);
        }
    }
    if (j < cnt) f[j] = make_double2(re.value(), im.value());
}

}  // namespace

void nudft_direct(const double* x, size_t nx, const double* w, const double2* c, size_t n, double2* f,
                  cudaStream_t s) {
    if (nx == 0) return;
    k_nudft_direct<<<(unsigned)((nx + kTile - 1) / kTile), kTile, 0, s>>>(x, (long long)nx, w, c, (long long)n, f);
    NB_LAUNCH();
}

void nudft2d_direct(const double* x, const double* y, size_t cnt, const double2* C, size_t m, size_t n,
                    double2* f, cudaStream_t s) {
    if (cnt == 0) return;
    k_nudft2d_direct<<<(unsigned)((cnt + kTile - 1) / kTile), kTile, 0, s>>>(x, y, (long long)cnt, C, (long long)m,
                                                                              (long long)n, f);
    NB_LAUNCH();
}

}  // namespace nb
