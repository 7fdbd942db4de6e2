// Inverse NUFFT: Toeplitz normal/Gram operators in
// their 2N circulant embedding and conjugate gradients, on the device.
//
// Reference: proj/include/nufft/inverse.hpp
//   toeplitz_from_first_column :37-50  (h_0..h_{N-1}, 0, conj(h_{N-1})..conj(h_1)),
//                                      forward FFT, imaginary parts truncated
//   toeplitz_from_normal       :54-58  first column = F2~* F2~ e_0
//   toeplitz_from_gram         :61-66  first column = F1~ F1~* e_0
//   toeplitz_matvec            :70-85  pad to 2N, forward, * Re(spectrum), backward, / 2N, truncate
//   cg_solve                   :118-157 plain CG, Hermitian inner product Re(a^H b)
//   inufft2 / inufft1          :171-200
// The vectors stay in HBM for the whole solve; inner products are two-stage
// fixed-order reductions (bit-reproducible run to run); the host reads one
// scalar per reduction to drive the reference's stopping rule.
#include <cmath>
#include <vector>

#include "plans.hpp"

namespace nb {

namespace {

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

constexpr int kRedBlocks = 296;  // 2 x 148 SMs; fixed, so the summation order is fixed
constexpr int kRedThreads = 256;

__global__ void k_embed(const double2* __restrict__ col, double2* __restrict__ sym, long long n) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= 2 * n) return;
    double2 z = make_double2(0.0, 0.0);
    if (j < n) {
        z = col[j];
    } else if (j > n) {
        const double2 c = col[2 * n - j];
        z = make_double2(c.x, -c.y);
    }
    sym[j] = z;
}

__global__ void k_real_part(const double2* __restrict__ spec, double* __restrict__ re, long long m) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < m) re[j] = spec[j].x;
}

__global__ void k_pad(const double2* __restrict__ v, double2* __restrict__ out, long long n) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < 2 * n) out[j] = j < n ? v[j] : make_double2(0.0, 0.0);
}

__global__ void k_spec_mul(double2* __restrict__ spec, const double* __restrict__ re, long long m) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < m) {
        const double s = re[j];
        spec[j] = make_double2(spec[j].x * s, spec[j].y * s);
    }
}

__global__ void k_truncate(const double2* __restrict__ back, double2* __restrict__ out, long long n,
                           double scale) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) out[j] = make_double2(back[j].x * scale, back[j].y * scale);
}

// stage 1: block b sums the products of its fixed strided index set
__global__ void __launch_bounds__(kRedThreads) k_dot_partial(const double2* __restrict__ a,
                                                             const double2* __restrict__ b, long long n,
                                                             double* __restrict__ partial) {
    __shared__ double sm[kRedThreads];
    double s = 0.0;
    for (long long j = static_cast<long long>(blockIdx.x) * kRedThreads + threadIdx.x; j < n;
         j += static_cast<long long>(gridDim.x) * kRedThreads) {
        const double2 x = a[j], y = b[j];
        s = __fma_rn(x.x, y.x, s);
        s = __fma_rn(x.y, y.y, s);
    }
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sm[0];
}

__global__ void __launch_bounds__(kRedThreads) k_dot_final(const double* __restrict__ partial, int nb,
                                                           double* __restrict__ out) {
    __shared__ double sm[kRedThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += kRedThreads) s += partial[i];
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sm[0];
}

__global__ void k_cg_xr(double2* __restrict__ x, double2* __restrict__ r, const double2* __restrict__ p,
                        const double2* __restrict__ ap, double alpha, long long n) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double2 pj = p[j], apj = ap[j];
    double2 xj = x[j], rj = r[j];
    xj.x += alpha * pj.x;
    xj.y += alpha * pj.y;
    rj.x -= alpha * apj.x;
    rj.y -= alpha * apj.y;
    x[j] = xj;
    r[j] = rj;
}

__global__ void k_cg_p(double2* __restrict__ p, const double2* __restrict__ r, double beta, long long n) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double2 rj = r[j], pj = p[j];
    p[j] = make_double2(rj.x + beta * pj.x, rj.y + beta * pj.y);
}

// Re(a^H b), fixed-order, result copied to the host
double dot_real(const double2* a, const double2* b, size_t n, double* partial, double* dres,
                double* hres, cudaStream_t s) {
    k_dot_partial<<<kRedBlocks, kRedThreads, 0, s>>>(a, b, (long long)n, partial);
    NB_LAUNCH();
    k_dot_final<<<1, kRedThreads, 0, s>>>(partial, kRedBlocks, dres);
    NB_LAUNCH();
    NB_CUDA(cudaMemcpyAsync(hres, dres, sizeof(double), cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaStreamSynchronize(s));
    return *hres;
}

}  // namespace

void toeplitz_from_column(ToeplitzState& op, const double2* col, cudaStream_t s) {
    const size_t n = op.n, m = 2 * n;
    op.first_col.alloc(sizeof(double2) * n);
    op.spectrum.alloc(sizeof(double) * m);
    NB_CUDA(cudaMemcpyAsync(op.first_col.as<double2>(), col, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    DevBuf sym(sizeof(double2) * m, s);
    k_embed<<<blocks(m), 256, 0, s>>>(col, sym.as<double2>(), (long long)n);
    NB_LAUNCH();
    fft_exec(sym.as<double2>(), sym.as<double2>(), m, 1, -1, s, op.device);
    fft_count(m);
    k_real_part<<<blocks(m), 256, 0, s>>>(sym.as<double2>(), op.spectrum.as<double>(), (long long)m);
    NB_LAUNCH();
}

void toeplitz_matvec(const ToeplitzState& op, const double2* v, double2* out, cudaStream_t s) {
    const size_t n = op.n, m = 2 * n;
    DevBuf w(sizeof(double2) * m, s);
    k_pad<<<blocks(m), 256, 0, s>>>(v, w.as<double2>(), (long long)n);
    NB_LAUNCH();
    fft_exec(w.as<double2>(), w.as<double2>(), m, 1, -1, s, op.device);
    k_spec_mul<<<blocks(m), 256, 0, s>>>(w.as<double2>(), op.spectrum.as<double>(), (long long)m);
    NB_LAUNCH();
    fft_exec(w.as<double2>(), w.as<double2>(), m, 1, +1, s, op.device);
    fft_count(m, 2);
    k_truncate<<<blocks(n), 256, 0, s>>>(w.as<double2>(), out, (long long)n, 1.0 / (double)m);
    NB_LAUNCH();
}

CgResult cg_solve_toeplitz(const ToeplitzState& op, const double2* rhs, double2* x, double tol,
                           size_t max_iter, std::vector<double>* history, cudaStream_t s) {
    const size_t n = op.n;
    CgResult res;
    DevBuf r(sizeof(double2) * n, s), p(sizeof(double2) * n, s), ap(sizeof(double2) * n, s);
    DevBuf partial(sizeof(double) * kRedBlocks, s), dres(sizeof(double), s);
    double* hres = nullptr;
    NB_CUDA(cudaMallocHost(&hres, sizeof(double)));
    struct Free {
        double* p;
        ~Free() { cudaFreeHost(p); }
    } free_h{hres};
    NB_CUDA(cudaMemsetAsync(x, 0, sizeof(double2) * n, s));
    auto dot = [&](const double2* a, const double2* b) {
        return dot_real(a, b, n, partial.as<double>(), dres.as<double>(), hres, s);
    };
    const double rhs_norm = std::sqrt(dot(rhs, rhs));
    if (rhs_norm == 0.0) {
        res.converged = true;
        return res;
    }
    NB_CUDA(cudaMemcpyAsync(r.get(), rhs, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    NB_CUDA(cudaMemcpyAsync(p.get(), rhs, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    double rho = dot(r.as<double2>(), r.as<double2>());
    for (size_t it = 1; it <= max_iter; ++it) {
        toeplitz_matvec(op, p.as<double2>(), ap.as<double2>(), s);
        const double denom = dot(p.as<double2>(), ap.as<double2>());
        if (denom <= 0.0) break;  // operator lost definiteness at roundoff level
        const double alpha = rho / denom;
        k_cg_xr<<<blocks(n), 256, 0, s>>>(x, r.as<double2>(), p.as<double2>(), ap.as<double2>(), alpha,
                                          (long long)n);
        NB_LAUNCH();
        const double rho_next = dot(r.as<double2>(), r.as<double2>());
        res.iterations = it;
        res.relative_residual = std::sqrt(rho_next) / rhs_norm;
        if (history) history->push_back(res.relative_residual);
        if (res.relative_residual <= tol) {
            res.converged = true;
            return res;
        }
        const double beta = rho_next / rho;
        k_cg_p<<<blocks(n), 256, 0, s>>>(p.as<double2>(), r.as<double2>(), beta, (long long)n);
        NB_LAUNCH();
        rho = rho_next;
    }
    res.relative_residual = std::sqrt(rho) / rhs_norm;
    return res;
}

size_t default_cg_max_iter(size_t n) {  // inverse.hpp:161-164
    const auto sqrt_n = static_cast<size_t>(std::ceil(std::sqrt(static_cast<double>(n))));
    return std::max<size_t>(100, 4 * sqrt_n);
}

}  // namespace nb
