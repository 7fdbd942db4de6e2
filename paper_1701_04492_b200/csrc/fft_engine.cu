// Generic uniform FFT engine (any length, batched, contiguous) — the device
// replacement for the reference's FFTW plans (proj/include/nufft/fft.hpp:46-109).
//
//   16 <= n <= 4096, n = 2^k : one shared-memory Stockham block FFT per transform
//   n = 2^k > 4096           : 2-3 global Stockham passes of radix L <= 4096
//   n < 16 or non-power-of-two, n <= 2048 : direct sum, exact index (j*k mod n),
//                                           Neumaier-compensated
//   larger non-power-of-two  : Bluestein chirp-z over power-of-two transforms
// The fused NUFFT kernels do not use this path for power-of-two sizes; it
// serves the uniform-FFT API, odd sizes and the 2D row/column stages.
#include <algorithm>

#include "engine.cuh"
#include "fft_block.cuh"

namespace nb {

namespace {

constexpr int kBlockThreads = 256;

// ---------------------------------------------------------- block FFT kernel
template <int L, int SIGN>
__global__ void __launch_bounds__(kBlockThreads) k_fft_block(const double2* in, double2* out,
                                                             size_t batch,
                                                             const double2* __restrict__ tw) {
    constexpr int G = L / 16;
    constexpr int GPC = (G >= kBlockThreads) ? 1 : kBlockThreads / G;
    extern __shared__ double2 smem[];
    const int g = threadIdx.x / G;
    const int tid = threadIdx.x % G;
    double2* buf0 = smem + g * 2 * padded_len(L);
    double2* buf1 = buf0 + padded_len(L);
    double2* t16 = smem + GPC * 2 * padded_len(L);
    twiddle_table_build<L>(t16, threadIdx.x, blockDim.x);
    Twiddles<L> T;
    twiddle_init<L>(T, t16, tid);
    const size_t b = static_cast<size_t>(blockIdx.x) * GPC + g;
    const bool live = b < batch;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
        v[q] = live ? in[b * L + tid + q * G] : make_double2(0.0, 0.0);
    __syncthreads();
    block_fft<L, SIGN>(v, buf0, buf1, tid, T, [] { __syncthreads(); });
    if (live) {
#pragma unroll
        for (int q = 0; q < 16; ++q) out[b * L + tid + q * G] = v[q];
    }
}

template <int L>
constexpr int block_groups() {
    return (L / 16 >= kBlockThreads) ? 1 : kBlockThreads / (L / 16);
}
template <int L>
constexpr size_t block_smem() {
    return sizeof(double2) * (2 * padded_len(L) * block_groups<L>() + FftShapeX<L>::TW_LEN);
}

template <int L, int SIGN>
void launch_fft_block(const double2* in, double2* out, size_t batch, cudaStream_t s,
                      const DeviceCtx& ctx) {
    constexpr int GPC = block_groups<L>();
    constexpr size_t SM = block_smem<L>();
    static std::once_flag once[64];  // per device (attribute is per function, per device)
    std::call_once(once[ctx.device & 63], [] {
        NB_CUDA(cudaFuncSetAttribute(k_fft_block<L, SIGN>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM));
    });
    const size_t grid = (batch + GPC - 1) / GPC;
    k_fft_block<L, SIGN><<<(unsigned)grid, GPC * (L / 16), SM, s>>>(in, out, batch, ctx.table(L));
    NB_LAUNCH();
}

template <int SIGN>
void dispatch_block(const double2* in, double2* out, size_t n, size_t batch, cudaStream_t s,
                    const DeviceCtx& ctx) {
    switch (n) {
        case 16: return launch_fft_block<16, SIGN>(in, out, batch, s, ctx);
        case 32: return launch_fft_block<32, SIGN>(in, out, batch, s, ctx);
        case 64: return launch_fft_block<64, SIGN>(in, out, batch, s, ctx);
        case 128: return launch_fft_block<128, SIGN>(in, out, batch, s, ctx);
        case 256: return launch_fft_block<256, SIGN>(in, out, batch, s, ctx);
        case 512: return launch_fft_block<512, SIGN>(in, out, batch, s, ctx);
        case 1024: return launch_fft_block<1024, SIGN>(in, out, batch, s, ctx);
        case 2048: return launch_fft_block<2048, SIGN>(in, out, batch, s, ctx);
        case 4096: return launch_fft_block<4096, SIGN>(in, out, batch, s, ctx);
        default: throw Error(kInternal, "dispatch_block: bad size");
    }
}

// ------------------------------------------------------ global Stockham pass
// Butterfly j of radix L over an n-point sequence with Ns points already
// combined: inputs x[j + t*n/L] * w_{Ns L}^{(j mod Ns) t}, outputs at
// (j/Ns)*Ns*L + (j mod Ns) + t*Ns.
template <int L, int SIGN>
__global__ void __launch_bounds__(kBlockThreads)
    k_stockham_pass(const double2* __restrict__ in, double2* __restrict__ out, long long n,
                    long long ns, long long nbutterfly, const double2* __restrict__ tw) {
    constexpr int G = L / 16;
    constexpr int GPC = (G >= kBlockThreads) ? 1 : kBlockThreads / G;
    extern __shared__ double2 smem[];
    const int g = threadIdx.x / G;
    const int tid = threadIdx.x % G;
    double2* buf0 = smem + g * 2 * padded_len(L);
    double2* buf1 = buf0 + padded_len(L);
    double2* t16 = smem + GPC * 2 * padded_len(L);
    twiddle_table_build<L>(t16, threadIdx.x, blockDim.x);
    Twiddles<L> T;
    twiddle_init<L>(T, t16, tid);
    const long long j = static_cast<long long>(blockIdx.x) * GPC + g;
    const bool live = j < nbutterfly;
    const size_t boff = static_cast<size_t>(blockIdx.y) * n;
    const long long k = live ? j % ns : 0;
    const long long stride = n / L;
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const long long t = tid + q * G;
        double2 x = live ? in[boff + j + t * stride] : make_double2(0.0, 0.0);
        if (ns > 1 && live) {
            double2 w = unit_root((k * t) % (ns * L), ns * L);
            if (SIGN > 0) w.y = -w.y;
            x = cmul(x, w);
        }
        v[q] = x;
    }
    __syncthreads();
    block_fft<L, SIGN>(v, buf0, buf1, tid, T, [] { __syncthreads(); });
    if (live) {
        const long long base = (j - k) * L + k;
#pragma unroll
        for (int q = 0; q < 16; ++q) out[boff + base + (tid + q * G) * ns] = v[q];
    }
}

template <int L, int SIGN>
void launch_stockham(const double2* in, double2* out, size_t n, size_t ns, size_t batch,
                     cudaStream_t s, const DeviceCtx& ctx) {
    constexpr int GPC = block_groups<L>();
    constexpr size_t SM = block_smem<L>();
    static std::once_flag once[64];
    std::call_once(once[ctx.device & 63], [] {
        NB_CUDA(cudaFuncSetAttribute(k_stockham_pass<L, SIGN>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM));
    });
    const size_t nb = n / L;
    dim3 grid((unsigned)((nb + GPC - 1) / GPC), (unsigned)batch);
    k_stockham_pass<L, SIGN><<<grid, GPC * (L / 16), SM, s>>>(in, out, (long long)n,
                                                              (long long)ns, (long long)nb,
                                                              ctx.table(L));
    NB_LAUNCH();
}

template <int SIGN>
void dispatch_stockham(int L, const double2* in, double2* out, size_t n, size_t ns, size_t batch,
                       cudaStream_t s, const DeviceCtx& ctx) {
    switch (L) {
        case 16: return launch_stockham<16, SIGN>(in, out, n, ns, batch, s, ctx);
        case 32: return launch_stockham<32, SIGN>(in, out, n, ns, batch, s, ctx);
        case 64: return launch_stockham<64, SIGN>(in, out, n, ns, batch, s, ctx);
        case 128: return launch_stockham<128, SIGN>(in, out, n, ns, batch, s, ctx);
        case 256: return launch_stockham<256, SIGN>(in, out, n, ns, batch, s, ctx);
        case 512: return launch_stockham<512, SIGN>(in, out, n, ns, batch, s, ctx);
        case 1024: return launch_stockham<1024, SIGN>(in, out, n, ns, batch, s, ctx);
        case 2048: return launch_stockham<2048, SIGN>(in, out, n, ns, batch, s, ctx);
        case 4096: return launch_stockham<4096, SIGN>(in, out, n, ns, batch, s, ctx);
        default: throw Error(kInternal, "dispatch_stockham: bad radix");
    }
}

// ------------------------------------------------------------ direct DFT
__global__ void k_twiddle_any(double2* tw, long long n, int sign) {
    const long long m = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (m < n) {
        double2 w = unit_root(m, n);
        if (sign > 0) w.y = -w.y;
        tw[m] = w;
    }
}

__device__ __forceinline__ void neumaier(double& sum, double& comp, double v) {
    const double t = sum + v;
    if (fabs(sum) >= fabs(v))
        comp += (sum - t) + v;
    else
        comp += (v - t) + sum;
    sum = t;
}

__global__ void k_dft_direct(const double2* __restrict__ in, double2* __restrict__ out,
                             long long n, long long batch, const double2* __restrict__ tw) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * batch) return;
    const long long b = idx / n, t = idx % n;
    const double2* x = in + b * n;
    double sr = 0, cr = 0, si = 0, ci = 0;
    long long m = 0;
    for (long long k = 0; k < n; ++k) {
        const double2 w = tw[m];
        const double2 xv = x[k];
        const double pr = xv.x * w.x, pi2 = xv.y * w.y, qr = xv.x * w.y, qi = xv.y * w.x;
        neumaier(sr, cr, pr);
        neumaier(sr, cr, -pi2);
        neumaier(si, ci, qr);
        neumaier(si, ci, qi);
        m += t;
        if (m >= n) m -= n;
    }
    out[idx] = make_double2(sr + cr, si + ci);
}

// ------------------------------------------------------------ Bluestein
// chirp w_k = exp(sign * i*pi*k^2/n) with k^2 reduced mod 2n exactly
__device__ __forceinline__ double2 chirp(long long k, long long n, int sign) {
    const unsigned long long kk = static_cast<unsigned long long>(k) * static_cast<unsigned long long>(k);
    const long long r = static_cast<long long>(kk % static_cast<unsigned long long>(2 * n));
    double s, c;
    sincospi((double)r / (double)n, &s, &c);
    return make_double2(c, sign * s);
}

__global__ void k_blue_pre(const double2* __restrict__ x, double2* __restrict__ a, long long n,
                           long long M, long long batch, int sign) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= M * batch) return;
    const long long b = idx / M, k = idx % M;
    a[idx] = (k < n) ? cmul(x[b * n + k], chirp(k, n, sign)) : make_double2(0.0, 0.0);
}
__global__ void k_blue_kernel(double2* __restrict__ bvec, long long n, long long M, int sign) {
    const long long m = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (m >= M) return;
    long long k = -1;
    if (m < n)
        k = m;
    else if (m > M - n)
        k = M - m;
    bvec[m] = (k >= 0) ? cconj(chirp(k, n, sign)) : make_double2(0.0, 0.0);
}
__global__ void k_blue_mul(double2* __restrict__ a, const double2* __restrict__ B, long long M,
                           long long batch) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= M * batch) return;
    a[idx] = cmul(a[idx], B[idx % M]);
}
__global__ void k_blue_post(const double2* __restrict__ conv, double2* __restrict__ out,
                            long long n, long long M, long long batch, int sign) {
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * batch) return;
    const long long b = idx / n, t = idx % n;
    out[idx] = cscale(cmul(conv[b * M + t], chirp(t, n, sign)), 1.0 / (double)M);
}

// ------------------------------------------------------------ transpose
__global__ void k_transpose(const double2* __restrict__ in, double2* __restrict__ out,
                            long long rows, long long cols) {
    __shared__ double2 tile[32][33];
    const size_t boff = static_cast<size_t>(blockIdx.z) * rows * cols;
    const long long c0 = static_cast<long long>(blockIdx.x) * 32, r0 = static_cast<long long>(blockIdx.y) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[boff + r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long long c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[boff + c * rows + r] = tile[threadIdx.x][i];
    }
}

inline unsigned blocks_for(long long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

template <int SIGN>
void fft_pow2_large(const double2* in, double2* out, size_t n, size_t batch, cudaStream_t s,
                    const DeviceCtx& ctx) {
    const int l = ilog2(n);
    std::vector<int> radices;
    if (l <= 24) {
        radices = {1 << ((l + 1) / 2), 1 << (l / 2)};
    } else {
        const int a = (l + 2) / 3, b = (l - a + 1) / 2, c = l - a - b;
        if (c > 12 || a > 12) throw_invalid("fft: size exceeds 2^36");
        radices = {1 << a, 1 << b, 1 << c};
    }
    DevBuf t0(sizeof(double2) * n * batch, s), t1;
    if (radices.size() == 3) t1.alloc(sizeof(double2) * n * batch, s);
    const double2* src = in;
    size_t ns = 1;
    for (size_t i = 0; i < radices.size(); ++i) {
        const bool last = i + 1 == radices.size();
        double2* dst = last ? out : (i == 0 ? t0.as<double2>() : t1.as<double2>());
        dispatch_stockham<SIGN>(radices[i], src, dst, n, ns, batch, s, ctx);
        ns *= radices[i];
        src = dst;
    }
}

void fft_direct(const double2* in, double2* out, size_t n, size_t batch, int sign, cudaStream_t s) {
    DevBuf tw(sizeof(double2) * n, s);
    k_twiddle_any<<<blocks_for(n), 256, 0, s>>>(tw.as<double2>(), (long long)n, sign);
    NB_LAUNCH();
    DevBuf tmp;
    double2* dst = out;
    if (in == out) {
        tmp.alloc(sizeof(double2) * n * batch, s);
        dst = tmp.as<double2>();
    }
    k_dft_direct<<<blocks_for((long long)(n * batch)), 256, 0, s>>>(in, dst, (long long)n,
                                                                    (long long)batch,
                                                                    tw.as<double2>());
    NB_LAUNCH();
    if (in == out)
        NB_CUDA(cudaMemcpyAsync(out, dst, sizeof(double2) * n * batch, cudaMemcpyDeviceToDevice, s));
}

void fft_bluestein(const double2* in, double2* out, size_t n, size_t batch, int sign,
                   cudaStream_t s, int device) {
    size_t M = 1;
    while (M < 2 * n - 1) M <<= 1;
    DevBuf a(sizeof(double2) * M * batch, s), B(sizeof(double2) * M, s);
    k_blue_pre<<<blocks_for((long long)(M * batch)), 256, 0, s>>>(in, a.as<double2>(), (long long)n,
                                                                   (long long)M, (long long)batch, sign);
    NB_LAUNCH();
    k_blue_kernel<<<blocks_for((long long)M), 256, 0, s>>>(B.as<double2>(), (long long)n, (long long)M, sign);
    NB_LAUNCH();
    fft_exec(B.as<double2>(), B.as<double2>(), M, 1, -1, s, device);
    fft_exec(a.as<double2>(), a.as<double2>(), M, batch, -1, s, device);
    k_blue_mul<<<blocks_for((long long)(M * batch)), 256, 0, s>>>(a.as<double2>(), B.as<double2>(),
                                                                   (long long)M, (long long)batch);
    NB_LAUNCH();
    fft_exec(a.as<double2>(), a.as<double2>(), M, batch, +1, s, device);
    k_blue_post<<<blocks_for((long long)(n * batch)), 256, 0, s>>>(a.as<double2>(), out, (long long)n,
                                                                    (long long)M, (long long)batch, sign);
    NB_LAUNCH();
}

}  // namespace

void fft_exec(const double2* in, double2* out, size_t n, size_t batch, int sign, cudaStream_t s,
              int device) {
    if (n == 0 || batch == 0) return;
    const DeviceCtx& ctx = DeviceCtx::get(device);
    if (n == 1) {
        if (in != out)
            NB_CUDA(cudaMemcpyAsync(out, in, sizeof(double2) * batch, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (is_pow2(n) && n >= 16 && n <= 4096) {
        if (sign < 0)
            dispatch_block<-1>(in, out, n, batch, s, ctx);
        else
            dispatch_block<+1>(in, out, n, batch, s, ctx);
        return;
    }
    if (is_pow2(n) && n > 4096) {
        if (sign < 0)
            fft_pow2_large<-1>(in, out, n, batch, s, ctx);
        else
            fft_pow2_large<+1>(in, out, n, batch, s, ctx);
        return;
    }
    if (n <= 2048) return fft_direct(in, out, n, batch, sign, s);
    fft_bluestein(in, out, n, batch, sign, s, device);
}

void transpose(const double2* in, double2* out, size_t rows, size_t cols, size_t batch,
               cudaStream_t s) {
    dim3 block(32, 8);
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32), (unsigned)batch);
    k_transpose<<<grid, block, 0, s>>>(in, out, (long long)rows, (long long)cols);
    NB_LAUNCH();
}

}  // namespace nb
