// Plan-stage kernels: sample normalization and nearest-node assignment with
// the exact perturbation, the gamma reduction, fused-path bucketing, and the
// reference-form factor materialization used by the API mirrors.
//
// Reference: normalize_samples transforms.hpp:35-45; grid_assign :77-92;
// exact_perturbation :60-64; snap_gamma :70-73; plan_nufft1 grid data
// :262-277; build_factors lowrank.hpp:161-210; cheb_eval_matrix :126-143.
#include <cub/device/device_radix_sort.cuh>

#include <cmath>

#include "lowrank_host.hpp"
#include "plans.hpp"

namespace nb {

namespace {

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// |delta| >= 0, so the IEEE bit pattern orders like the value.  Reduced over
// the warp first (one atomic per warp instead of one per sample: a single
// contended address otherwise serializes 2^24 atomics).
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* dst, double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, b, o);
        b = other > b ? other : b;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(dst, b);
}

// transforms.hpp:35-45 + :77-92 (+ :60-64 exact delta)
__global__ void k_assign_samples(const double* __restrict__ raw, long long n, long long grid,
                                 double* __restrict__ x, long long* __restrict__ s,
                                 long long* __restrict__ t, double* __restrict__ delta,
                                 unsigned long long* gamma_bits, int* bad) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    double gam = 0.0;
    if (j < n) {
        const double r = raw[j];
        if (!isfinite(r)) {
            atomicOr(bad, 1);
        } else {
            double v = __dsub_rn(r, floor(r));
            if (v >= 1.0) v = 0.0;
            const double dn = (double)grid;
            const double p = __dmul_rn(dn, v);
            const long long sj = (long long)round(p);
            const double err = __fma_rn(dn, v, -p);
            const double d = __dadd_rn(__dsub_rn(p, (double)sj), err);
            x[j] = v;
            s[j] = sj;
            t[j] = sj % grid;
            delta[j] = d;
            gam = fabs(d);
        }
    }
    atomic_max_nonneg(gamma_bits, gam);
}

// transforms.hpp:246-277: omega in [0, N] (type I) or [0, N) (type III, upper_open)
__global__ void k_assign_freqs(const double* __restrict__ omega, long long n, int upper_open,
                               double* __restrict__ x, long long* __restrict__ s,
                               long long* __restrict__ t, double* __restrict__ delta,
                               unsigned long long* gamma_bits, int* bad) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    double gam = 0.0;
    if (k < n) {
        const double w = omega[k];
        const double dn = (double)n;
        if (!isfinite(w) || w < 0.0 || w > dn || (upper_open && !(w < dn))) {
            atomicOr(bad, 1);
        } else {
            const double scaled = __ddiv_rn(w, dn);
            double v = __dsub_rn(scaled, floor(scaled));
            if (v >= 1.0) v = 0.0;
            const long long sk = (long long)round(w);
            const double d = __dsub_rn(w, (double)sk);
            x[k] = v;
            s[k] = sk;
            t[k] = sk % n;
            delta[k] = d;
            gam = fabs(d);
        }
    }
    atomic_max_nonneg(gamma_bits, gam);
}

__global__ void k_bucket_keys(const long long* __restrict__ t, long long n, int log_n1, int log_n2,
                              unsigned* __restrict__ keys, int* __restrict__ idx) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const unsigned long long tj = (unsigned long long)t[j];
    const unsigned long long n1m = (1ull << log_n1) - 1;
    keys[j] = (unsigned)(((tj & n1m) << log_n2) | (tj >> log_n1));
    idx[j] = (int)j;
}

__global__ void k_plain_keys(const long long* __restrict__ t, long long n,
                             unsigned long long* __restrict__ keys, int* __restrict__ idx) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    keys[j] = (unsigned long long)t[j];
    idx[j] = (int)j;
}

// offsets[b] = first sorted position whose bucket >= b, b in [0, nbuckets]
template <class Key>
__global__ void k_bucket_offsets(const Key* __restrict__ keys, long long n, int shift,
                                 long long nbuckets, int* __restrict__ off) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > n) return;
    const long long cur = (i < n) ? (long long)(keys[i] >> shift) : nbuckets;
    const long long prev = (i > 0) ? (long long)(keys[i - 1] >> shift) : -1;
    for (long long b = prev + 1; b <= cur; ++b) off[b] = (int)i;
}

// key t_j (< 2^31) and the wraparound flag beta_j = (s_j != t_j) in bit 31
__global__ void k_t3_keys(const long long* __restrict__ sv, const long long* __restrict__ tv, long long n,
                          unsigned* __restrict__ keys, unsigned* __restrict__ flags, int* __restrict__ idx) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    keys[j] = (unsigned)tv[j];
    flags[j] = (unsigned)tv[j] | (sv[j] != tv[j] ? 0x80000000u : 0u);
    idx[j] = (int)j;
}
__global__ void k_t3_gather(const int* __restrict__ perm, const unsigned* __restrict__ flags,
                            const double* __restrict__ delta, long long n, unsigned* __restrict__ key,
                            double* __restrict__ ds) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j = perm[i];
    key[i] = flags[j];
    ds[i] = delta[j];
}

__global__ void k_invert_perm(const int* __restrict__ perm, long long n, int* __restrict__ inv) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) inv[perm[i]] = (int)i;
}

__global__ void k_gather_x(const double* __restrict__ x, const int* __restrict__ perm, long long n,
                           double* __restrict__ xs) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) xs[i] = x[perm[i]];
}

// reference-form factor u (lowrank.hpp:174-199), fp64 Chebyshev recurrence and sum
__global__ void k_factors_u(const double* __restrict__ delta, long long n, double gamma, int K,
                            int P, const double* __restrict__ a, double2* __restrict__ u) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double d = delta[j];
    double y = __ddiv_rn(d, gamma);
    y = fmin(1.0, fmax(-1.0, y));
    double sn, cs;
    sincos(__dmul_rn(-3.141592653589793, d), &sn, &cs);
    for (int r = 0; r < K; ++r) {
        double ar = 0.5 * a[2 * r], ai = 0.5 * a[2 * r + 1];
        double tm1 = 1.0, tp = y;
        for (int p = 1; p < P; ++p) {
            if (p >= 2) {
                const double tn = __fma_rn(2.0 * y, tp, -tm1);
                tm1 = tp;
                tp = tn;
            }
            ar = __fma_rn(a[2 * (p * P + r)], tp, ar);
            ai = __fma_rn(a[2 * (p * P + r) + 1], tp, ai);
        }
        u[(long long)r * n + j] = make_double2(__dsub_rn(__dmul_rn(cs, ar), __dmul_rn(sn, ai)),
                                               __dadd_rn(__dmul_rn(cs, ai), __dmul_rn(sn, ar)));
    }
}

// v_r(w) = (r==0 ? 1/2 : 1) T_r(2w - 1)  (lowrank.hpp:201-209)
__global__ void k_factors_v(const double* __restrict__ omega_scaled, long long m, int K,
                            double2* __restrict__ v, int* bad) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= m) return;
    double w = __dsub_rn(__dmul_rn(2.0, omega_scaled[k]), 1.0);
    if (fabs(w) > 1.0 + 1e-12) {
        atomicOr(bad, 1);
        return;
    }
    w = fmin(1.0, fmax(-1.0, w));
    double tm1 = 1.0, t = w;
    for (int r = 0; r < K; ++r) {
        double val;
        if (r == 0) {
            val = 0.5;
        } else if (r == 1) {
            val = t;
        } else {
            const double tn = __fma_rn(2.0 * w, t, -tm1);
            tm1 = t;
            t = tn;
            val = t;
        }
        v[(long long)r * m + k] = make_double2(val, 0.0);
    }
}

__global__ void k_cheb_eval(const double* __restrict__ pts, long long n, int K,
                            double* __restrict__ out, int* bad) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double x = pts[j];
    if (fabs(x) > 1.0 + 1e-12) {
        atomicOr(bad, 1);
        return;
    }
    x = fmin(1.0, fmax(-1.0, x));
    double tm1 = 1.0, t = x;
    out[j * K] = 1.0;
    if (K > 1) out[j * K + 1] = x;
    for (int p = 2; p < K; ++p) {
        const double tn = __fma_rn(2.0 * x, t, -tm1);
        tm1 = t;
        t = tn;
        out[j * K + p] = t;
    }
}

struct Reduce {
    unsigned long long gamma_bits;
    int bad;
};

double snap_gamma(double gamma, double grid) {  // transforms.hpp:70-73
    constexpr double quarter_eps = 0x1p-54;
    return gamma <= grid * quarter_eps ? 0.0 : gamma;
}

}  // namespace

void assign_samples(Axis& ax, const double* raw, bool raw_on_device, size_t n, size_t grid,
                    cudaStream_t s) {
    if (grid < 1) throw_invalid("grid_assign: grid size must be >= 1");
    ax.n = n;
    ax.grid = grid;
    ax.x.alloc(8 * n);
    ax.s.alloc(8 * n);
    ax.t.alloc(8 * n);
    ax.delta.alloc(8 * n);
    DevBuf red(sizeof(Reduce), s), tmp;
    NB_CUDA(cudaMemsetAsync(red.get(), 0, sizeof(Reduce), s));
    const double* src = raw;
    if (!raw_on_device) {
        tmp.alloc(8 * n, s);
        NB_CUDA(cudaMemcpyAsync(tmp.get(), raw, 8 * n, cudaMemcpyHostToDevice, s));
        src = tmp.as<double>();
    }
    Reduce* r = red.as<Reduce>();
    if (n) {
        k_assign_samples<<<blocks(n), 256, 0, s>>>(src, (long long)n, (long long)grid,
                                                   ax.x.as<double>(), ax.s.as<long long>(),
                                                   ax.t.as<long long>(), ax.delta.as<double>(),
                                                   &r->gamma_bits, &r->bad);
        NB_LAUNCH();
    }
    Reduce h{};
    NB_CUDA(cudaMemcpyAsync(&h, r, sizeof(Reduce), cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaStreamSynchronize(s));
    if (h.bad) throw_invalid("normalize_samples: sample is not finite");
    double g;
    std::memcpy(&g, &h.gamma_bits, 8);
    ax.gamma_raw = g;
    ax.gamma = snap_gamma(g, (double)grid);
}

void assign_frequencies(Axis& ax, const double* omega, bool on_device, size_t n, bool upper_open,
                        cudaStream_t s) {
    ax.n = n;
    ax.grid = n;
    ax.x.alloc(8 * n);
    ax.s.alloc(8 * n);
    ax.t.alloc(8 * n);
    ax.delta.alloc(8 * n);
    DevBuf red(sizeof(Reduce), s), tmp;
    NB_CUDA(cudaMemsetAsync(red.get(), 0, sizeof(Reduce), s));
    const double* src = omega;
    if (!on_device) {
        tmp.alloc(8 * n, s);
        NB_CUDA(cudaMemcpyAsync(tmp.get(), omega, 8 * n, cudaMemcpyHostToDevice, s));
        src = tmp.as<double>();
    }
    Reduce* r = red.as<Reduce>();
    k_assign_freqs<<<blocks(n), 256, 0, s>>>(src, (long long)n, upper_open ? 1 : 0,
                                             ax.x.as<double>(), ax.s.as<long long>(),
                                             ax.t.as<long long>(), ax.delta.as<double>(),
                                             &r->gamma_bits, &r->bad);
    NB_LAUNCH();
    Reduce h{};
    NB_CUDA(cudaMemcpyAsync(&h, r, sizeof(Reduce), cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaStreamSynchronize(s));
    if (h.bad)
        throw_invalid(upper_open ? "plan_nufft3: frequency outside [0, N)"
                                 : "plan_nufft1: frequency outside [0, N]");
    double g;
    std::memcpy(&g, &h.gamma_bits, 8);
    ax.gamma_raw = g;
    ax.gamma = snap_gamma(g, (double)n);
}

void finish_core(CorePlan& p, double gamma_for_factors, cudaStream_t s) {
    (void)s;
    p.gamma_factors = gamma_for_factors;
    p.uniform = gamma_for_factors == 0.0;
    p.K = p.uniform ? 1 : select_rank(gamma_for_factors, p.epsilon);
    p.series_deg = bessel_series_degrees(gamma_for_factors, p.K);
    const size_t n = p.n;
    p.fused = is_pow2(n) && n >= 16 && n <= (size_t(1) << 24);
    if (p.fused) build_buckets(p, s);
}

// flag[0] = 1 when three consecutive sorted keys are equal (a bin with >= 3 samples)
__global__ void k_crowded_bins(const unsigned* __restrict__ skey, long long n, int* __restrict__ flag) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i + 2 < n && skey[i] == skey[i + 2]) flag[0] = 1;
}

void build_buckets(CorePlan& p, cudaStream_t s) {
    const size_t n = p.n;
    const int l = ilog2(n);
    int log_n2, log_n1;
    if (l < 8) {
        log_n1 = 0;
        log_n2 = l;
    } else {
        log_n2 = (l + 1) / 2;
        log_n1 = l - log_n2;
    }
    p.bk.log_n1 = log_n1;
    p.bk.log_n2 = log_n2;
    DevBuf keys(4 * n, s), idx(4 * n, s);
    p.bk.perm.alloc(4 * n);
    p.bk.skey.alloc(4 * n);
    DevArray& keys_out = p.bk.skey;
    k_bucket_keys<<<blocks(n), 256, 0, s>>>(p.ax.t.as<long long>(), (long long)n, log_n1, log_n2,
                                            keys.as<unsigned>(), idx.as<int>());
    NB_LAUNCH();
    size_t temp = 0;
    NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.as<unsigned>(),
                                            keys_out.as<unsigned>(), idx.as<int>(),
                                            p.bk.perm.as<int>(), (int)n, 0, l > 0 ? l : 1, s));
    DevBuf tb(temp, s);
    NB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), temp, keys.as<unsigned>(),
                                            keys_out.as<unsigned>(), idx.as<int>(),
                                            p.bk.perm.as<int>(), (int)n, 0, l > 0 ? l : 1, s));
    const size_t n1 = size_t(1) << log_n1;
    p.bk.rowoff.alloc(4 * (n1 + 1));
    k_bucket_offsets<unsigned><<<blocks(n + 1), 256, 0, s>>>(
        keys_out.as<unsigned>(), (long long)n, log_n2, (long long)n1, p.bk.rowoff.as<int>());
    NB_LAUNCH();
    p.bk.rowoff_host.resize(n1 + 1);  // row ranges -> sample ranges on the host (multi-GPU chunking)
    NB_CUDA(cudaMemcpyAsync(p.bk.rowoff_host.data(), p.bk.rowoff.as<int>(), 4 * (n1 + 1),
                            cudaMemcpyDeviceToHost, s));
    {   // bin occupancy class for the transpose core's bin sums (transpose_fused.cu)
        DevBuf flag(sizeof(int), s);
        NB_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
        k_crowded_bins<<<blocks(n), 256, 0, s>>>(keys_out.as<unsigned>(), (long long)n, flag.as<int>());
        NB_LAUNCH();
        p.bk.crowded.assign(1, 1);
        NB_CUDA(cudaMemcpyAsync(p.bk.crowded.data(), flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaStreamSynchronize(s));  // flag is released below; the plan call synchronizes anyway
    }
    p.bk.invperm.alloc(4 * n);
    k_invert_perm<<<blocks(n), 256, 0, s>>>(p.bk.perm.as<int>(), (long long)n, p.bk.invperm.as<int>());
    NB_LAUNCH();
    p.bk.xs.alloc(8 * n);
    k_gather_x<<<blocks(n), 256, 0, s>>>(p.ax.x.as<double>(), p.bk.perm.as<int>(), (long long)n,
                                         p.bk.xs.as<double>());
    NB_LAUNCH();
    p.bk.ds.alloc(8 * n);
    k_gather_x<<<blocks(n), 256, 0, s>>>(p.ax.delta.as<double>(), p.bk.perm.as<int>(), (long long)n,
                                         p.bk.ds.as<double>());
    NB_LAUNCH();
}

void build_bins(CorePlan& p, cudaStream_t s) {
    const size_t n = p.n;
    DevBuf keys(8 * n, s), keys_out(8 * n, s), idx(4 * n, s);
    p.bk.sort_perm.alloc(4 * n);
    k_plain_keys<<<blocks(n), 256, 0, s>>>(p.ax.t.as<long long>(), (long long)n,
                                           keys.as<unsigned long long>(), idx.as<int>());
    NB_LAUNCH();
    const int bits = std::max(1, ilog2(n + 1));
    size_t temp = 0;
    NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.as<unsigned long long>(),
                                            keys_out.as<unsigned long long>(), idx.as<int>(),
                                            p.bk.sort_perm.as<int>(), (int)n, 0, bits, s));
    DevBuf tb(temp, s);
    NB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), temp, keys.as<unsigned long long>(),
                                            keys_out.as<unsigned long long>(), idx.as<int>(),
                                            p.bk.sort_perm.as<int>(), (int)n, 0, bits, s));
    p.bk.bin_off.alloc(4 * (n + 1));
    k_bucket_offsets<unsigned long long><<<blocks(n + 1), 256, 0, s>>>(
        keys_out.as<unsigned long long>(), (long long)n, 0, (long long)n, p.bk.bin_off.as<int>());
    NB_LAUNCH();
    p.have_bins = true;
}

void factors_u(const double* delta_dev, size_t n, double gamma, size_t K, double2* u_dev,
               cudaStream_t s) {
    const size_t P = K + kCoefficientPadding;
    const std::vector<double> a = cheb_coefficients(gamma, P);
    DevBuf ad(8 * a.size(), s);
    NB_CUDA(cudaMemcpyAsync(ad.get(), a.data(), 8 * a.size(), cudaMemcpyHostToDevice, s));
    k_factors_u<<<blocks(n, 128), 128, 0, s>>>(delta_dev, (long long)n, gamma, (int)K, (int)P,
                                               ad.as<double>(), u_dev);
    NB_LAUNCH();
    NB_CUDA(cudaStreamSynchronize(s));  // `a` is pageable host memory
}

void factors_v(const double* omega_scaled_dev, size_t m, size_t K, double2* v_dev, cudaStream_t s) {
    DevBuf bad(4, s);
    NB_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
    k_factors_v<<<blocks(m), 256, 0, s>>>(omega_scaled_dev, (long long)m, (int)K, v_dev,
                                          bad.as<int>());
    NB_LAUNCH();
    int h = 0;
    NB_CUDA(cudaMemcpyAsync(&h, bad.get(), 4, cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaStreamSynchronize(s));
    if (h) throw_domain("cheb_eval_matrix: point outside [-1, 1]");
}

void cheb_eval(const double* pts_dev, size_t n, size_t K, double* out_dev, cudaStream_t s) {
    if (K < 1) throw_invalid("cheb_eval_matrix: K must be >= 1");
    DevBuf bad(4, s);
    NB_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
    if (n) {
        k_cheb_eval<<<blocks(n), 256, 0, s>>>(pts_dev, (long long)n, (int)K, out_dev, bad.as<int>());
        NB_LAUNCH();
    }
    int h = 0;
    NB_CUDA(cudaMemcpyAsync(&h, bad.get(), 4, cudaMemcpyDeviceToHost, s));
    NB_CUDA(cudaStreamSynchronize(s));
    if (h) throw_domain("cheb_eval_matrix: point outside [-1, 1]");
}

}  // namespace nb

namespace nb {
void build_type3_order(Plan3State& st, cudaStream_t s) {
    const size_t n = st.a.n;
    DevBuf keys(4 * n, s), keys_out(4 * n, s), flags(4 * n, s), idx(4 * n, s);
    st.ord_perm.alloc(4 * n);
    k_t3_keys<<<blocks(n), 256, 0, s>>>(st.a.ax.s.as<long long>(), st.a.ax.t.as<long long>(), (long long)n,
                                        keys.as<unsigned>(), flags.as<unsigned>(), idx.as<int>());
    NB_LAUNCH();
    const int bits = std::max(1, ilog2(n));
    size_t temp = 0;
    NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.as<unsigned>(), keys_out.as<unsigned>(),
                                            idx.as<int>(), st.ord_perm.as<int>(), (int)n, 0, bits, s));
    DevBuf tb(temp, s);
    NB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), temp, keys.as<unsigned>(), keys_out.as<unsigned>(),
                                            idx.as<int>(), st.ord_perm.as<int>(), (int)n, 0, bits, s));
    st.ord_key.alloc(4 * n);
    st.ord_delta.alloc(8 * n);
    k_t3_gather<<<blocks(n), 256, 0, s>>>(st.ord_perm.as<int>(), flags.as<unsigned>(), st.a.ax.delta.as<double>(),
                                          (long long)n, st.ord_key.as<unsigned>(), st.ord_delta.as<double>());
    NB_LAUNCH();
}
}  // namespace nb
