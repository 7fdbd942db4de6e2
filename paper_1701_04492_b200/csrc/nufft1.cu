// Type-I (transpose core), type-II adjoint and type-III execution.
//
// Reference: exec_transpose_core transforms.hpp:206-221
//   F2~^T g = sum_r v_r .* F^T scatter_t(u_r .* g)     (F symmetric: F^T = F)
// with duplicate bins summed in ascending sample order; exec_nufft3 :382-394
//   f = sum_{q<Kc} U_q .* gather_t(F1~(V_q .* c)),  Kc = K or 2K (wraparound B).
// Scatter determinism: samples are pre-sorted by bin t at plan time (stable
// radix sort keeps ascending j inside a bin), one thread sums one bin in that
// order — no floating-point atomics.
#include <algorithm>

#include "bessel.cuh"
#include "plans.hpp"

namespace nb {

namespace {

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// bins[t] = sum_{j: t_j = t} u_r[j] g[j], ascending j
__global__ void k1_scatter(const double2* __restrict__ g, const int* __restrict__ sort_perm,
                           const int* __restrict__ bin_off, const double* __restrict__ delta,
                           double2* __restrict__ bins, long long n, int r, int deg, int uniform) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = bin_off[t]; i < bin_off[t + 1]; ++i) {
        const int j = sort_perm[i];
        const double2 gj = g[j];
        acc = cadd(acc, uniform ? gj : cmul(u_factor(delta[j], r, deg), gj));
    }
    bins[t] = acc;
}

// f[k] (+)= v_r(k) X[k]
__global__ void k1_accum(const double2* __restrict__ X, double2* __restrict__ f, long long n, int r,
                         int first, int uniform) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double vr = uniform ? 1.0 : v_factor_from_s(grid_s(k, n), r);
    const double2 x = X[k];
    const double2 term = make_double2(x.x * vr, x.y * vr);
    f[k] = first ? term : cadd(f[k], term);
}

__global__ void k_conj(const double2* __restrict__ in, double2* __restrict__ out, long long n) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = cconj(in[i]);
}

// scaled[i] = v^A_r(omega_i / N) c[i]   (the first family's V_r, transforms.hpp:337-340)
__global__ void k3_scale(const double2* __restrict__ c, const double* __restrict__ omega,
                         double2* __restrict__ out, long long n, int r, int uniform) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double vr = 1.0;
    if (!uniform) {
        const double s = __dsub_rn(__dmul_rn(2.0, __ddiv_rn(omega[i], (double)n)), 1.0);
        vr = v_factor_from_s(fmin(1.0, fmax(-1.0, s)), r);
    }
    const double2 x = c[i];
    out[i] = make_double2(vr * x.x, vr * x.y);
}

// The beta family of a non-trivial B (transforms.hpp:355-370): only samples with
// beta_j = 1 see it, and for those t_j = 0, so the inner type-I output is needed at
// index 0 only, where every phase exp(-2 pi i 0 omega_k / N) is exactly 1:
//     D_r = sum_k v^A_r(omega_k / N) exp(-2 pi i omega_k) c_k,   r < K
// (SURVEY.md §8(a18)).  Stage 1: each block sums a strided slice of k for terms
// [r0, r0 + 8) into part[block][r]; stage 2 adds the blocks in index order —
// a fixed summation order, so D is bit-reproducible.
constexpr int kDotTerms = 8;
constexpr int kDotBlocks = 592;  // 4 x 148 SMs
constexpr int kDotThreads = 256;
__global__ void __launch_bounds__(kDotThreads)
    k3_beta_dot_part(const double2* __restrict__ c, const double* __restrict__ omega, long long n, int r0,
                     int nr, int uniform, double2* __restrict__ part) {
    __shared__ double2 red[kDotTerms][kDotThreads];
    double2 acc[kDotTerms];
#pragma unroll
    for (int q = 0; q < kDotTerms; ++q) acc[q] = make_double2(0.0, 0.0);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const double w = omega[k];
        double sn, cs;
        sincospi(-2.0 * (w - floor(w)), &sn, &cs);  // exp(-2 pi i omega), argument reduced exactly
        const double2 ec = cmul(make_double2(cs, sn), c[k]);
        // v_r for r = r0 .. r0 + nr - 1 by the recurrence from T_0, T_1
        const double s = fmin(1.0, fmax(-1.0, __dsub_rn(__dmul_rn(2.0, __ddiv_rn(w, (double)n)), 1.0)));
        double tm1 = 1.0, t = s;
        for (int r = 1; r < r0; ++r) {
            const double tn = __fma_rn(2.0 * s, t, -tm1);
            tm1 = t;
            t = tn;
        }
#pragma unroll
        for (int q = 0; q < kDotTerms; ++q) {
            const int r = r0 + q;
            if (q < nr) {
                const double vr = uniform ? 1.0 : (r == 0 ? 0.5 : t);
                acc[q].x = __fma_rn(vr, ec.x, acc[q].x);
                acc[q].y = __fma_rn(vr, ec.y, acc[q].y);
                if (r >= 1) {
                    const double tn = __fma_rn(2.0 * s, t, -tm1);
                    tm1 = t;
                    t = tn;
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kDotTerms; ++q) red[q][threadIdx.x] = acc[q];
    __syncthreads();
    for (int half = kDotThreads / 2; half > 0; half >>= 1) {
        if (threadIdx.x < half)
#pragma unroll
            for (int q = 0; q < kDotTerms; ++q) red[q][threadIdx.x] = cadd(red[q][threadIdx.x], red[q][threadIdx.x + half]);
        __syncthreads();
    }
    if (threadIdx.x < nr) part[(long long)blockIdx.x * kDotTerms + threadIdx.x] = red[threadIdx.x][0];
}
// stage 2: one warp per term; lane l adds the blocks b = l, l + 32, ... in ascending order and
// the lanes are combined by a fixed xor tree — a fixed order, so D is bit-reproducible.  (One
// thread per term walking the 592 partials took ~0.12 ms per launch: dependent-latency bound.)
__global__ void __launch_bounds__(32 * kDotTerms)
    k3_beta_dot_final(const double2* __restrict__ part, int r0, int nr, double2* __restrict__ D) {
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (q >= nr) return;
    double2 s = make_double2(0.0, 0.0);
    for (int b = lane; b < kDotBlocks; b += 32) s = cadd(s, part[(long long)b * kDotTerms + q]);
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, m);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, m);
    }
    if (lane == 0) D[r0 + q] = s;
}

// f[j] = sum_r u^A_r(delta_j) Z_r,j with Z_r,j = y_r[t_j] (beta_j = 0) or D_r
// (beta_j = 1) — both families and the K per-term accumulations of the
// reference's exec_nufft3 (transforms.hpp:386-392) in one pass over the samples
// in ascending t (plan order, Plan3State::ord_*), so consecutive threads read
// neighbouring y_r[t] and only f[j] is scattered.
// u_r = 2 exp(2ih) (ih)^r g_r(h^2): Horner in r over acc <- acc (ih) + g_r Z_r,
// g_r by the backward Bessel recurrence g_{r-1} = r g_r - w g_{r+1} from two
// series values (as in the type-II pass 2, nufft2.cu).
__global__ void k3_epilogue(const double2* __restrict__ Y, const double2* __restrict__ D,
                            const int* __restrict__ ord_perm, const unsigned* __restrict__ ord_key,
                            const double* __restrict__ ord_delta, long long n, int r0, int r1, int deg_top0,
                            int deg_top1, int uniform, double2* __restrict__ f) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned key = ord_key[i];
    const long long t = key & 0x7fffffffu;
    const bool beta = (key >> 31) != 0;  // s = N, t = 0: the node at 1 (transforms.hpp:345-350)
    const int j = ord_perm[i];
    if (uniform) {  // K = 1, u = v = 1
        f[j] = beta ? D[0] : Y[t];
        return;
    }
    // Y holds the terms [r0, r1) (slice r - r0); D is indexed by the absolute r
    const double h = half_phase(ord_delta[i]);
    const double w = h * h;
    double g1 = bessel_g_rt(r1, deg_top1, w);      // g_{r1}
    double g0 = bessel_g_rt(r1 - 1, deg_top0, w);  // g_{r1-1}
    double2 acc = make_double2(0.0, 0.0);
    for (int r = r1 - 1; r >= r0; --r) {
        const double2 z = beta ? D[r] : __ldg(Y + (long long)(r - r0) * n + t);
        const double ax = acc.x;
        acc.x = __fma_rn(g0, z.x, -h * acc.y);
        acc.y = __fma_rn(g0, z.y, h * ax);
        const double gm1 = __fma_rn((double)r, g0, -w * g1);  // g_{r-1}
        g1 = g0;
        g0 = gm1;
    }
    if (r0 > 0) {  // a partial term range (multi-GPU): restore (ih)^r0
        double hr = 1.0;
        for (int m = 0; m < r0; ++m) hr *= h;
        acc = cscale(acc, hr);
        switch (r0 & 3) {
            case 1: acc = make_double2(-acc.y, acc.x); break;
            case 2: acc = make_double2(-acc.x, -acc.y); break;
            case 3: acc = make_double2(acc.y, -acc.x); break;
            default: break;
        }
    }
    double sn, cs;
    sincos(2.0 * h, &sn, &cs);
    __stcs(f + j, cmul(make_double2(2.0 * cs, 2.0 * sn), acc));
}

}  // namespace

void conj_copy(const double2* in, double2* out, size_t n, cudaStream_t s) {
    k_conj<<<blocks(n), 256, 0, s>>>(in, out, (long long)n);
    NB_LAUNCH();
}

void exec_transpose(const CorePlan& p, const double2* g, double2* f, size_t batch,
                    cudaStream_t s, size_t r_begin, size_t r_end) {
    if (p.fused) return exec_transpose_fused(p, g, f, batch, s, nullptr, r_begin, r_end);
    ensure_bessel_constants(p.device);
    if (!p.have_bins) throw Error(kInternal, "transpose core: plan has no bins");
    const size_t N = p.n;
    DevBuf bins(sizeof(double2) * N, s);
    const size_t r1 = std::min(r_end, p.K);
    if (r1 <= r_begin) {
        NB_CUDA(cudaMemsetAsync(f, 0, sizeof(double2) * N * batch, s));
        return;
    }
    for (size_t b = 0; b < batch; ++b) {
        for (size_t r = r_begin; r < r1; ++r) {
            k1_scatter<<<blocks(N), 256, 0, s>>>(g + b * N, p.bk.sort_perm.as<int>(),
                                                 p.bk.bin_off.as<int>(), p.ax.delta.as<double>(),
                                                 bins.as<double2>(), (long long)N, (int)r,
                                                 p.series_deg[r], p.uniform ? 1 : 0);
            NB_LAUNCH();
            fft_exec(bins.as<double2>(), bins.as<double2>(), N, 1, -1, s, p.device);
            k1_accum<<<blocks(N), 256, 0, s>>>(bins.as<double2>(), f + b * N, (long long)N, (int)r,
                                               r == r_begin ? 1 : 0, p.uniform ? 1 : 0);
            NB_LAUNCH();
        }
    }
}

void exec_type3(const Plan3State& p, const double2* c, double2* f, size_t batch, cudaStream_t s, size_t r_begin,
                size_t r_end) {
    ensure_bessel_constants(p.a.device);
    const size_t N = p.a.n;
    const size_t K = p.a.K;
    const size_t r0 = r_begin, r1 = std::min(r_end, K);
    if (r1 <= r0) {
        NB_CUDA(cudaMemsetAsync(f, 0, sizeof(double2) * N * batch, s));
        return;
    }
    const size_t nt = r1 - r0;
    const int uni = p.a.uniform ? 1 : 0;
    // y_r = F1~(v_r .* c) for the first family (the inner type-I transforms of terms
    // [r0, r1)), kept for the single sample-ordered epilogue; the beta family reduces to
    // dot products (D_r) whenever B is non-trivial
    // the inner transforms go to the transpose core kGroup at a time (one stacked pass-A launch
    // per group when the row FFT is 2048 points, transpose_fused.cu)
    constexpr size_t kGroup = 4;
    DevBuf scaled(sizeof(double2) * N * kGroup, s), Y(sizeof(double2) * N * nt, s), D(sizeof(double2) * K, s);
    DevBuf part(p.btrivial ? 16 : sizeof(double2) * kDotBlocks * kDotTerms, s);
    const int deg0 = bessel_series_degree_rel(p.a.gamma_factors, (int)r1 - 1);
    const int deg1 = bessel_series_degree_rel(p.a.gamma_factors, (int)r1);
    for (size_t b = 0; b < batch; ++b) {
        const double2* cb = c + b * N;
        for (size_t g0 = r0; g0 < r1; g0 += kGroup) {
            const size_t ng = std::min(kGroup, r1 - g0);
            for (size_t r = g0; r < g0 + ng; ++r) {
                k3_scale<<<blocks(N), 256, 0, s>>>(cb, p.omega.as<double>(), scaled.as<double2>() + (r - g0) * N,
                                                   (long long)N, (int)r, uni);
                NB_LAUNCH();
            }
            exec_transpose(p.inner, scaled.as<double2>(), Y.as<double2>() + (g0 - r0) * N, ng, s);
        }
        if (!p.btrivial) {
            for (size_t q0 = r0; q0 < r1; q0 += kDotTerms) {
                const int nr = (int)std::min<size_t>(kDotTerms, r1 - q0);
                k3_beta_dot_part<<<kDotBlocks, kDotThreads, 0, s>>>(cb, p.omega.as<double>(), (long long)N, (int)q0,
                                                                     nr, uni, part.as<double2>());
                NB_LAUNCH();
                k3_beta_dot_final<<<1, 32 * kDotTerms, 0, s>>>(part.as<double2>(), (int)q0, nr, D.as<double2>());
                NB_LAUNCH();
            }
        } else {
            NB_CUDA(cudaMemsetAsync(D.get(), 0, sizeof(double2) * K, s));
        }
        k3_epilogue<<<blocks(N), 256, 0, s>>>(Y.as<double2>(), D.as<double2>(), p.ord_perm.as<int>(),
                                              p.ord_key.as<unsigned>(), p.ord_delta.as<double>(), (long long)N,
                                              (int)r0, (int)r1, deg0, deg1, uni, f + b * N);
        NB_LAUNCH();
    }
}

}  // namespace nb
