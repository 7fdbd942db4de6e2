// Type-I (transpose core), type-II adjoint and type-III execution.
//
// Reference: exec_transpose_core transforms.hpp:206-221
//   F2~^T g = sum_r v_r .* F^T scatter_t(u_r .* g)     (F symmetric: F^T = F)
// with duplicate bins summed in ascending sample order; exec_nufft3 :382-394
//   f = sum_{q<Kc} U_q .* gather_t(F1~(V_q .* c)),  Kc = K or 2K (wraparound B).
// Scatter determinism: samples are pre-sorted by bin t at plan time (stable
// radix sort keeps ascending j inside a bin), one thread sums one bin in that
// order — no floating-point atomics.
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

// scaled[i] = V_q(omega_i) c[i]; V_q = v^A_r(omega/N) [* exp(-2 pi i omega) for the beta family]
__global__ void k3_scale(const double2* __restrict__ c, const double* __restrict__ omega,
                         double2* __restrict__ out, long long n, int r, int phase, int uniform) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double w = omega[i];
    double vr = 1.0;
    if (!uniform) {
        const double s = __dsub_rn(__dmul_rn(2.0, __ddiv_rn(w, (double)n)), 1.0);
        vr = v_factor_from_s(fmin(1.0, fmax(-1.0, s)), r);
    }
    double2 v = make_double2(vr, 0.0);
    if (phase) {
        const double fr = w - floor(w);  // exact
        double sn, cs;
        sincospi(-2.0 * fr, &sn, &cs);
        v = make_double2(vr * cs, vr * sn);
    }
    out[i] = cmul(v, c[i]);
}

// f[j] (+)= U_q[j] y[t_j];  U_q = u^A_r(delta_j) * (1 - beta_j | beta_j | 1)
__global__ void k3_accum(const double2* __restrict__ y, double2* __restrict__ f,
                         const double* __restrict__ delta, const long long* __restrict__ s,
                         const long long* __restrict__ t, long long n, int r, int deg, int family,
                         int first, int uniform) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double2 u = uniform ? make_double2(1.0, 0.0) : u_factor(delta[j], r, deg);
    if (family) {  // 1: (1 - beta), 2: beta ; beta = (s - t)/N in {0, 1}
        const double beta = (double)(s[j] - t[j]) / (double)n;
        u = cscale(u, family == 1 ? 1.0 - beta : beta);
    }
    const double2 term = cmul(u, y[t[j]]);
    f[j] = first ? term : cadd(f[j], term);
}

}  // namespace

void conj_copy(const double2* in, double2* out, size_t n, cudaStream_t s) {
    k_conj<<<blocks(n), 256, 0, s>>>(in, out, (long long)n);
    NB_LAUNCH();
}

void exec_transpose(const CorePlan& p, const double2* g, double2* f, size_t batch,
                    cudaStream_t s) {
    if (p.fused) return exec_transpose_fused(p, g, f, batch, s);
    ensure_bessel_constants(p.device);
    if (!p.have_bins) throw Error(kInternal, "transpose core: plan has no bins");
    const size_t N = p.n;
    DevBuf bins(sizeof(double2) * N, s);
    for (size_t b = 0; b < batch; ++b) {
        for (size_t r = 0; r < p.K; ++r) {
            k1_scatter<<<blocks(N), 256, 0, s>>>(g + b * N, p.bk.sort_perm.as<int>(),
                                                 p.bk.bin_off.as<int>(), p.ax.delta.as<double>(),
                                                 bins.as<double2>(), (long long)N, (int)r,
                                                 p.series_deg[r], p.uniform ? 1 : 0);
            NB_LAUNCH();
            fft_exec(bins.as<double2>(), bins.as<double2>(), N, 1, -1, s, p.device);
            k1_accum<<<blocks(N), 256, 0, s>>>(bins.as<double2>(), f + b * N, (long long)N, (int)r,
                                               r == 0 ? 1 : 0, p.uniform ? 1 : 0);
            NB_LAUNCH();
        }
    }
}

void exec_type3(const Plan3State& p, const double2* c, double2* f, size_t batch, cudaStream_t s) {
    ensure_bessel_constants(p.a.device);
    const size_t N = p.a.n;
    const size_t K = p.a.K;
    DevBuf scaled(sizeof(double2) * N, s), y(sizeof(double2) * N, s);
    for (size_t b = 0; b < batch; ++b) {
        for (size_t q = 0; q < p.kc; ++q) {
            const size_t r = q % K;
            const bool second = q >= K;
            k3_scale<<<blocks(N), 256, 0, s>>>(c + b * N, p.omega.as<double>(), scaled.as<double2>(),
                                               (long long)N, (int)r, second ? 1 : 0,
                                               p.a.uniform ? 1 : 0);
            NB_LAUNCH();
            exec_transpose(p.inner, scaled.as<double2>(), y.as<double2>(), 1, s);
            const int family = p.btrivial ? 0 : (second ? 2 : 1);
            k3_accum<<<blocks(N), 256, 0, s>>>(y.as<double2>(), f + b * N, p.a.ax.delta.as<double>(),
                                               p.a.ax.s.as<long long>(), p.a.ax.t.as<long long>(),
                                               (long long)N, (int)r, p.a.series_deg[r], family,
                                               q == 0 ? 1 : 0, p.a.uniform ? 1 : 0);
            NB_LAUNCH();
        }
    }
}

}  // namespace nb
