// 2D type-II execution (tensor-product low-rank form).
//
// Reference: exec_nufft2d2_impl transform2d.hpp:107-140
//   f_j = sum_{r1,r2} ux_r1[j] uy_r2[j] [F_m D_vy_r2 C D_vx_r1 F_n^T](ty_j, tx_j)
// with the row stage (C D_vx F_n^T, m FFTs of size n) computed once per r1
// and reused for every r2 (n column FFTs of size m each).  The row stage is
// kept TRANSPOSED in HBM (n x m), so every column FFT is a contiguous batch
// and the gather index is exactly the reference's flatIndex = m*tx + ty
// (transform2d.hpp:89-91).
#include "bessel.cuh"
#include "plans.hpp"

namespace nb {

namespace {

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// rs[r][c] = C[r][c] * vx_r1(c/n)
__global__ void k2d_colscale(const double2* __restrict__ C, double2* __restrict__ rs, long long m,
                             long long n, int r1, int uniform) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m * n) return;
    const long long c = i % n;
    const double v = uniform ? 1.0 : v_factor_from_s(grid_s(c, n), r1);
    const double2 z = C[i];
    rs[i] = make_double2(z.x * v, z.y * v);
}

// full[c][r] = rsT[c][r] * vy_r2(r/m)   (transposed layout, rows of length m)
__global__ void k2d_rowscale(const double2* __restrict__ rsT, double2* __restrict__ full,
                             long long m, long long n, int r2, int uniform) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m * n) return;
    const long long r = i % m;
    const double v = uniform ? 1.0 : v_factor_from_s(grid_s(r, m), r2);
    const double2 z = rsT[i];
    full[i] = make_double2(z.x * v, z.y * v);
}

// f[j] (+)= (ux_r1[j] * uy_r2[j]) * fullT[flat_j]
__global__ void k2d_accum(const double2* __restrict__ fullT, double2* __restrict__ f,
                          const double* __restrict__ dx, const double* __restrict__ dy,
                          const long long* __restrict__ flat, long long count, int r1, int degx,
                          int ux_uniform, int r2, int degy, int uy_uniform, int first) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= count) return;
    const double2 ux = ux_uniform ? make_double2(1.0, 0.0) : u_factor(dx[j], r1, degx);
    const double2 uy = uy_uniform ? make_double2(1.0, 0.0) : u_factor(dy[j], r2, degy);
    const double2 term = cmul(cmul(ux, uy), fullT[flat[j]]);
    f[j] = first ? term : cadd(f[j], term);
}

}  // namespace

void exec_2d(const Plan2DState& p, const double2* C, double2* f, size_t batch, bool reuse_rows,
             cudaStream_t s) {
    if (p.fused) {
        exec_2d_fused(p, C, f, batch, s);
        for (size_t b = 0; b < batch; ++b) {  // logical transform counts as the reference
            fft_count(p.n, p.m * p.kx * (reuse_rows ? 1 : p.ky));
            fft_count(p.m, p.n * p.kx * p.ky);
        }
        return;
    }
    ensure_bessel_constants(p.device);
    const size_t m = p.m, n = p.n, mn = m * n, count = p.count;
    DevBuf rs(sizeof(double2) * mn, s), rsT(sizeof(double2) * mn, s), full(sizeof(double2) * mn, s);
    auto row_stage = [&](const double2* Cb, size_t r1) {
        k2d_colscale<<<blocks(mn), 256, 0, s>>>(Cb, rs.as<double2>(), (long long)m, (long long)n,
                                                (int)r1, p.ux_uniform ? 1 : 0);
        NB_LAUNCH();
        fft_exec(rs.as<double2>(), rs.as<double2>(), n, m, -1, s, p.device);  // m FFTs of size n
        fft_count(n, m);
        transpose(rs.as<double2>(), rsT.as<double2>(), m, n, 1, s);
    };
    for (size_t b = 0; b < batch; ++b) {
        const double2* Cb = C + b * mn;
        double2* fb = f + b * count;
        bool first = true;
        for (size_t r1 = 0; r1 < p.kx; ++r1) {
            if (reuse_rows) row_stage(Cb, r1);
            for (size_t r2 = 0; r2 < p.ky; ++r2) {
                if (!reuse_rows) row_stage(Cb, r1);
                k2d_rowscale<<<blocks(mn), 256, 0, s>>>(rsT.as<double2>(), full.as<double2>(),
                                                        (long long)m, (long long)n, (int)r2,
                                                        p.uy_uniform ? 1 : 0);
                NB_LAUNCH();
                fft_exec(full.as<double2>(), full.as<double2>(), m, n, -1, s, p.device);  // n FFTs of size m
                fft_count(m, n);
                k2d_accum<<<blocks(count), 256, 0, s>>>(
                    full.as<double2>(), fb, p.ax.delta.as<double>(), p.ay.delta.as<double>(),
                    p.flat.as<long long>(), (long long)count, (int)r1, p.deg_x[r1],
                    p.ux_uniform ? 1 : 0, (int)r2, p.deg_y[r2], p.uy_uniform ? 1 : 0, first ? 1 : 0);
                NB_LAUNCH();
                first = false;
            }
        }
    }
}

}  // namespace nb
