// Device-resident plan state for the four transform families.
//
// HBM layout (per 1D plan of size N; bytes per sample in brackets):
//   x      normalized samples                       fp64   [8]
//   t      grid node t_j = s_j mod N                int64  [8]   (generic path, mirrors)
//   s      nearest node s_j                         int64  [8]   (mirrors, type III beta)
//   delta  exact N*x_j - s_j                        fp64   [8]   (generic path)
// fused power-of-two path (N = N1*N2, bucket = row t1 = t mod N1):
//   xs     x sorted by (t mod N1, t div N1)         fp64   [8]
//   perm   original index of each sorted sample     int32  [4]
//   rowoff N1+1 bucket offsets                       int32
//   ds     delta sorted like xs (transpose core)      fp64   [8]
//   skey   sorted bucket key (t1 << log2 N2) | t2     uint32 [4]
// The exec kernels read only xs + perm (12 B/sample) and recompute s, t,
// delta from x exactly as the reference does (transforms.hpp:60-64,84-86).
#pragma once

#include <cstdint>

#include <cstddef>
#include <memory>
#include <vector>

#include "engine.cuh"

namespace nb {

enum class AssignMode { kSamples, kFrequencies };

// One axis of nearest-node assignment (transforms.hpp:25-32, 77-102, 262-277).
struct Axis {
    size_t n = 0;           // number of samples
    size_t grid = 0;        // grid size
    DevArray x, s, t, delta;
    double gamma = 0.0;      // snapped (what plan.gamma() reports)
    double gamma_raw = 0.0;  // un-snapped max |delta| (type I passes it to the factors)
};

// Bucketing of an axis for the fused two-pass kernels.
struct Buckets {
    int log_n1 = 0, log_n2 = 0;  // N = N1*N2
    DevArray xs, perm, rowoff;   // see header comment
    DevArray invperm;            // invperm[perm[i]] = i: sample j -> its bucket-order slot
    DevArray ds, skey;           // fused transpose core (type I / adjoint / III inner)
    DevArray sort_perm;          // generic transpose core: samples sorted by t (int32)
    DevArray bin_off;            // generic transpose core: N+1 offsets (int32)
    std::vector<int> rowoff_host;  // host copy of rowoff (row chunk -> sample range)
    std::vector<int> crowded;      // [0] != 0: some bin holds three or more samples (pass A's bin-sum depth)
};

// Type-I/II core plan: a sample axis, a rank, and the factor parameters.
struct CorePlan {
    int device = 0;
    size_t n = 0;
    double epsilon = 0.0;
    Axis ax;
    size_t K = 1;
    bool uniform = true;        // gamma used for the factors == 0  ->  u = v = 1
    double gamma_factors = 0;   // gamma passed to build_factors
    std::vector<int> series_deg;  // Horner degree per r
    bool fused = false;         // power-of-two fused two-pass path
    Buckets bk;
    bool have_bins = false;     // bin_off / sort_perm built (transpose core)
    bool delta_from_freq = false;  // type-I axis: delta = omega - round(omega), not N x - s
};

struct Plan3State {
    CorePlan a;        // samples x on the N-grid, factors A (v over omega/N)
    CorePlan inner;    // type-I plan on omega
    DevArray omega;    // raw frequencies (fp64)
    bool btrivial = true;
    size_t kc = 0;
    // samples in ascending t (stable in j) for the sample-ordered epilogue of
    // exec_type3: original index, key = t | beta << 31, delta
    DevArray ord_perm, ord_key, ord_delta;
};

struct Plan2DState {
    int device = 0;
    size_t m = 0, n = 0, count = 0;
    double epsilon = 0;
    Axis ax, ay;                 // x on the n-grid, y on the m-grid
    size_t kx = 1, ky = 1;
    bool ux_uniform = true, uy_uniform = true;
    std::vector<int> deg_x, deg_y;
    DevArray flat;               // m*tx + ty (int64)
    // fused path (nufft2d_fused.cu): samples sorted by column tx (stable)
    bool fused = false;
    struct {
        DevArray perm, coloff;   // int32 original index, n+1 column offsets
        DevArray dxs, dys, tys;  // sorted delta_x, delta_y (fp64), ty (uint16)
        DevArray vyt;            // vy_r2(ky) table, ky x m (fp64)
    } fz;
};

// ---- plan construction (plan_kernels.cu) --------------------------------
// type II / III sample axis: normalize raw, assign to `grid` nodes
void assign_samples(Axis& ax, const double* raw, bool raw_on_device, size_t n, size_t grid,
                    cudaStream_t s);
// type I axis from frequencies omega in [0, N] (transforms.hpp:246-277)
void assign_frequencies(Axis& ax, const double* omega, bool on_device, size_t n, bool upper_open,
                        cudaStream_t s);
void finish_core(CorePlan& p, double gamma_for_factors, cudaStream_t s);
void build_buckets(CorePlan& p, cudaStream_t s);
void build_bins(CorePlan& p, cudaStream_t s);
// Plan3State::ord_* from a's samples (type-III epilogue order)
void build_type3_order(Plan3State& st, cudaStream_t s);

// materialize the reference-form factors u (K x n) and v (K x m) on the device
void factors_u(const double* delta_dev, size_t n, double gamma, size_t K, double2* u_dev,
               cudaStream_t s);
void factors_v(const double* omega_scaled_dev, size_t m, size_t K, double2* v_dev, cudaStream_t s);
void cheb_eval(const double* pts_dev, size_t n, size_t K, double* out_dev, cudaStream_t s);

// ---- execution (nufft2.cu, nufft1.cu, nufft3.cu, nufft2d.cu) -------------
// ev (optional): 3 events recorded before pass 1, between the passes, after
// pass 2 (batch 1) — per-kernel timing on the launching stream for the bench
void exec_type2(const CorePlan& p, const double2* c, double2* f, size_t batch, size_t r0,
                size_t r1, cudaStream_t s, cudaEvent_t* ev = nullptr);
// building blocks of the multi-GPU r-split (nufft2_multi.cu), fused plans with
// N1 > 1 only: pass 1 of terms [r0, r1) into Y (16 (r1 - r0) N bytes), and
// pass 2 over rows [row0, row1) writing the partial sum either to f[perm]
// (natural order) or, sorted_out, to fs[i] in bucket order (rowoff ranges)
void exec_type2_pass1(const CorePlan& p, const double2* c, double2* Y, size_t r0, size_t r1,
                      cudaStream_t s);
void exec_type2_pass2_rows(const CorePlan& p, const double2* Y, double2* f, size_t r0, size_t r1,
                           long long row0, long long row1, bool sorted_out, cudaStream_t s);
// f[j] = fs[invperm[j]] (bucket order -> natural order; coalesced f writes), batch vectors of N
void unpermute(const CorePlan& p, const double2* fs, double2* f, size_t batch, cudaStream_t s);
// F2~^T g = sum_r v_r .* F scatter_t(u_r .* g)   (transforms.hpp:206-221)
void exec_transpose(const CorePlan& p, const double2* g, double2* f, size_t batch,
                    cudaStream_t s, size_t r_begin = 0, size_t r_end = SIZE_MAX);
// fused two-pass form of exec_transpose for power-of-two N (transpose_fused.cu);
// ev as for exec_type2
// conj: transform conj(g) and write conj(f) (the adjoints, with no separate conjugation passes)
void exec_transpose_fused(const CorePlan& p, const double2* g, double2* f, size_t batch,
                          cudaStream_t s, cudaEvent_t* ev = nullptr, size_t r_begin = 0,
                          size_t r_end = SIZE_MAX, bool conj = false);
void exec_type3(const Plan3State& p, const double2* c, double2* f, size_t batch, cudaStream_t s,
                size_t r_begin = 0, size_t r_end = SIZE_MAX);
void exec_2d(const Plan2DState& p, const double2* C, double2* f, size_t batch, bool reuse_rows,
             cudaStream_t s);

// ---- inverse (inverse.cu): Toeplitz operator in its 2N circulant embedding
struct ToeplitzState {
    int device = 0;
    size_t n = 0;
    DevArray spectrum;   // 2n doubles: Re(FFT_2n(symbol)) (inverse.hpp:37-50)
    DevArray first_col;  // n complex
};
struct CgResult {
    size_t iterations = 0;
    double relative_residual = 0.0;
    bool converged = false;
};
void toeplitz_from_column(ToeplitzState& op, const double2* col_dev, cudaStream_t s);
void toeplitz_matvec(const ToeplitzState& op, const double2* v, double2* out, cudaStream_t s);
CgResult cg_solve_toeplitz(const ToeplitzState& op, const double2* rhs, double2* x, double tol,
                           size_t max_iter, std::vector<double>* history, cudaStream_t s);
size_t default_cg_max_iter(size_t n);

// ---- direct sums (direct.cu): oracle.hpp:70-107 on the device
void nudft_direct(const double* x, size_t nx, const double* w, const double2* c, size_t n, double2* f,
                  cudaStream_t s);
void nudft2d_direct(const double* x, const double* y, size_t cnt, const double2* C, size_t m, size_t n,
                    double2* f, cudaStream_t s);

bool fused_2d_eligible(size_t m, size_t n, size_t count);
void build_2d_fused(Plan2DState& st, cudaStream_t s);
void exec_2d_fused(const Plan2DState& st, const double2* C, double2* f, size_t batch, cudaStream_t s,
                   size_t r1_begin = 0, size_t r1_end = SIZE_MAX);

// elementwise helpers shared by the generic paths (generic_kernels.cu)
void conj_copy(const double2* in, double2* out, size_t n, cudaStream_t s);

}  // namespace nb
