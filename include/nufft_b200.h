/* nufft_b200.h — C-ABI of the B200-native low-rank NUFFT (arXiv:1701.04492).
 *
 * This is the drop-in boundary for the reference's hot path.  Every entry
 * point replaces one reference C++ function (cited below, paths relative to
 * proj/include/nufft/ of the reference); the header-only C++ layer in
 * include/nufft/*.hpp re-exposes them under the reference's own names and
 * signatures, and INTEGRATION.md shows the binding a maintainer would add.
 *
 * Conventions
 *   - complex values are interleaved (re, im) doubles, byte-compatible with
 *     std::complex<double> / cuDoubleComplex (fft.hpp:22-23);
 *   - *_host entry points take host pointers and do the host<->device copies;
 *     the others take device pointers and a cudaStream_t passed as void*
 *     (NULL = the calling thread's default stream);
 *   - every function returns a status code; nufft_last_error() returns the
 *     calling thread's message.  The C++ layer maps INVALID_ARGUMENT to
 *     std::invalid_argument and DOMAIN_ERROR to std::domain_error, matching
 *     the reference's exception types (SURVEY.md §8b "Errors");
 *   - plans are immutable after creation and may be executed concurrently from
 *     several host threads (transforms_test.cpp:225-241); results are
 *     bit-identical across repeated executions (transforms_test.cpp:183-195).
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns NUFFT_CUDA_ERROR.
 */
#ifndef NUFFT_B200_H
#define NUFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NUFFT_B200_ABI_VERSION 1

enum nufft_status {
    NUFFT_OK = 0,
    NUFFT_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    NUFFT_DOMAIN_ERROR = 2,     /* std::domain_error in the reference */
    NUFFT_CUDA_ERROR = 3,
    NUFFT_NCCL_ERROR = 4,
    NUFFT_OUT_OF_MEMORY = 5,
    NUFFT_INTERNAL = 6
};

typedef struct nufft_plan2 nufft_plan2;   /* Plan2  transforms.hpp:105-114 */
typedef struct nufft_plan1 nufft_plan1;   /* Plan1  transforms.hpp:237-244 */
typedef struct nufft_plan3 nufft_plan3;   /* Plan3  transforms.hpp:308-319 */
typedef struct nufft_plan2d nufft_plan2d; /* Plan2D transform2d.hpp:51-59 */

/* Scalar plan properties callers read (SURVEY.md §8b "Plan members"). */
typedef struct nufft_plan_info {
    size_t n;              /* samples (1D: also the number of frequencies)      */
    size_t rank;           /* K; plan3: factorsA.rank; 2D: rank_x()             */
    size_t rank2;          /* plan3: inner (type-I) rank; 2D: rank_y()          */
    size_t effective_rank; /* plan3: effective_rank() (K or 2K); else rank     */
    double gamma;          /* samples.gamma (snapped); 2D: grid.gammaX          */
    double gamma2;         /* plan3: inner gamma; 2D: grid.gammaY               */
    double epsilon;
    int btrivial;          /* plan3: bTrivial                                    */
    size_t m, ncols;       /* 2D grid: m rows (y axis), n columns (x axis)      */
    int device;
    int path;              /* 0 generic term loop, 1 fused two-pass (power of two) */
} nufft_plan_info;

const char* nufft_last_error(void);
int nufft_abi_version(void);
int nufft_device_count(int* count);

/* ------------------------------------------------------------- special.hpp */
int nufft_lambert_w(double x, double* out);                 /* special.hpp:15-31 */
int nufft_bessel_j_int(int order, double z, double* out);   /* special.hpp:56-61 */
int nufft_bessel_j_signed(int order, double z, double* out);/* special.hpp:64-68 */

/* ------------------------------------------------------------- lowrank.hpp */
int nufft_select_rank(double gamma, double epsilon, size_t* rank);        /* lowrank.hpp:95-119 */
/* a: K*K complex, row-major a[p*K + r]                                        lowrank.hpp:36-65 */
int nufft_cheb_coefficients(double gamma, size_t K, double* a);
/* out: n*K row-major T_0..T_{K-1}(points[j]) (device-evaluated)               lowrank.hpp:126-143 */
int nufft_cheb_eval_matrix(const double* points, size_t n, size_t K, double* out);
/* Rank-K factors of A_jk = exp(-2 pi i delta_j omega_k)                         lowrank.hpp:161-210
 * Call with u = v = NULL to query *rank; then u: rank*n complex (row r at u + 2*r*n),
 * v: rank*m complex.  Evaluated on the device.                                                 */
int nufft_build_factors(const double* delta, size_t n, double gamma, const double* omega_scaled,
                        size_t m, double epsilon, size_t* rank, double* u, double* v);

/* ------------------------------------------------------------- fft.hpp */
int nufft_fft_forward_host(const double* in, double* out, size_t n);      /* fft.hpp:140-145 */
int nufft_fft_inverse_host(const double* in, double* out, size_t n);      /* fft.hpp:148-156 */
int nufft_fft_2d_forward_host(const double* in, double* out, size_t rows, size_t cols); /* :185-193 */
int nufft_fft_cols_forward_host(double* inout, size_t rows, size_t cols); /* fft.hpp:170-178 */
int nufft_fft_rows_forward_host(double* inout, size_t rows, size_t cols); /* fft.hpp:161-167 */
/* batch contiguous transforms of length n on the device; sign -1 forward, +1 backward (raw) */
int nufft_fft_exec(const double* in_dev, double* out_dev, size_t n, size_t batch, int sign,
                   void* stream);
uint64_t nufft_fft_exec_count(size_t n);                                  /* fft.hpp:126-132 */
void nufft_fft_reset_exec_counts(void);                                   /* fft.hpp:134-137 */
/* number of CUDA kernels this library has launched (benchmark evidence) */
uint64_t nufft_kernel_launch_count(void);

/* ---- seeded sampler: GaussianSampler, random.hpp:14-60 (host-only) --------
 * mt19937_64, uniform = (draw >> 11) * 2^-53, Box-Muller normals in pairs;
 * the same seed gives the reference's x and c bit for bit.                    */
typedef struct nufft_sampler nufft_sampler;
int nufft_sampler_create(uint64_t seed, nufft_sampler** out);           /* GaussianSampler(seed)  :16  */
void nufft_sampler_destroy(nufft_sampler* s);
double nufft_sampler_normal(nufft_sampler* s);                          /* operator()             :18-34 */
double nufft_sampler_uniform(nufft_sampler* s);                         /* uniform()              :36-38 */
int nufft_sampler_uniform_vector(nufft_sampler* s, size_t n, double lo, double hi,
                                 double* out);                          /* uniform_vector         :50-54 */
int nufft_sampler_complex_vector(nufft_sampler* s, size_t n, double* out); /* complex_vector (re, im) :40-48 */

/* ------------------------------------------------------------- samples */
int nufft_normalize_samples(const double* raw, size_t n, double* out);    /* transforms.hpp:35-45 */
int nufft_grid_assign(const double* x, size_t n, size_t grid, long* s, size_t* t,
                      double* gamma);                                     /* transforms.hpp:77-92 */

/* ------------------------------------------------------------- type II */
int nufft_plan2_create(const double* x_raw, size_t n, double epsilon, int device,
                       nufft_plan2** out);                                /* transforms.hpp:133-147 */
int nufft_plan2_create_device(const double* x_raw_dev, size_t n, double epsilon, int device,
                              nufft_plan2** out);
void nufft_plan2_destroy(nufft_plan2* plan);
int nufft_plan2_info(const nufft_plan2* plan, nufft_plan_info* info);
/* host mirrors of SampleSet x, s, t (transforms.hpp:25-32)                          */
int nufft_plan2_samples(const nufft_plan2* plan, double* x, long* s, size_t* t);
/* host copies of factors.u / factors.v (K*n complex each), reference Chebyshev form */
int nufft_plan2_factors(const nufft_plan2* plan, double* u, double* v);
/* f = sum_{r<K} diag(u_r) P_t F diag(v_r) c for `batch` vectors (device pointers)   transforms.hpp:168-199 */
int nufft_plan2_exec(const nufft_plan2* plan, const double* c_dev, double* f_dev, size_t batch,
                     void* stream);
/* partial sum over r in [r_begin, r_end) — the unit of r-term sharding across GPUs */
int nufft_plan2_exec_terms(const nufft_plan2* plan, const double* c_dev, double* f_dev,
                           size_t batch, size_t r_begin, size_t r_end, void* stream);
int nufft_plan2_exec_host(const nufft_plan2* plan, const double* c, size_t len, double* f,
                          size_t batch);

/* ---- multi-GPU type II: the rank-K sum split across GPUs --
 * Replaces the reference's threaded exec (exec_nufft2 with threads > 1,
 * transforms.hpp:174-197: contiguous r-ranges per worker, partials merged):
 * one process per GPU, an NCCL communicator between them.  Rank g evaluates
 * terms [K g/G, K (g+1)/G) (nufft_multi_term_range), pass 2 writes its partial
 * in bucket order in row chunks, and each chunk is summed (fp64) on the
 * communicator's stream while the next one is computed; the receiving ranks
 * un-permute once.  NCCL is loaded at run time (libnufft_b200.so does not link
 * it).  Every rank passes the same c (device pointer, batch vectors of N);
 * f receives the full transform on `root` (NUFFT_MULTI_REDUCE) or on every
 * rank (NUFFT_MULTI_ALLREDUCE).  Ordered on `stream`.                          */
typedef struct nufft_comm nufft_comm;
#define NUFFT_UNIQUE_ID_BYTES 128
enum nufft_multi_mode { NUFFT_MULTI_REDUCE = 0, NUFFT_MULTI_ALLREDUCE = 1 };
int nufft_comm_unique_id(unsigned char* id);  /* ncclGetUniqueId; id: NUFFT_UNIQUE_ID_BYTES bytes */
int nufft_comm_init(const unsigned char* id, int nranks, int rank, int device, nufft_comm** out);
int nufft_comm_wrap(void* nccl_comm, int device, nufft_comm** out); /* adopt a caller-owned ncclComm_t */
void nufft_comm_destroy(nufft_comm* comm);
int nufft_comm_info(const nufft_comm* comm, int* nranks, int* rank, int* device);
int nufft_multi_term_range(size_t K, int nranks, int rank, size_t* r_begin, size_t* r_end); /* host-only */
int nufft_plan2_exec_multi(const nufft_plan2* plan, const double* c_dev, double* f_dev, size_t batch,
                           nufft_comm* comm, int root, int mode, void* stream);
/* host pointers (f written on the receiving ranks only; pageable memory is staged) */
int nufft_plan2_exec_multi_host(const nufft_plan2* plan, const double* c, size_t len, double* f, size_t batch,
                                nufft_comm* comm, int root, int mode);
/* Type I (the transpose core) over G GPUs: rank g evaluates terms [K g/G, K (g+1)/G)
 * (both passes) and the partial f are summed (one reduce at the end; pass B writes f by
 * columns).  exec_terms: one rank's partial, for callers with their own collective.     */
int nufft_plan1_exec_terms(const nufft_plan1* plan, const double* c_dev, double* f_dev, size_t batch,
                           size_t r_begin, size_t r_end, void* stream);
int nufft_plan1_exec_multi(const nufft_plan1* plan, const double* c_dev, double* f_dev, size_t batch,
                           nufft_comm* comm, int root, int mode, void* stream);
/* Type III over G GPUs: rank g takes the outer terms [K g/G, K (g+1)/G) (inner type-I
 * transforms, beta dot products, the partial epilogue) and the partial f are summed.   */
int nufft_plan3_exec_terms(const nufft_plan3* plan, const double* c_dev, double* f_dev, size_t batch,
                           size_t r_begin, size_t r_end, void* stream);
int nufft_plan3_exec_multi(const nufft_plan3* plan, const double* c_dev, double* f_dev, size_t batch,
                           nufft_comm* comm, int root, int mode, void* stream);
/* 2D over G GPUs: rank g takes the row-stage terms r1 in [Kx g/G, Kx (g+1)/G) (its row stage
 * and its Kx/G x Ky column steps) and the partial f are summed (fused plans: power-of-two
 * m, n in [16, 4096]; other plans run whole on the root).                                  */
int nufft_plan2d2_exec_terms(const nufft_plan2d* plan, const double* C_dev, double* f_dev, size_t batch,
                             size_t r1_begin, size_t r1_end, void* stream);
int nufft_plan2d2_exec_multi(const nufft_plan2d* plan, const double* C_dev, double* f_dev, size_t batch,
                             nufft_comm* comm, int root, int mode, void* stream);
/* The pieces exec_multi is built from, for callers that bring their own
 * collective (e.g. torch.distributed): the partial over terms [r_begin, r_end)
 * of one vector in bucket order, the bucket-order ranges of the row chunks
 * exec_multi reduces one at a time (offsets[0..nchunks]), and the final
 * bucket-order -> natural-order permutation f[perm[i]] = fs[i].  Fused plans
 * (power-of-two N >= 256) only.                                               */
int nufft_plan2_exec_terms_sorted(const nufft_plan2* plan, const double* c_dev, double* fs_dev,
                                  size_t r_begin, size_t r_end, void* stream);
int nufft_plan2_reduce_chunks(const nufft_plan2* plan, int nchunks, size_t* offsets);
int nufft_plan2_unpermute(const nufft_plan2* plan, const double* fs_dev, double* f_dev, size_t batch,
                          void* stream);
/* exec (batch 1, fused path) recording CUDA events before pass 1, between the passes
 * and after pass 2 on `stream` into timing slot `slot` (no synchronization);
 * timing_read sums the per-pass device times of slots [0, nslots).  Used by
 * bench.py to time each kernel inside the timed region for the roofline line. */
int nufft_plan2_exec_timed(const nufft_plan2* plan, const double* c_dev, double* f_dev,
                           void* stream, int slot);
int nufft_plan2_timing_read(const nufft_plan2* plan, int nslots, double* ms_pass1,
                            double* ms_pass2);
/* F2~* f (transforms.hpp:226-232) */
int nufft_plan2_adjoint(const nufft_plan2* plan, const double* f_dev, double* out_dev,
                        void* stream);
int nufft_plan2_adjoint_host(const nufft_plan2* plan, const double* f, size_t len, double* out);

/* ------------------------------------------------------------- type I */
int nufft_plan1_create(const double* omega, size_t n, double epsilon, int device,
                       nufft_plan1** out);                                /* transforms.hpp:246-285 */
void nufft_plan1_destroy(nufft_plan1* plan);
int nufft_plan1_info(const nufft_plan1* plan, nufft_plan_info* info);
int nufft_plan1_samples(const nufft_plan1* plan, double* x, long* s, size_t* t);
int nufft_plan1_exec(const nufft_plan1* plan, const double* c_dev, double* f_dev, size_t batch,
                     void* stream);                                       /* transforms.hpp:287-289 */
int nufft_plan1_exec_host(const nufft_plan1* plan, const double* c, size_t len, double* f,
                          size_t batch);
/* F1~* g = conj(F2~ conj(g)) on the inner plan (detail::exec_nufft1_adjoint transforms.hpp:294-300) */
int nufft_plan1_adjoint(const nufft_plan1* plan, const double* g_dev, double* out_dev, void* stream);
int nufft_plan1_adjoint_host(const nufft_plan1* plan, const double* g, size_t len, double* out);

/* ------------------------------------------------------------- inverse (inverse.hpp) */
typedef struct nufft_toeplitz nufft_toeplitz; /* ToeplitzOperator inverse.hpp:22-27 */
/* CgReport inverse.hpp:89-95; the solution and residualHistory go to caller buffers */
typedef struct nufft_cg_report {
    size_t iterations;
    double relative_residual;
    int converged;
    size_t history_len; /* entries written to the history buffer (min(iterations, cap)) */
} nufft_cg_report;
/* detail::toeplitz_from_first_column inverse.hpp:37-50 (column: n complex, host) */
int nufft_toeplitz_from_first_column(const double* column, size_t n, int device, nufft_toeplitz** out);
int nufft_toeplitz_from_normal(const nufft_plan2* plan, nufft_toeplitz** out); /* inverse.hpp:54-58 */
int nufft_toeplitz_from_gram(const nufft_plan1* plan, nufft_toeplitz** out);   /* inverse.hpp:61-66 */
void nufft_toeplitz_destroy(nufft_toeplitz* op);
int nufft_toeplitz_size(const nufft_toeplitz* op, size_t* n);
/* members: spectrum 2n complex (imaginary parts 0), firstColumn n complex; NULL skips */
int nufft_toeplitz_members(const nufft_toeplitz* op, double* spectrum, double* first_column);
int nufft_toeplitz_matvec(const nufft_toeplitz* op, const double* v_dev, double* out_dev,
                          void* stream);                                   /* inverse.hpp:70-85 */
int nufft_toeplitz_matvec_host(const nufft_toeplitz* op, const double* v, size_t len, double* out);
/* cg_solve inverse.hpp:118-157 with the Toeplitz matvec as the operator */
int nufft_cg_toeplitz_host(const nufft_toeplitz* op, const double* rhs, size_t len, double tol,
                           size_t max_iter, double* solution, nufft_cg_report* report,
                           double* history, size_t history_cap);
/* inufft2 inverse.hpp:171-183 / inufft1 :187-200; op NULL = built from the plan */
int nufft_inufft2_host(const nufft_plan2* plan, const nufft_toeplitz* op, const double* f, size_t len,
                       double tol, double* solution, nufft_cg_report* report, double* history,
                       size_t history_cap);
int nufft_inufft2(const nufft_plan2* plan, const nufft_toeplitz* op, const double* f_dev, double tol,
                  double* solution_dev, nufft_cg_report* report, void* stream);
int nufft_inufft1_host(const nufft_plan1* plan, const nufft_toeplitz* op, const double* f, size_t len,
                       double tol, double* solution, nufft_cg_report* report, double* history,
                       size_t history_cap);
size_t nufft_default_cg_max_iter(size_t n); /* detail::default_cg_max_iter inverse.hpp:161-164 */

/* ------------------------------------------------------------- direct sums (oracle.hpp) */
/* nudft_direct oracle.hpp:70-86 on the device: f_j = sum_k c_k exp(-2 pi i x_j w_k) for
 * j < nx (the reference requires nx == n; a subset of outputs is allowed here),
 * exact product split + double-double reduction of the phase, Neumaier sums in
 * ascending k.  nudft2d_direct :90-107 (C row-major m x n, rows <-> y). */
int nufft_nudft_direct_host(const double* x, size_t nx, const double* omega, const double* c, size_t n,
                            double* f, int device);
int nufft_nudft_direct(const double* x_dev, size_t nx, const double* omega_dev, const double* c_dev,
                       size_t n, double* f_dev, void* stream);
int nufft_nudft2d_direct_host(const double* x, const double* y, size_t count, const double* C, size_t m,
                              size_t n, double* f, int device);

/* ------------------------------------------------------------- type III */
int nufft_plan3_create(const double* x_raw, const double* omega, size_t n_x, size_t n_omega,
                       double epsilon, int device, nufft_plan3** out);   /* transforms.hpp:321-380 */
void nufft_plan3_destroy(nufft_plan3* plan);
int nufft_plan3_info(const nufft_plan3* plan, nufft_plan_info* info);
int nufft_plan3_samples(const nufft_plan3* plan, double* x, long* s, size_t* t);
int nufft_plan3_exec(const nufft_plan3* plan, const double* c_dev, double* f_dev, size_t batch,
                     void* stream);                                       /* transforms.hpp:382-394 */
int nufft_plan3_exec_host(const nufft_plan3* plan, const double* c, size_t len, double* f,
                          size_t batch);

/* ------------------------------------------------------------- 2D type II */
int nufft_plan2d2_create(const double* x_raw, const double* y_raw, size_t count_x,
                         size_t count_y, size_t m, size_t n, double epsilon, int device,
                         nufft_plan2d** out);                             /* transform2d.hpp:65-100 */
void nufft_plan2d2_destroy(nufft_plan2d* plan);
int nufft_plan2d2_info(const nufft_plan2d* plan, nufft_plan_info* info);
/* host mirrors: normalized x, y; grid sx, sy, tx, ty; flatIndex (transform2d.hpp:24-49,89-91) */
int nufft_plan2d2_samples(const nufft_plan2d* plan, double* x, double* y, long* sx, long* sy,
                          size_t* tx, size_t* ty, size_t* flat_index);
/* C: m x n row-major complex (rows <-> y / m-grid, columns <-> x / n-grid) */
int nufft_plan2d2_exec(const nufft_plan2d* plan, const double* C_dev, double* f_dev,
                       size_t batch, void* stream);                       /* transform2d.hpp:145-147 */
int nufft_plan2d2_exec_host(const nufft_plan2d* plan, const double* C, size_t rows, size_t cols,
                            double* f, size_t batch);
/* detail::exec_nufft2d2_impl (transform2d.hpp:107-140): reuse_row_stage = 0 recomputes the
 * r2-independent row stage inside the r2 loop; results are bit-identical either way */
int nufft_plan2d2_exec_host_impl(const nufft_plan2d* plan, const double* C, size_t rows,
                                 size_t cols, double* f, size_t batch, int reuse_row_stage);

#ifdef __cplusplus
}
#endif
#endif /* NUFFT_B200_H */
