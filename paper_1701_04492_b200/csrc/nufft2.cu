// Type-II NUFFT execution — the north-star hot path.
//
// Reference: exec_nufft2 (proj/include/nufft/transforms.hpp:168-199) evaluates
//   f = sum_{r<K} diag(u_r) I_N(t,:) F diag(v_r) c
// as K separate passes of {scale, FFTW, gather} over HBM-sized vectors
// (accumulate_term :152-161).  Here the K terms are fused into two passes of
// a four-step FFT, N = N1 * N2 (k = k1*N2 + k2, t = t1 + N1*t2):
//
//  pass 1 (CTA per column k2, persistent): the column c[k1*N2 + k2] is read
//    from HBM once into shared memory; for every r it is scaled by
//    v_r = T_r(2k/N - 1) (Chebyshev recurrence state in registers), the
//    N1-point column FFT runs in registers + shared exchange buffers, the
//    inter-pass twiddle w_N^{t1 k2} is applied and Y_r[t1][k2] is written
//    (the only HBM round trip of the K spectra; full-sector stores, see y_index).
//  pass 2 (CTA per row t1, persistent, warp-specialized): FFT warps transform
//    Y_r[t1][:] for r = K-1 .. 0 into X_r[t1 + N1 t2] (double-buffered shared
//    memory); sample warps (1.5x as many), overlapped one r behind, gather X_r[t2_j] for every
//    sample bucketed on this row (t_j mod N1 == t1, plan-time sort) into a
//    per-sample register accumulator by Horner in r,
//        acc <- acc * (i h_j) + g_r(h_j^2) X_r[t2_j],
//    which sums u_r[j] X_r[t_j] over r without materializing u (Bessel form,
//    bessel.cuh).  2 exp(2 i h_j) acc is written once to f[j].
//
// HBM bytes per point (batch 1): c 16 + f 16 + xs/perm 12 + 32 K (Y written
// and read once) — SURVEY.md §8(d).  No atomics: every f[j] is owned by one
// thread and sums run in a fixed order, so results are bit-reproducible.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "bessel.cuh"
#include "fft_block.cuh"
#include "plans.hpp"
#include "tmem.cuh"

// second-level twiddle mode of block_fft_2l (fft_block.cuh) per kernel
#ifndef NB_P1_TW2
#define NB_P1_TW2 2
#endif
#ifndef NB_P2_TW2
#define NB_P2_TW2 0
#endif
#ifndef NB_P1_LDPIPE
#define NB_P1_LDPIPE 1
#endif
// staging the pass-1 box inside each warp's own exchange regions (a __syncwarp instead of a group
// barrier before the staging writes; box order (e pair, u, b, warp)): measured SLOWER, pass 1
// 1.56 -> 1.97 ms — the TMA engine drains that box order more slowly than (e pair, u, warp, b)
#ifndef NB_P1_STAGE_WARP
#define NB_P1_STAGE_WARP 0
#endif

namespace nb {

namespace {

constexpr int kMaxSamplesPerThread = 18;

__device__ __forceinline__ void nbar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Y layout (N1 >= 2): term rr of spectrum element (t1, k2) lives at
//   rr*N + 2*((t1 >> 1)*N2 + k2) + (t1 & 1)
// i.e. rows t1 and t1^1 are interleaved element by element.  In pass 1,
// adjacent lanes hold adjacent t1 of one column, so every warp store writes
// complete 32-byte sectors (16-byte column stores otherwise reach DRAM as
// partial sectors that need a read-modify-write whenever the CTAs writing
// the neighbouring columns drift apart).  Pass 2 reads a row at 32-byte
// stride; the other half of each sector is the neighbouring row, transformed
// concurrently by the adjacent CTA, and is served from L2.  N1 == 1 keeps
// the natural layout rr*N + k2.
__host__ __device__ __forceinline__ long long y_index(int rr, long long N, int log_n2, long long t1,
                                                      long long k2) {
    return rr * N + 2 * (((t1 >> 1) << log_n2) + k2) + (t1 & 1);
}

struct Pass1Params {
    long long n;  // N
    int log_n1, log_n2;
    int r0, r1;  // terms [r0, r1)
};

// ------------------------------------------------------------------ pass 1
// The c column (N1 values, 16 B each) is read from HBM once per column into
// shared memory (each thread only reads back its own slots); the Chebyshev
// state (T_{r-1}, T_r) of the thread's 16 points lives in registers.
template <int L1, bool UNIFORM>
__global__ void __launch_bounds__(L1 / 16, 1)
    k2_pass1(const double2* __restrict__ c, double2* __restrict__ Y, Pass1Params p) {
    constexpr int G = L1 / 16;
    extern __shared__ double2 smem[];
    double2* cbuf = smem;                   // L1, own-thread slots
    double2* buf0 = cbuf + L1;              // padded exchange buffers
    double2* buf1 = buf0 + padded_len(L1);
    double2* step = buf1 + padded_len(L1);  // 16 inter-pass twiddle steps
    double2* t16 = step + 16;               // Ns=16 stage twiddles
    const int tid = threadIdx.x;
    twiddle_table_build<L1>(t16, tid, G);
    Twiddles<L1> T;
    twiddle_init<L1>(T, t16, tid);
    const long long n2 = 1ll << p.log_n2;
    const long long N = p.n;
    for (long long k2 = blockIdx.x; k2 < n2; k2 += gridDim.x) {
        __syncthreads();  // previous column's readers of step are done
#pragma unroll
        for (int q = 0; q < 16; ++q) cbuf[tid + q * G] = __ldg(c + (((long long)(tid + q * G)) << p.log_n2) + k2);
        for (int q = tid; q < 16; q += G) step[q] = unit_root(k2 * q * G, N);  // w_N^{k2 q G}
        const double2 base = unit_root(k2 * tid, N);                          // w_N^{k2 tid}
        // 2 s_q = 4k/N - 2 with k = (tid + q G) N2 + k2  ->  two_s0 + q/4   (exact)
        const double two_s0 = (double)(4 * ((((long long)tid) << p.log_n2) + k2)) / (double)N - 2.0;
        double tcur[16], tprev[16];
        if constexpr (!UNIFORM) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                tprev[q] = 1.0;                       // T_0
                tcur[q] = 0.5 * (two_s0 + 0.25 * q);  // T_1 = s
            }
            for (int r = 1; r < p.r0; ++r) {  // state for r0: (T_{r0-1}, T_{r0})
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const double tn = __fma_rn(two_s0 + 0.25 * q, tcur[q], -tprev[q]);
                    tprev[q] = tcur[q];
                    tcur[q] = tn;
                }
            }
        }
        __syncthreads();
        for (int r = p.r0; r < p.r1; ++r) {
            if constexpr (FftShape<L1>::STAGES < 3) __syncthreads();  // buf0 reuse across r
            double2 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 cv = cbuf[tid + q * G];
                if constexpr (UNIFORM) {
                    v[q] = cv;
                } else {
                    const double vr = (r == 0) ? 0.5 : tcur[q];
                    v[q] = make_double2(cv.x * vr, cv.y * vr);
                }
            }
            block_fft<L1, -1>(v, buf0, buf1, tid, T, [] { __syncthreads(); });
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 w = cmul(base, step[q]);
                const long long t1 = tid + q * G;
                Y[y_index(r - p.r0, N, p.log_n2, t1, k2)] = cmul(v[q], w);
            }
            if constexpr (!UNIFORM) {
                if (r > 0) {  // (tprev, tcur) <- (T_r, T_{r+1}); after r == 0 the state already is (T_0, T_1)
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const double tn = __fma_rn(two_s0 + 0.25 * q, tcur[q], -tprev[q]);
                        tprev[q] = tcur[q];
                        tcur[q] = tn;
                    }
                }
            }
        }
    }
}

// Two-group pass 1 (L1 = 2048, 4096): a CTA runs two independent column
// workers of G threads each (columns 2*blockIdx + g, stride 2*gridDim), so
// twice as many warps hide the exchange and store latencies.  What kept the
// single-group kernel at one worker per SM — the cached c column (64 KB of
// shared memory) and the Chebyshev state (64 registers per thread) — lives in
// tensor memory instead (tmem.cuh): per thread 128 columns, [c re/im lo/hi x
// 16 points][T_{r-1}, T_r lo/hi x 16 points], read and advanced 4 points at a
// time.  Each worker exchanges through one padded buffer of its own.
template <int L1>
struct P1TmShape {
    static constexpr int G = L1 / 16;
    static constexpr int THREADS = 2 * G;
    static constexpr size_t SMEM = sizeof(double2) * (2 * padded_len(L1) + 2 * 16 + FftShapeX<L1>::TW_LEN);
    static_assert((THREADS / 32 + 3) / 4 * 128 <= 512, "TMEM columns");
};

// F2L (L1 = 4096): the column FFT is block_fft_2l (two group barriers per
// term instead of four); each thread then holds outputs t1 = t1_0 + 256 q with
// t1_0 = fft2l_out_index(tid, 0), lanes 2i and 2i + 1 the two rows of one
// 32-byte Y sector.
template <int L1, bool UNIFORM, bool F2L = false>
__global__ void __launch_bounds__(2 * (L1 / 16), 1)
    k2_pass1_tm(const double2* __restrict__ c, double2* __restrict__ Y, Pass1Params p) {
    static_assert(!F2L || L1 == 4096, "two-level FFT is 4096-point");
    constexpr int G = L1 / 16;
    extern __shared__ double2 smem[];
    __shared__ unsigned tmem_base;
    const int grp = threadIdx.x / G;
    const int tid = threadIdx.x - grp * G;
    double2* buf = smem + grp * padded_len(L1);
    double2* step = smem + 2 * padded_len(L1) + grp * 16;
    double2* tw = smem + 2 * padded_len(L1) + 32;
    twiddle_table_build<L1>(tw, threadIdx.x, 2 * G);
    Twiddles<L1> T;
    twiddle_init<L1>(T, tw, tid);
    if (threadIdx.x < 32) tm_alloc(&tmem_base, 512u);
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const unsigned tcol = tm_lane_base(tmem_base) + (unsigned)((threadIdx.x >> 7) * 128);
    const unsigned tc_c = tcol, tc_s = tcol + 64;
    const int bar = 1 + grp;
    auto gsync = [bar] { nbar_sync(bar, G); };
    const long long n2 = 1ll << p.log_n2;
    const long long N = p.n;
    for (long long k2 = 2ll * blockIdx.x + grp; k2 < n2; k2 += 2ll * gridDim.x) {
        gsync();  // previous column's readers of step are done
        for (int q = tid; q < 16; q += G) step[q] = unit_root(k2 * q * G, N);  // w_N^{k2 q G}
        const int t1_0 = F2L ? fft2l_out_index(tid, 0) : tid;                 // first output row
        const double2 base = unit_root(k2 * t1_0, N);                         // w_N^{k2 t1_0}
        const double two_s0 = (double)(4 * ((((long long)tid) << p.log_n2) + k2)) / (double)N - 2.0;
        // column of c and the Chebyshev state (T_{r0-1}, T_r0) into TMEM
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            unsigned cv[16], sv[16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = 4 * j + u;
                const double2 x = __ldg(c + (((long long)(tid + q * G)) << p.log_n2) + k2);
                cv[4 * u] = lo32(x.x);
                cv[4 * u + 1] = hi32(x.x);
                cv[4 * u + 2] = lo32(x.y);
                cv[4 * u + 3] = hi32(x.y);
                const double ts = two_s0 + 0.25 * q;
                double tprev = 1.0, tcur = 0.5 * ts;
                for (int r = 1; r < p.r0; ++r) {
                    const double tn = __fma_rn(ts, tcur, -tprev);
                    tprev = tcur;
                    tcur = tn;
                }
                sv[4 * u] = lo32(tprev);
                sv[4 * u + 1] = hi32(tprev);
                sv[4 * u + 2] = lo32(tcur);
                sv[4 * u + 3] = hi32(tcur);
            }
            tm_st16(tc_c + 16 * j, cv);
            if constexpr (!UNIFORM) tm_st16(tc_s + 16 * j, sv);
        }
        tm_wait_st();
        gsync();  // step visible
        for (int r = p.r0; r < p.r1; ++r) {
            double2 v[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                unsigned cv[16], sv[16];
                tm_ld16(tc_c + 16 * j, cv);
                if constexpr (!UNIFORM) tm_ld16(tc_s + 16 * j, sv);
                tm_wait_ld();
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = 4 * j + u;
                    const double2 x = make_double2(mk64(cv[4 * u], cv[4 * u + 1]), mk64(cv[4 * u + 2], cv[4 * u + 3]));
                    if constexpr (UNIFORM) {
                        v[q] = x;
                    } else {
                        const double tprev = mk64(sv[4 * u], sv[4 * u + 1]);
                        const double tcur = mk64(sv[4 * u + 2], sv[4 * u + 3]);
                        const double vr = (r == 0) ? 0.5 : tcur;
                        v[q] = make_double2(x.x * vr, x.y * vr);
                        if (r > 0) {  // (T_{r-1}, T_r) -> (T_r, T_{r+1})
                            const double tn = __fma_rn(two_s0 + 0.25 * q, tcur, -tprev);
                            sv[4 * u] = sv[4 * u + 2];
                            sv[4 * u + 1] = sv[4 * u + 3];
                            sv[4 * u + 2] = lo32(tn);
                            sv[4 * u + 3] = hi32(tn);
                        }
                    }
                }
                if constexpr (!UNIFORM) {
                    if (r > 0) tm_st16(tc_s + 16 * j, sv);
                }
            }
            gsync();  // previous term's last-stage reads of buf are done
            if constexpr (F2L) {
                block_fft_2l<-1, false, 0>(v, buf, tid, T, gsync);
            } else {
                block_fft_1buf<L1, -1>(v, buf, tid, T, gsync);
            }
            // y_index(rr, t1 = t1_0 + q G, k2) = base(t1_0) + q G N2   (G even)
            double2* yb = Y + y_index(r - p.r0, N, p.log_n2, t1_0, k2);
            const long long ystride = (long long)G << p.log_n2;
#pragma unroll
            for (int q = 0; q < 16; ++q) yb[q * ystride] = cmul(v[q], cmul(base, step[q]));
        }
        tm_wait_st();
    }
    tm_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc(tmem_base, 512u);
}

// Pass 1 with the Y column stored by the tensor-memory-access engine (TMA)
// instead of 16 per-thread 16-byte stores: on the LSU path every 32-byte Y
// sector costs an L1 data-pipe wavefront, and pass 1 ran its L1 pipe at 74 %
// (2048 of its ~5100 wavefronts per column-term were those stores).  After
// the two-level FFT each worker writes its twiddled column into its own
// exchange buffer in the order (b, warp, u, e) — contiguous 512 B per warp
// store, conflict-free — and one thread issues a single 5-D
// cp.async.bulk.tensor store of the 64 KiB box, which is exactly that order
// seen through the Y layout: t1 = e + 2 warp + 16 u + 256 b, dims
// (e + re/im: 4 doubles, u: 16, warp: 8, 16 rr + b, k2) with strides
// (-, 8 N2 * 32 B, N2 * 32 B, 128 N2 * 32 B, 32 B) (y_index, N1 = 4096).
// The next term's exchange waits (wait_group.read) until the engine has read
// the buffer.
__global__ void __launch_bounds__(512, 1)
    k2_pass1_tma(const double2* __restrict__ c, const __grid_constant__ CUtensorMap ymap, Pass1Params p) {
    constexpr int L1 = 4096, G = 256;
    extern __shared__ __align__(1024) double2 smem[];
    __shared__ unsigned tmem_base;
    const int grp = threadIdx.x / G;
    const int tid = threadIdx.x - grp * G;
    double2* buf = smem + grp * padded_len(L1);
    double2* step = smem + 2 * padded_len(L1) + grp * 16;
    // per-column FFT twiddles with the inter-pass twiddle folded in (see below)
    double2* tbw = smem + 2 * padded_len(L1) + 32 + grp * 1024;        // [e][tid]
    double2* t16c = smem + 2 * padded_len(L1) + 32 + 2048 + grp * 256;  // [a][u]
    Twiddles<L1> T;
    T.tb = tbw;
    T.t16 = t16c;
    if (threadIdx.x < 32) tm_alloc(&tmem_base, 512u);
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const unsigned tcol = tm_lane_base(tmem_base) + (unsigned)((threadIdx.x >> 7) * 128);
    const unsigned tc_c = tcol, tc_s = tcol + 64;
    const int bar = 1 + grp;
    auto gsync = [bar] { nbar_sync(bar, G); };
    const long long n2 = 1ll << p.log_n2;
    const long long N = p.n;
    const int warp = tid >> 5, e = tid & 1, u = (tid >> 1) & 15;
#if NB_P1_STAGE_WARP
    // staging inside the warp's own two exchange regions (slots [512 warp, 512 warp + 512): the
    // only ones its last exchange read), order (warp, b, u, e): a __syncwarp, not a group
    // barrier, separates the exchange reads from the staging writes
    double2* stg = buf + (warp * 512 + u * 2 + e);    // + 32 b: staging slot of output b
    constexpr int kStgStride = 32;
#else
    double2* stg = buf + ((warp * 16 + u) * 2 + e);  // + 256 b: staging slot of output b
    constexpr int kStgStride = 256;
#endif
    const unsigned buf_s = (unsigned)__cvta_generic_to_shared(buf);
#ifdef NB_P1_TRACE
    long long t1_set = 0, t1_ld = 0, t1_fft = 0, t1_out = 0, t1_cols = 0, t1_terms = 0, t1_t = clock64(), t1_x;
    const long long t1_begin = t1_t;
#define NB_T1(acc)       \
    t1_x = clock64();    \
    acc += t1_x - t1_t;  \
    t1_t = t1_x;
#else
#define NB_T1(acc)
#endif
    for (long long k2 = 2ll * blockIdx.x + grp; k2 < n2; k2 += 2ll * gridDim.x) {
        gsync();  // previous column's readers of step / t16c are done
        // The inter-pass twiddle w_N^{k2 t1} of output t1 = g + 16 a + 256 b of the
        // two-level FFT (block_fft_2l) splits as w_N^{k2 g} w_N^{16 k2 a} w_N^{256 k2 b}:
        //  * g is the first-level output index k1: w_N^{k2 k1} joins the first-level
        //    twiddle w_4096^{tid k1} = w_N^{N2 tid k1}, i.e. the power bases become
        //    w_N^{(N2 tid + k2) 2^e} (thread-private entries, no barrier needed);
        //  * a is the second-level twiddle index: w_256^{u a} w_N^{16 k2 a} = t16c[a][u];
        //  * b is the last DFT's output index: step[b] = w_N^{256 k2 b}, applied below.
        // 15 complex products per thread and term instead of 32 (base * step[b], then
        // times the value); every factor comes from one correctly rounded sincospi.
        for (int q = tid; q < 16; q += G) step[q] = unit_root(k2 * q * G, N);  // w_N^{k2 q G}
#pragma unroll
        for (int e = 0; e < 4; ++e)
            tbw[e * 256 + tid] = unit_root(((((long long)tid << p.log_n2) + k2) << e) & (N - 1), N);
        if constexpr (NB_P1_TW2 == 0) {
            const long long a = tid >> 4, uu = tid & 15;
            t16c[tid] = unit_root(((uu * (N >> 8) + 16 * k2) * a) & (N - 1), N);
        } else if (tid < 64) {  // block_fft_2l reads the rows a = 1, 2, 4, 8 only
            const long long a = 1ll << (tid >> 4), uu = tid & 15;
            t16c[16 * a + uu] = unit_root(((uu * (N >> 8) + 16 * k2) * a) & (N - 1), N);
        }
        const double two_s0 = (double)(4 * ((((long long)tid) << p.log_n2) + k2)) / (double)N - 2.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            unsigned cv[16], sv[16];
#pragma unroll
            for (int uu = 0; uu < 4; ++uu) {
                const int q = 4 * j + uu;
                const double2 x = __ldg(c + (((long long)(tid + q * G)) << p.log_n2) + k2);
                cv[4 * uu] = lo32(x.x);
                cv[4 * uu + 1] = hi32(x.x);
                cv[4 * uu + 2] = lo32(x.y);
                cv[4 * uu + 3] = hi32(x.y);
                const double ts = two_s0 + 0.25 * q;
                double tprev = 1.0, tcur = 0.5 * ts;
                for (int r = 1; r < p.r0; ++r) {
                    const double tn = __fma_rn(ts, tcur, -tprev);
                    tprev = tcur;
                    tcur = tn;
                }
                sv[4 * uu] = lo32(tprev);
                sv[4 * uu + 1] = hi32(tprev);
                sv[4 * uu + 2] = lo32(tcur);
                sv[4 * uu + 3] = hi32(tcur);
            }
            tm_st16(tc_c + 16 * j, cv);
            tm_st16(tc_s + 16 * j, sv);
        }
        tm_wait_st();
        gsync();  // step visible
        NB_T1(t1_set)
#ifdef NB_P1_TRACE
        ++t1_cols;
#endif
        NB_T1(t1_set)
#ifdef NB_P1_TRACE
        ++t1_cols;
#endif
        for (int r = p.r0; r < p.r1; ++r) {
            double2 v[16];
#if NB_P1_LDPIPE
            // TMEM chunk j + 1 is in flight while chunk j is scaled
            unsigned cvb[2][16], svb[2][16];
            tm_ld16(tc_c, cvb[0]);
            tm_ld16(tc_s, svb[0]);
#endif
#pragma unroll
            for (int j = 0; j < 4; ++j) {
#if NB_P1_LDPIPE
                tm_wait_ld();
                if (j < 3) {
                    tm_ld16(tc_c + 16 * (j + 1), cvb[(j + 1) & 1]);
                    tm_ld16(tc_s + 16 * (j + 1), svb[(j + 1) & 1]);
                }
                unsigned(&cv)[16] = cvb[j & 1];
                unsigned(&sv)[16] = svb[j & 1];
#else
                unsigned cv[16], sv[16];
                tm_ld16(tc_c + 16 * j, cv);
                tm_ld16(tc_s + 16 * j, sv);
                tm_wait_ld();
#endif
#pragma unroll
                for (int uu = 0; uu < 4; ++uu) {
                    const int q = 4 * j + uu;
                    const double2 x = make_double2(mk64(cv[4 * uu], cv[4 * uu + 1]), mk64(cv[4 * uu + 2], cv[4 * uu + 3]));
                    const double tprev = mk64(sv[4 * uu], sv[4 * uu + 1]);
                    const double tcur = mk64(sv[4 * uu + 2], sv[4 * uu + 3]);
                    const double vr = (r == 0) ? 0.5 : tcur;
                    v[q] = make_double2(x.x * vr, x.y * vr);
                    if (r > 0) {  // (T_{r-1}, T_r) -> (T_r, T_{r+1})
                        const double tn = __fma_rn(two_s0 + 0.25 * q, tcur, -tprev);
                        sv[4 * uu] = sv[4 * uu + 2];
                        sv[4 * uu + 1] = sv[4 * uu + 3];
                        sv[4 * uu + 2] = lo32(tn);
                        sv[4 * uu + 3] = hi32(tn);
                    }
                }
                if (r > 0) tm_st16(tc_s + 16 * j, sv);
            }
            NB_T1(t1_ld)
            // buf must be free (the engine has read the previous term's box) only when the
            // exchange first writes it: wait there, after the first-level DFT, so the TMA
            // drain of the previous column-term overlaps that compute
            block_fft_2l<-1, false, NB_P1_TW2>(v, buf, tid, T, gsync, [&] {
                if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                gsync();
            });
            // the last inter-pass twiddle factor in registers first: the products do not depend on
            // the barrier below, so they fill the wait for the group's slowest warp
#pragma unroll
            for (int b = 1; b < 16; ++b) v[b] = cmul(v[b], step[b]);
#if NB_P1_STAGE_WARP
            __syncwarp();  // the warp's exchange reads are done: its regions become its part of the box
#else
            gsync();  // exchange reads done: buf becomes the staging box
#endif
            NB_T1(t1_fft)
#pragma unroll
            for (int b = 0; b < 16; ++b) stg[kStgStride * b] = v[b];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            gsync();  // box complete
#ifdef NB_P1_SKIP_TMA  // timing ablation only (no output)
            if (false) {
#else
            if (tid == 0) {
#endif
                asm volatile(
                    "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                        &ymap),
#if NB_P1_STAGE_WARP
                    "r"(0), "r"(0), "r"(16 * (r - p.r0)), "r"(0), "r"((int)k2), "r"(buf_s)
#else
                    "r"(0), "r"(0), "r"(0), "r"(16 * (r - p.r0)), "r"((int)k2), "r"(buf_s)
#endif
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            NB_T1(t1_out)
#ifdef NB_P1_TRACE
            ++t1_terms;
#endif
        }
        tm_wait_st();
    }
#ifdef NB_P1_TRACE
    if (blockIdx.x == 3 && (tid == 0 || tid == 200))
        printf("pass1 trace grp %d tid %d: columns %lld, per column set-up %lld; per term: tmem-load+scale %lld fft %lld twiddle+stage+tma %lld; total %lld cycles\n",
               grp, tid, t1_cols, t1_set / t1_cols, t1_ld / t1_terms, t1_fft / t1_terms, t1_out / t1_terms, clock64() - t1_begin);
#endif
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    tm_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc(tmem_base, 512u);
}

// Y as the 5-D tensor k2_pass1_tma stores into (N1 = 4096, N2 = 2^log_n2)
bool make_y_tensor_map(CUtensorMap* map, double2* Y, int log_n2, int nterms) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }();
    if (!encode) return false;
    const cuuint64_t n2 = 1ull << log_n2;
    const cuuint64_t row = n2 * 32ull;  // bytes per (t1 >> 1)
#if NB_P1_STAGE_WARP
    // box order (e pair, u, b, warp): t1 = e + 2 warp + 16 u + 256 b
    cuuint64_t dims[5] = {4, 16, 16ull * (cuuint64_t)nterms, 8, n2};
    cuuint64_t strides[4] = {8 * row, 128 * row, row, 32};
    cuuint32_t box[5] = {4, 16, 16, 8, 1};
#else
    cuuint64_t dims[5] = {4, 16, 8, 16ull * (cuuint64_t)nterms, n2};
    cuuint64_t strides[4] = {8 * row, row, 128 * row, 32};
    cuuint32_t box[5] = {4, 16, 8, 16, 1};
#endif
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult rc = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)Y, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return rc == CUDA_SUCCESS;
}

// pass 1 for N1 == 1: Y_r[k] = v_r(k) c[k]
__global__ void k2_scale(const double2* __restrict__ c, double2* __restrict__ Y, long long N,
                         int r0, int r1, int uniform) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const double2 cv = c[k];
    if (uniform) {
        Y[k] = cv;
        return;
    }
    const double s = __dsub_rn(__dmul_rn(2.0, (double)k / (double)N), 1.0);
    double tprev = 1.0, tcur = s;
    for (int r = 0; r < r1; ++r) {
        double vr;
        if (r == 0) {
            vr = 0.5;
        } else {
            if (r >= 2) {
                const double tn = __fma_rn(2.0 * s, tcur, -tprev);
                tprev = tcur;
                tcur = tn;
            }
            vr = tcur;
        }
        if (r >= r0) Y[(long long)(r - r0) * N + k] = make_double2(cv.x * vr, cv.y * vr);
    }
}

// ------------------------------------------------------------------ pass 2
struct Pass2Params {
    long long n;
    int log_n1, log_n2;
    int r0, r1;
    const double* xs;
    const double* ds;        // type-I cores: delta and key in bucket order (xs would round omega/N)
    const unsigned* skey;
    const int* perm;
    const int* rowoff;
    long long row0, row1;  // rows [row0, row1) of this launch (multi-GPU chunked pass 2)
    int deg[kRankCap];
    int deg_rel0, deg_rel1;  // relative-accuracy degrees of g_{r1-1}, g_{r1} (recurrence start)
};

// One Horner step in r for the thread's samples: acc <- acc*(i h) + g_r(h^2) X_r[t2].
// Samples go in chunks of C with a straight-line series per chunk; slots past
// the chunk's sample count hold h = 0, t2 = 0 (load_samples) so no lane
// predication is needed (their accumulators are never stored).
template <int Q, int G>
__device__ __forceinline__ void horner_step(double2 (&acc)[Q], int r, int deg, const double2* xb,
                                            const int* st2, const double* sh, int tid) {
    constexpr int C = 4;
    const double* a = kBes + r * kSeriesTerms;
#pragma unroll
    for (int q0 = 0; q0 < Q; q0 += C) {
        double h[C], w[C], g[C];
#pragma unroll
        for (int u = 0; u < C; ++u) {
            h[u] = (q0 + u < Q) ? sh[tid + (q0 + u) * G] : 0.0;
            w[u] = h[u] * h[u];
        }
        series_deg<C>(g, w, a, deg);
#pragma unroll
        for (int u = 0; u < C; ++u) {
            const int q = q0 + u;
            if (q < Q) {
                const double2 X = xb[st2[tid + q * G]];
                const double ax = acc[q].x;
                acc[q].x = __fma_rn(g[u], X.x, -h[u] * acc[q].y);
                acc[q].y = __fma_rn(g[u], X.y, h[u] * ax);
            }
        }
    }
}

// t2 and h = -pi delta / 2 of sorted sample idx: recomputed from x exactly
// as the reference does (transforms.hpp:60-64,84-86), or — for type-I cores,
// whose delta = omega - round(omega) is not recoverable from omega/N
// (transforms.hpp:262-272) — read from the plan's sorted copies.
// where sample idx (bucket order) of this launch writes: f[perm[idx]], or the
// bucket-order partial fs[idx] when perm is null (multi-GPU r-split: the partials
// are reduced in bucket order and un-permuted once, nufft2_multi.cu)
__device__ __forceinline__ long long out_index(const Pass2Params& p, int idx) {
    return p.perm ? (long long)p.perm[idx] : (long long)idx;
}

__device__ __forceinline__ void sample_geom(const Pass2Params& p, int idx, int& t2, double& h) {
    if (p.ds) {
        h = half_phase(p.ds[idx]);
        t2 = (int)(p.skey[idx] & ((1u << p.log_n2) - 1u));
        return;
    }
    const double dn = (double)p.n;
    const double x = p.xs[idx];
    const double pr = __dmul_rn(dn, x);
    const long long sj = (long long)round(pr);
    const double d = __dadd_rn(__dsub_rn(pr, (double)sj), __fma_rn(dn, x, -pr));
    t2 = (int)((sj & (p.n - 1)) >> p.log_n1);
    h = half_phase(d);
}

// sample setup: recompute s, t, delta exactly (transforms.hpp:60-64,84-86) from sorted x
template <int Q, int G>
__device__ __forceinline__ void load_samples(const Pass2Params& p, int cb, int cnt, int tid,
                                             int* st2, double* sh, double2 (&acc)[Q]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        acc[q] = make_double2(0.0, 0.0);
        const int i = tid + q * G;
        if (i < cnt) {
            int t2;
            double h;
            sample_geom(p, cb + i, t2, h);
            st2[i] = t2;
            sh[i] = h;
        } else {  // idle slot: harmless inputs for the unpredicated Horner step
            st2[i] = 0;
            sh[i] = 0.0;
        }
    }
}

template <int Q, int G, bool UNIFORM>
__device__ __forceinline__ void store_samples(const Pass2Params& p, int cb, int cnt, int tid,
                                              const double* sh, double2 (&acc)[Q],
                                              double2* __restrict__ f) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int i = tid + q * G;
        if (i < cnt) {
            double2 out = acc[q];
            if constexpr (!UNIFORM) {
                const double h = sh[i];
                if (p.r0 > 0) {  // restore the (i h)^r0 factor of a partial term range
                    double hr = 1.0;
                    for (int k = 0; k < p.r0; ++k) hr *= h;
                    out = cscale(out, hr);
                    switch (p.r0 & 3) {
                        case 1: out = make_double2(-out.y, out.x); break;
                        case 2: out = make_double2(-out.x, -out.y); break;
                        case 3: out = make_double2(out.y, -out.x); break;
                        default: break;
                    }
                }
                double sn, cs;
                sincos(2.0 * h, &sn, &cs);
                out = cmul(make_double2(2.0 * cs, 2.0 * sn), out);
            }
            __stcs(f + out_index(p, cb + i), out);
        }
    }
}

// Small rows (L2 < 1024): one group does both the FFT and the samples.
template <int L2, bool UNIFORM>
__global__ void __launch_bounds__(L2 / 16)
    k2_pass2_small(const double2* __restrict__ Y, double2* __restrict__ f, Pass2Params p) {
    constexpr int G = L2 / 16;
    constexpr int Q = kMaxSamplesPerThread;
    constexpr int CAP = Q * G;
    extern __shared__ double2 smem[];
    double2* buf0 = smem;
    double2* buf1 = buf0 + padded_len(L2);
    double2* t16 = buf1 + padded_len(L2);
    double* sh = reinterpret_cast<double*>(t16 + FftShapeX<L2>::TW_LEN);
    int* st2 = reinterpret_cast<int*>(sh + CAP);
    const int tid = threadIdx.x;
    twiddle_table_build<L2>(t16, tid, G);
    Twiddles<L2> T;
    twiddle_init<L2>(T, t16, tid);
    __syncthreads();
    const long long N = p.n;
    double2* xb = block_fft_free_buf<L2>(buf0, buf1);
    for (long long row = p.row0 + blockIdx.x; row < p.row1; row += gridDim.x) {
        const int beg = p.rowoff[row], end = p.rowoff[row + 1];
        for (int cb = beg; cb < end; cb += CAP) {
            const int cnt = min(CAP, end - cb);
            double2 acc[Q];
            load_samples<Q, G>(p, cb, cnt, tid, st2, sh, acc);
            for (int r = p.r1 - 1; r >= p.r0; --r) {
                const int ys = p.log_n1 ? 2 : 1;  // element stride of a row in Y
                const double2* row_in = Y + (p.log_n1 ? y_index(r - p.r0, N, p.log_n2, row, 0)
                                                      : (long long)(r - p.r0) * N);
                double2 v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] = __ldcg(row_in + ys * (tid + q * G));
                block_fft<L2, -1>(v, buf0, buf1, tid, T, [] { __syncthreads(); });
#pragma unroll
                for (int q = 0; q < 16; ++q) xb[tid + q * G] = v[q];
                __syncthreads();
                if constexpr (UNIFORM) {
#pragma unroll
                    for (int q = 0; q < Q; ++q) {
                        const int i = tid + q * G;
                        if (i < cnt) acc[q] = xb[st2[i]];
                    }
                } else {
                    horner_step<Q, G>(acc, r, p.deg[r], xb, st2, sh, tid);
                }
                __syncthreads();
            }
            store_samples<Q, G, UNIFORM>(p, cb, cnt, tid, sh, acc, f);
            __syncthreads();
        }
    }
}

// Warp-specialized rows (L2 = 1024, e.g. N = 2^20): threads [0, G) run the
// row FFTs, threads [G, G + S) own the samples.  X_r alternates between two
// shared buffers:
//   FULL_b  (named barrier): X_r is in buffer b -> sample warps may gather;
//   EMPTY_b (named barrier): the gathers from b are done -> FFT of step i + 2.
// The sample warps' Horner updates of step r overlap the FFT of r-1.
// Sample role width: S = 1.5 G threads holding QS = 12 samples each
// (capacity 18 G = 1.125 N2, above the Poisson spread of an iid row): more
// warps than the FFT role, because the per-term sample update is a chain of
// dependent shared loads and FMAs that needs many warps in flight.
template <int L2>
struct WsShape {
    static constexpr int G = L2 / 16;                // FFT role threads
    static constexpr int S = G * 3 / 2;              // sample role threads
    static constexpr int QS = (18 * G + S - 1) / S;  // samples per sample thread
    static constexpr int CAP = QS * S;               // samples per chunk
    static constexpr int ALL = G + S;
};

template <int L2, bool UNIFORM>
__global__ void __launch_bounds__(WsShape<L2>::ALL, 1)
    k2_pass2_ws(const double2* __restrict__ Y, double2* __restrict__ f, Pass2Params p) {
    using W = WsShape<L2>;
    constexpr int G = W::G;
    constexpr int S = W::S;
    constexpr int Q = W::QS;
    constexpr int CAP = W::CAP;
    constexpr int ALL = W::ALL;
    constexpr int BAR_FULL = 1, BAR_EMPTY = 3, BAR_FFT = 5;
    extern __shared__ double2 smem[];
    double2* bufs = smem;  // 2 x padded_len(L2)
    double2* t16 = bufs + 2 * padded_len(L2);
    double* sh = reinterpret_cast<double*>(t16 + FftShapeX<L2>::TW_LEN);
    int* st2 = reinterpret_cast<int*>(sh + CAP);
    const bool fft_warp = threadIdx.x < G;
    const int tid = fft_warp ? threadIdx.x : threadIdx.x - G;
    twiddle_table_build<L2>(t16, threadIdx.x, ALL);
    Twiddles<L2> T;
    if (fft_warp) twiddle_init<L2>(T, t16, tid);
    __syncthreads();
    const long long N = p.n;
    const long long n2 = 1ll << p.log_n2;
    for (long long row = p.row0 + blockIdx.x; row < p.row1; row += gridDim.x) {
        const int beg = p.rowoff[row], end = p.rowoff[row + 1];
        for (int cb = beg; cb < end; cb += CAP) {
            const int cnt = min(CAP, end - cb);
            const int nt = p.r1 - p.r0;
            if (fft_warp) {
                for (int i = 0; i < nt; ++i) {
                    const int r = p.r1 - 1 - i;
                    const int b = i & 1;
                    double2* buf = bufs + b * padded_len(L2);
                    const int rr = r - p.r0;
                    if (tid == 0 && rr >= 2 && (row & 1) == 0) {  // warm L2 with a later row pair
                        const void* nxt = Y + y_index(rr - 2, N, p.log_n2, row, 0);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt),
                                     "r"((unsigned)(2 * n2 * sizeof(double2))) : "memory");
                    }
                    double2 v[16];
                    const double2* row_in = Y + y_index(rr, N, p.log_n2, row, 0);
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = __ldcg(row_in + 2 * (tid + q * G));
                    if (i >= 2) nbar_sync(BAR_EMPTY + b, ALL);  // samples done with X_{r+2}
                    block_fft_1buf<L2, -1>(v, buf, tid, T, [] { nbar_sync(BAR_FFT, G); });
                    nbar_sync(BAR_FFT, G);  // last-stage reads of buf done
#pragma unroll
                    for (int q = 0; q < 16; ++q) buf[tid + q * G] = v[q];
                    nbar_arrive(BAR_FULL + b, ALL);
                }
                for (int i = max(0, nt - 2); i < nt; ++i) nbar_sync(BAR_EMPTY + (i & 1), ALL);
            } else {
                double2 acc[Q];
                load_samples<Q, S>(p, cb, cnt, tid, st2, sh, acc);
                for (int i = 0; i < nt; ++i) {
                    const int r = p.r1 - 1 - i;
                    const int b = i & 1;
                    double2* xb = bufs + b * padded_len(L2);
                    nbar_sync(BAR_FULL + b, ALL);
                    if constexpr (UNIFORM) {
#pragma unroll
                        for (int q = 0; q < Q; ++q) {
                            const int j = tid + q * S;
                            if (j < cnt) acc[q] = xb[st2[j]];
                        }
                    } else {
                        horner_step<Q, S>(acc, r, p.deg[r], xb, st2, sh, tid);
                    }
                    nbar_arrive(BAR_EMPTY + b, ALL);
                }
                store_samples<Q, S, UNIFORM>(p, cb, cnt, tid, sh, acc, f);
            }
            __syncthreads();  // st2 / sh / buffers free for the next chunk
        }
    }
}

// ---------------------------------------------------------------- two FFT groups
// Pass 2 with two FFT worker groups (steps alternate between them) and one
// sample warpgroup whose per-sample state — accumulator, h, t2 — lives in
// tensor memory (7 columns per sample, tmem.cuh), so all 640 threads fit in
// 96 registers.  X_r rotates through three shared buffers (b = step % 3):
//   FULL_b  (named barrier, producing group + sample warps): X of the step is in b;
//   EMPTY_b (named barrier, sample warps + next user of b): the gathers from b are done.
// Each group loads its next Y row from HBM before waiting for its buffer and
// has two sample periods per transform, so two transforms are in flight.
template <int L2, int SWG = 1>
struct G2Shape {
    static constexpr int G = L2 / 16;
    static constexpr int S = 128 * SWG;         // sample warpgroups
    static constexpr int CH = SWG == 1 ? 4 : 2;  // samples per TMEM chunk
    static constexpr int Q = (18 * G / S + CH - 1) / CH * CH;  // samples per sample thread (capacity >= 1.125 L2)
    static constexpr int CAP = Q * S;
    static constexpr int ALL = 2 * G + S;
    // TMEM columns per sample: acc (4), h (2), t2 (1), Bessel state g_r, g_{r+1} (4), delta (2)
    static constexpr int COL_ACC = 0, COL_H = 4 * Q, COL_T = 6 * Q, COL_G = 7 * Q, COL_D = 11 * Q, COLS = 13 * Q;
    static constexpr unsigned TM_COLS = (SWG * COLS <= 128) ? 128u : (SWG * COLS <= 256 ? 256u : 512u);
    // registers: FFT groups 96, sample warps what is left of the CTA's allocation
    // (SWG = 2 with setmaxnreg 96/48 was tried: ptxas compiled the whole kernel at
    // the 768-thread launch bound of 80 registers and spilled 2.2 KB, so only
    // SWG = 1 is instantiated)
    static constexpr int REG_FFT = 96;
    static constexpr int REG_SMP = SWG == 1 ? 96 : 48;
    static constexpr size_t SMEM = sizeof(double2) * (3 * padded_len(L2) + FftShapeX<L2>::TW_LEN);
    static_assert(Q % CH == 0 && SWG * COLS <= 512, "sample layout");
    static_assert(SMEM <= 227 * 1024, "pass 2 (two groups) shared memory");
};

// F2L (L2 = 4096): the row FFT is block_fft_2l (two group barriers per step
// instead of four plus one before the X write): each thread writes its X
// values into the buffer slots it read last (fft2l_slot), and samples store
// their gather slot fft2l_slot_of(t2) in TMEM instead of t2.
template <int L2, bool UNIFORM, bool DSRC, int SWG, bool F2L = false>
__global__ void __launch_bounds__(G2Shape<L2, SWG>::ALL, 1)
    k2_pass2_g2(const double2* __restrict__ Y, double2* __restrict__ f, Pass2Params p) {
    static_assert(!F2L || L2 == 4096, "two-level FFT is 4096-point");
    using W = G2Shape<L2, SWG>;
    constexpr int CH = W::CH;
    constexpr int G = W::G;
    constexpr int S = W::S;
    constexpr int Q = W::Q;
    constexpr int CAP = W::CAP;
    constexpr int PAIR = G + S;                  // FULL/EMPTY participants
    constexpr int BAR_FULL = 1, BAR_EMPTY = 4, BAR_GRP = 7;  // FULL 1..3, EMPTY 4..6, groups 7..8
    extern __shared__ double2 smem[];
    __shared__ unsigned tmem_base;
    double2* bufs = smem;
    double2* t16 = bufs + 3 * padded_len(L2);
    const int role = threadIdx.x < 2 * G ? threadIdx.x / G : 2;  // 0, 1: FFT groups; 2: samples
    const int tid = role < 2 ? threadIdx.x - role * G : threadIdx.x - 2 * G;
    twiddle_table_build<L2>(t16, threadIdx.x, W::ALL);
    Twiddles<L2> T;
    twiddle_init<L2>(T, t16, tid);
    if (role == 2 && tid < 32) tm_alloc(&tmem_base, W::TM_COLS);
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if constexpr (W::REG_SMP != W::REG_FFT) {  // hand the sample warps' spare registers to the FFT groups
        if (role < 2)
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(W::REG_FFT));
        else
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(W::REG_SMP));
    }
    // sample warps 2G/32.. map to TMEM quarters (warp % 4); column block per extra warpgroup
    const unsigned tl = tm_lane_base(tmem_base) +
                        (unsigned)(role == 2 ? (tid >> 7) * W::COLS : 0);
    const long long N = p.n;
    const long long n2 = 1ll << p.log_n2;
    for (long long row = p.row0 + blockIdx.x; row < p.row1; row += gridDim.x) {
        const int beg = p.rowoff[row], end = p.rowoff[row + 1];
        for (int cb = beg; cb < end; cb += CAP) {
            const int cnt = min(CAP, end - cb);
            const int nt = p.r1 - p.r0;
            if (role < 2) {
                const int bar = BAR_GRP + role;
                auto gsync = [bar] { nbar_sync(bar, G); };
                for (int i = role; i < nt; i += 2) {
                    const int b = i % 3;
                    double2* buf = bufs + b * padded_len(L2);
                    const int rr = p.r1 - 1 - i - p.r0;
                    if (tid == 0 && i + 2 < nt) {  // warm L2 with this group's next row
                        const void* nxt = Y + y_index(rr - 2, N, p.log_n2, row, 0);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt),
                                     "r"((unsigned)(2 * n2 * sizeof(double2))) : "memory");
                    }
                    const double2* row_in = Y + y_index(rr, N, p.log_n2, row, 0);
                    double2 v[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = __ldcg(row_in + 2 * (tid + q * G));
                    if (i >= 3) nbar_sync(BAR_EMPTY + b, PAIR);  // gathers of step -3 from b done
                    if constexpr (F2L) {
                        block_fft_2l<-1, false, 0>(v, buf, tid, T, gsync);
                        // X in place: each thread overwrites only the slots it read last
#pragma unroll
                        for (int q = 0; q < 16; ++q) buf[fft2l_slot(tid, q)] = v[q];
                    } else {
                        block_fft_1buf<L2, -1>(v, buf, tid, T, gsync);
                        gsync();  // last-stage reads of buf done
#pragma unroll
                        for (int q = 0; q < 16; ++q) buf[tid + q * G] = v[q];
                    }
                    nbar_arrive(BAR_FULL + b, PAIR);
                }
            } else {
                const double dn = (double)p.n;
                // per-sample state into TMEM: acc = 0, h, t2
#pragma unroll 1
                for (int k = 0; k < Q / CH; ++k) {
                    unsigned av[4 * CH], hv[2 * CH], dv[2 * CH];
                    unsigned t2v[CH];
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const int i = tid + (CH * k + u) * S;
                        double d = 0.0;
                        int t2 = 0;
                        if (i < cnt) {
                            if constexpr (DSRC) {  // type-I core: stored delta and key
                                d = p.ds[cb + i];
                                t2 = (int)(p.skey[cb + i] & ((1u << p.log_n2) - 1u));
                            } else {
                                const double x = p.xs[cb + i];
                                const double pr = __dmul_rn(dn, x);
                                const long long sj = (long long)round(pr);
                                d = __dadd_rn(__dsub_rn(pr, (double)sj), __fma_rn(dn, x, -pr));
                                t2 = (int)((sj & (p.n - 1)) >> p.log_n1);
                            }
                        }
                        const double h = half_phase(d);
#pragma unroll
                        for (int c = 0; c < 4; ++c) av[4 * u + c] = 0u;
                        hv[2 * u] = lo32(h);
                        hv[2 * u + 1] = hi32(h);
                        dv[2 * u] = lo32(d);
                        dv[2 * u + 1] = hi32(d);
                        t2v[u] = (unsigned)(F2L ? fft2l_slot_of(t2) : t2);
                    }
                    tm_stn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
                    tm_stn<2 * CH>(tl + W::COL_H + 2 * CH * k, hv);
                    tm_stn<2 * CH>(tl + W::COL_D + 2 * CH * k, dv);
                    tm_stn<CH>(tl + W::COL_T + CH * k, t2v);
                    if constexpr (!UNIFORM) {
                        // (g_{r1-1}, g_{r1}) by the full series; lower orders follow from
                        // the backward recurrence g_{r-1} = r g_r - w g_{r+1}, stable for
                        // the minimal (Bessel) solution
                        double w[CH], ga[CH], gb[CH];
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            const double h = mk64(hv[2 * u], hv[2 * u + 1]);
                            w[u] = h * h;
                        }
                        series_deg<CH>(ga, w, kBes + (p.r1 - 1) * kSeriesTerms, p.deg_rel0);
                        series_deg<CH>(gb, w, kBes + p.r1 * kSeriesTerms, p.deg_rel1);
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            av[4 * u] = lo32(ga[u]);
                            av[4 * u + 1] = hi32(ga[u]);
                            av[4 * u + 2] = lo32(gb[u]);
                            av[4 * u + 3] = hi32(gb[u]);
                        }
                        tm_stn<4 * CH>(tl + W::COL_G + 4 * CH * k, av);
                    }
                }
                tm_wait_st();
                for (int i = 0; i < nt; ++i) {
                    const int r = p.r1 - 1 - i;
                    const int b = i % 3;
                    const double2* xb = bufs + b * padded_len(L2);
                    nbar_sync(BAR_FULL + b, PAIR);
                    const double* a = kBes + r * kSeriesTerms;
                    const int deg = p.deg[r];
                    (void)a;
                    (void)deg;
                    const double rd = (double)r;
#pragma unroll 1
                    for (int k = 0; k < Q / CH; ++k) {
                        unsigned av[4 * CH], gv[4 * CH], hv[2 * CH], t2v[CH];
                        tm_ldn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
                        tm_ldn<2 * CH>(tl + W::COL_H + 2 * CH * k, hv);
                        tm_ldn<CH>(tl + W::COL_T + CH * k, t2v);
                        if constexpr (!UNIFORM) tm_ldn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
                        tm_wait_ld();
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            const double2 X = xb[t2v[u]];
                            double2 acc;
                            if constexpr (UNIFORM) {
                                acc = X;
                            } else {
                                const double h = mk64(hv[2 * u], hv[2 * u + 1]);
                                const double gr = mk64(gv[4 * u], gv[4 * u + 1]);
                                const double gr1 = mk64(gv[4 * u + 2], gv[4 * u + 3]);
                                const double ax = mk64(av[4 * u], av[4 * u + 1]);
                                const double ay = mk64(av[4 * u + 2], av[4 * u + 3]);
                                acc.x = __fma_rn(gr, X.x, -h * ay);
                                acc.y = __fma_rn(gr, X.y, h * ax);
                                const double gm1 = __fma_rn(rd, gr, -(h * h) * gr1);  // g_{r-1}
                                gv[4 * u] = lo32(gm1);
                                gv[4 * u + 1] = hi32(gm1);
                                gv[4 * u + 2] = lo32(gr);
                                gv[4 * u + 3] = hi32(gr);
                            }
                            av[4 * u] = lo32(acc.x);
                            av[4 * u + 1] = hi32(acc.x);
                            av[4 * u + 2] = lo32(acc.y);
                            av[4 * u + 3] = hi32(acc.y);
                        }
                        tm_stn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
                        if constexpr (!UNIFORM) tm_stn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
                    }
                    // release b only to a later step (an EMPTY arrival nobody waits
                    // for would pair with the next use of the barrier)
                    if (i + 3 < nt) nbar_arrive(BAR_EMPTY + b, PAIR);
                }
                tm_wait_st();
                // f[perm] = 2 exp(2ih) (ih)^r0 acc
#pragma unroll 1
                for (int k = 0; k < Q / CH; ++k) {
                    unsigned av[4 * CH], hv[2 * CH], dv[2 * CH];
                    tm_ldn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
                    tm_ldn<2 * CH>(tl + W::COL_H + 2 * CH * k, hv);
                    tm_ldn<2 * CH>(tl + W::COL_D + 2 * CH * k, dv);
                    tm_wait_ld();
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const int i = tid + (CH * k + u) * S;
                        if (i >= cnt) continue;
                        double2 out = make_double2(mk64(av[4 * u], av[4 * u + 1]), mk64(av[4 * u + 2], av[4 * u + 3]));
                        if constexpr (!UNIFORM) {
                            const double h = mk64(hv[2 * u], hv[2 * u + 1]);
                            if (p.r0 > 0) {
                                double hr = 1.0;
                                for (int m = 0; m < p.r0; ++m) hr *= h;
                                out = cscale(out, hr);
                                switch (p.r0 & 3) {
                                    case 1: out = make_double2(-out.y, out.x); break;
                                    case 2: out = make_double2(-out.x, -out.y); break;
                                    case 3: out = make_double2(out.y, -out.x); break;
                                    default: break;
                                }
                            }
                            double sn, cs;  // exp(2ih) = exp(-i pi delta), argument exact
                            sincospi(-mk64(dv[2 * u], dv[2 * u + 1]), &sn, &cs);
                            out = cmul(make_double2(2.0 * cs, 2.0 * sn), out);
                        }
                        __stcs(f + out_index(p, cb + i), out);
                    }
                }
            }
            __syncthreads();  // buffers and TMEM state free for the next chunk
        }
    }
    tm_fence_before();
    __syncthreads();
    if (role == 2 && tid < 32) tm_dealloc(tmem_base, W::TM_COLS);
}

// ---------------------------------------------------------------- fused samples
// Pass 2 (L2 = 4096) without a sample warpgroup: two FFT groups of 256
// threads (128 registers each) take the steps S of one continuous sequence
// over the CTA's (row, chunk) units in turn (group S % 2), and each group
// updates every sample of the unit right after its own row FFT:
//   FFT_r (block_fft_2l, X left in place in the group's own buffer)
//   -> wait for the other group's update of step S-1   (named barrier H)
//   -> acc <- acc (i h) + g_r X_r[t2], g_{r-1} = r g_r - w g_{r+1}  (TMEM state)
//   -> hand off to the other group                      (named barrier H)
// The FFT of one group overlaps the sample update of the other (FP64-dense
// butterflies next to latency-bound gathers), the update is spread over 256
// threads instead of 128, the row spectra never leave their group's buffer,
// and no group waits for a whole-CTA barrier inside a row.  At a unit
// boundary the group that did the last update writes f for half the samples
// and sets up half of the next unit's, while the other group transforms the
// first row of the next unit and then does the other halves.
// Sample slot j of thread t is unit sample t + 256 j; its state lives in the
// thread's TMEM lane (shared by the same t of both groups), 13 columns:
// acc (4), g_r, g_{r+1} (4), h (2), gather slot (1), delta (2).
// L2 prefetch distance of k2_pass2_fs, in steps of the group (2 measured best:
// 2.32 -> 2.21 ms; 3: 2.26, 4: 2.33).  Only even rows prefetch: the row pair
// (t1, t1 ^ 1) shares its 128 KiB range (y_index).
constexpr int kFsL2Prefetch = 2;

struct FsShape {
    static constexpr int G = 256;
    static constexpr int SLOTS = 18;  // CAP = 4608 = 1.125 x 4096 samples per unit
    static constexpr int CAP = SLOTS * G;
    static constexpr int CH = 2;      // samples per TMEM chunk
    static constexpr int COL_ACC = 0, COL_G = 4 * SLOTS, COL_H = 8 * SLOTS, COL_T = 10 * SLOTS,
                         COL_D = 11 * SLOTS, COLS = 13 * SLOTS;
    static constexpr size_t SMEM = sizeof(double2) * (2 * kBuf2l + FftShapeX<4096>::TW_LEN);
    static_assert(COLS <= 256 && SLOTS % CH == 0, "TMEM layout");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

// load one Y row (stride-2 layout, y_index), transform it and leave X_r in
// place in the group's buffer (fft2l_slot order)
__device__ __forceinline__ void fs_load_row(double2 (&v)[16], const double2* row_in, int tid) {
#ifdef NB_P2_SKIP_LOAD  // timing ablation only (wrong results)
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(1e-3 * tid + q, (double)(long long)row_in * 1e-18);
#else
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __ldcg(row_in + 2 * (tid + q * 256));
#endif
}
template <class Bar>
__device__ __forceinline__ void fs_fft_regs(double2 (&v)[16], double2* buf, int tid, const Twiddles<4096>& T,
                                            Bar gsync) {
    // the group's gathers from its buffer (its previous step) are done.  (Waiting only
    // at the first exchange write, after the first-level DFT, measured slower here:
    // pass 2 2.19 -> 2.44 ms.)
    gsync();
#ifndef NB_P2_SKIP_FFT  // timing ablation only (wrong results): scripts/gpu_job_trace.sh
    block_fft_2l<-1, false, NB_P2_TW2>(v, buf, tid, T, gsync);
#endif
#pragma unroll
    for (int q = 0; q < 16; ++q) buf[fft2l_slot(tid, q)] = v[q];
    gsync();  // X complete
}


template <bool UNIFORM, bool DSRC>
__global__ void __launch_bounds__(512, 1)
    k2_pass2_fs(const double2* __restrict__ Y, double2* __restrict__ f, Pass2Params p) {
    using W = FsShape;
    constexpr int L2 = 4096, G = 256, CH = W::CH;
    constexpr int BAR_G = 1, BAR_H = 3, BAR_E = 5, BAR_U = 6;  // groups 1-2, handoff 3-4 (by arriving group)
    extern __shared__ double2 smem[];
    __shared__ unsigned tmem_base;
    const int grp = threadIdx.x >> 8;
    const int tid = threadIdx.x & (G - 1);
    double2* buf = smem + grp * kBuf2l;
    double2* tw = smem + 2 * kBuf2l;
    twiddle_table_build<L2>(tw, threadIdx.x, 2 * G);
    Twiddles<L2> T;
    twiddle_init<L2>(T, tw, tid);
    if (threadIdx.x < 32) tm_alloc(&tmem_base, 512u);
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const unsigned tl = tm_lane_base(tmem_base) + (unsigned)(((tid >> 7) & 1) * 256);
    const int gbar = BAR_G + grp;
    auto gsync = [gbar] { nbar_sync(gbar, G); };
    const long long N = p.n;
    const int nt = p.r1 - p.r0;
    const double dn = (double)p.n;

    // per-sample state of chunk k (slots CH k .. CH k + CH - 1) of a unit
    // per-sample state of this group's chunks k = grp, grp + 2, ... of a unit
    // (slots CH k .. CH k + CH - 1); all global loads are issued first
    constexpr int KMAX = (W::SLOTS / CH + 1) / 2;  // chunks per group
    auto init_half = [&](int cb, int cnt) {
        double dsrc[KMAX * CH];
        unsigned ksrc[KMAX * CH];
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk)
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int i = tid + (CH * (grp + 2 * kk) + u) * G;
                dsrc[CH * kk + u] = 0.0;
                ksrc[CH * kk + u] = 0u;
                if (i < cnt) {
                    if constexpr (DSRC) {
                        dsrc[CH * kk + u] = p.ds[cb + i];
                        ksrc[CH * kk + u] = p.skey[cb + i];
                    } else {
                        dsrc[CH * kk + u] = p.xs[cb + i];
                    }
                }
            }
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk) {
            const int k = grp + 2 * kk;
            if (CH * k * G >= cnt) break;
            unsigned av[4 * CH], hv[2 * CH], dv[2 * CH], t2v[CH];
            double h[CH];
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int i = tid + (CH * k + u) * G;
                double d = 0.0;
                int t2 = 0;
                if (i < cnt) {
                    if constexpr (DSRC) {  // type-I core: stored delta and key
                        d = dsrc[CH * kk + u];
                        t2 = (int)(ksrc[CH * kk + u] & ((1u << p.log_n2) - 1u));
                    } else {
                        const double x = dsrc[CH * kk + u];
                        const double pr = __dmul_rn(dn, x);
                        const long long sj = (long long)round(pr);
                        d = __dadd_rn(__dsub_rn(pr, (double)sj), __fma_rn(dn, x, -pr));
                        t2 = (int)((sj & (p.n - 1)) >> p.log_n1);
                    }
                }
                h[u] = half_phase(d);
#pragma unroll
                for (int c = 0; c < 4; ++c) av[4 * u + c] = 0u;
                hv[2 * u] = lo32(h[u]);
                hv[2 * u + 1] = hi32(h[u]);
                dv[2 * u] = lo32(d);
                dv[2 * u + 1] = hi32(d);
                t2v[u] = (unsigned)fft2l_slot_of(t2);
            }
            tm_stn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
            tm_stn<2 * CH>(tl + W::COL_H + 2 * CH * k, hv);
            tm_stn<2 * CH>(tl + W::COL_D + 2 * CH * k, dv);
            tm_stn<CH>(tl + W::COL_T + CH * k, t2v);
            if constexpr (!UNIFORM) {
                // (g_{r1-1}, g_{r1}) by the series; lower orders by the backward recurrence
                double w[CH], ga[CH], gb[CH];
#pragma unroll
                for (int u = 0; u < CH; ++u) w[u] = h[u] * h[u];
                // rolled Horner (uniform degree; same operations as series_fixed): this code
                // runs once per unit, and the unrolled switch made it ~10x larger
                {
                    const double* a0 = kBes + (p.r1 - 1) * kSeriesTerms;
                    const double* a1 = kBes + p.r1 * kSeriesTerms;
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        ga[u] = a0[p.deg_rel0];
                        gb[u] = a1[p.deg_rel1];
                    }
#pragma unroll 1
                    for (int m = p.deg_rel0 - 1; m >= 0; --m) {
                        const double am = a0[m];
#pragma unroll
                        for (int u = 0; u < CH; ++u) ga[u] = __fma_rn(ga[u], w[u], am);
                    }
#pragma unroll 1
                    for (int m = p.deg_rel1 - 1; m >= 0; --m) {
                        const double am = a1[m];
#pragma unroll
                        for (int u = 0; u < CH; ++u) gb[u] = __fma_rn(gb[u], w[u], am);
                    }
                }
                unsigned gv[4 * CH];
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    gv[4 * u] = lo32(ga[u]);
                    gv[4 * u + 1] = hi32(ga[u]);
                    gv[4 * u + 2] = lo32(gb[u]);
                    gv[4 * u + 3] = hi32(gb[u]);
                }
                tm_stn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
            }
        }
    };
    // f[perm] = 2 exp(2ih) (ih)^r0 acc for this group's chunks (perm loads first)
    auto epi_half = [&](int cb, int cnt) {
        int pm[KMAX * CH];
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk)
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int i = tid + (CH * (grp + 2 * kk) + u) * G;
                pm[CH * kk + u] = i < cnt ? out_index(p, cb + i) : 0;
            }
#pragma unroll
        for (int kk = 0; kk < KMAX; ++kk) {
            const int k = grp + 2 * kk;
            if (CH * k * G >= cnt) break;
            unsigned av[4 * CH], hv[2 * CH], dv[2 * CH];
            tm_ldn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
            tm_ldn<2 * CH>(tl + W::COL_H + 2 * CH * k, hv);
            tm_ldn<2 * CH>(tl + W::COL_D + 2 * CH * k, dv);
            tm_wait_ld();
#pragma unroll
            for (int u = 0; u < CH; ++u) {
                const int i = tid + (CH * k + u) * G;
                if (i >= cnt) continue;
                double2 out = make_double2(mk64(av[4 * u], av[4 * u + 1]), mk64(av[4 * u + 2], av[4 * u + 3]));
                if constexpr (!UNIFORM) {
                    const double h = mk64(hv[2 * u], hv[2 * u + 1]);
                    if (p.r0 > 0) {
                        double hr = 1.0;
                        for (int m = 0; m < p.r0; ++m) hr *= h;
                        out = cscale(out, hr);
                        switch (p.r0 & 3) {
                            case 1: out = make_double2(-out.y, out.x); break;
                            case 2: out = make_double2(-out.x, -out.y); break;
                            case 3: out = make_double2(out.y, -out.x); break;
                            default: break;
                        }
                    }
                    double sn, cs;  // exp(2ih) = exp(-i pi delta), argument exact
                    sincospi(-mk64(dv[2 * u], dv[2 * u + 1]), &sn, &cs);
                    out = cmul(make_double2(2.0 * cs, 2.0 * sn), out);
                }
                __stcs(f + pm[CH * kk + u], out);
            }
        }
    };
    // set-up and write-out are split between the groups by chunk parity (the
    // same chunks in every unit, so no group re-initializes a chunk the other
    // one is still writing out)
    auto nchunks = [](int c) { return ((c + G - 1) / G + CH - 1) / CH; };
    // first unit of the CTA
    const long long n1 = p.row1;  // end of this launch's row range
    long long row = p.row0 + blockIdx.x;
    int cb = 0, cnt = 0;
    auto seek = [&](long long r, int c) {  // first non-empty unit at or after (row r, sample c)
        for (; r < n1; r += gridDim.x) {
            const int beg = p.rowoff[r], end = p.rowoff[r + 1];
            const int c0 = c < 0 ? beg : c;
            if (c0 < end) {
                row = r;
                cb = c0;
                cnt = min(W::CAP, end - c0);
                return;
            }
            c = -1;
        }
        row = n1;
    };
    seek(row, -1);
    if (row < n1) {
        init_half(cb, cnt);
        tm_wait_st();
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
#ifdef NB_P2_TRACE
    long long tr_fft = 0, tr_wait = 0, tr_upd = 0, tr_edge = 0, tr_n = 0, tr_t = clock64(), tr_x;
    long long tr_e1 = 0, tr_e2 = 0, tr_e3 = 0, tr_e4 = 0, tr_units = 0;
    const long long tr_begin = tr_t;
#define NB_TR(acc)       \
    tr_x = clock64();    \
    acc += tr_x - tr_t;  \
    tr_t = tr_x;
#else
#define NB_TR(acc)
#endif
    int S0 = 0;         // global index of the unit's first step
    bool pre = false;   // this group's first step of the unit is already transformed
    bool have = false;  // v holds this group's next row (loaded ahead)
    double2 v[16];
    while (row < n1) {
        const long long urow = row;
        const int ucb = cb, ucnt = cnt;
        const int nch = nchunks(ucnt);  // occupied chunks (CTA-uniform)
        // the next unit: the rest of this row, else the CTA's next non-empty row
        if (ucb + ucnt < p.rowoff[urow + 1])
            seek(urow, ucb + ucnt);
        else
            seek(urow + gridDim.x, -1);
        const bool has_next = row < n1;
        const int last = nt - 1;
        const int lastgrp = (S0 + last) & 1;  // group of the unit's last update
        NB_TR(tr_edge)
        for (int i = (grp - S0) & 1; i < nt; i += 2) {
            const int rr = last - i;  // term index relative to r0 (r = r1 - 1 - i)
            const int r = p.r1 - 1 - i;
            NB_TR(tr_edge)
            if (i > 0 || !pre) {
                if (!have) fs_load_row(v, Y + y_index(rr, N, p.log_n2, urow, 0), tid);
                fs_fft_regs(v, buf, tid, T, gsync);
            }
            // this group's next row (step i + 2) is in flight during the update; a later
            // one (step i + 2 kFsL2Prefetch) is warmed in L2.  (Loading / prefetching the
            // next unit's first row across the unit boundary measured slower: 2.44 vs 2.48.)
            have = i + 2 < nt;
            if (have) fs_load_row(v, Y + y_index(rr - 2, N, p.log_n2, urow, 0), tid);
            if (tid == 0 && i + 2 * kFsL2Prefetch < nt && (urow & 1) == 0) {
                const void* nxt = Y + y_index(rr - 2 * kFsL2Prefetch, N, p.log_n2, urow, 0);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt),
                             "r"((unsigned)(2 * 4096 * sizeof(double2))) : "memory");
            }
            NB_TR(tr_fft)
            if (i > 0) {  // the other group's update of step i-1 is done
                nbar_sync(BAR_H + (grp ^ 1), 2 * G);
                tm_fence_after();
            }
            NB_TR(tr_wait)
            const double rd = (double)r;
#ifdef NB_P2_SKIP_UPD  // timing ablation only (wrong results)
            const int nch_u = 0;
#else
            const int nch_u = nch;
#endif
#pragma unroll 1
            for (int k = 0; k < nch_u; ++k) {
                unsigned av[4 * CH], gv[4 * CH], hv[2 * CH], t2v[CH];
                tm_ldn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
                tm_ldn<2 * CH>(tl + W::COL_H + 2 * CH * k, hv);
                tm_ldn<CH>(tl + W::COL_T + CH * k, t2v);
                if constexpr (!UNIFORM) tm_ldn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
                tm_wait_ld();
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const double2 X = buf[t2v[u]];
                    double2 acc;
                    if constexpr (UNIFORM) {
                        acc = X;
                    } else {
                        const double h = mk64(hv[2 * u], hv[2 * u + 1]);
                        const double gr = mk64(gv[4 * u], gv[4 * u + 1]);
                        const double gr1 = mk64(gv[4 * u + 2], gv[4 * u + 3]);
                        const double ax = mk64(av[4 * u], av[4 * u + 1]);
                        const double ay = mk64(av[4 * u + 2], av[4 * u + 3]);
                        acc.x = __fma_rn(gr, X.x, -h * ay);
                        acc.y = __fma_rn(gr, X.y, h * ax);
                        const double gm1 = __fma_rn(rd, gr, -(h * h) * gr1);  // g_{r-1}
                        gv[4 * u] = lo32(gm1);
                        gv[4 * u + 1] = hi32(gm1);
                        gv[4 * u + 2] = lo32(gr);
                        gv[4 * u + 3] = hi32(gr);
                    }
                    av[4 * u] = lo32(acc.x);
                    av[4 * u + 1] = hi32(acc.x);
                    av[4 * u + 2] = lo32(acc.y);
                    av[4 * u + 3] = hi32(acc.y);
                }
                tm_stn<4 * CH>(tl + W::COL_ACC + 4 * CH * k, av);
                if constexpr (!UNIFORM) tm_stn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
            }
            tm_wait_st();
            tm_fence_before();
            if (i < last) nbar_arrive(BAR_H + grp, 2 * G);  // hand off step i+1
            else nbar_arrive(BAR_E, 2 * G);                   // unit's last update done
            NB_TR(tr_upd)
#ifdef NB_P2_TRACE
            ++tr_n;
#endif
        }
        // unit boundary.  The group that did not do the last update transforms the
        // next unit's first row first (its first step), then joins.
        pre = false;
        NB_TR(tr_edge)
        if (grp != lastgrp) {
            if (has_next) {
                fs_load_row(v, Y + y_index(last, N, p.log_n2, row, 0), tid);
                fs_fft_regs(v, buf, tid, T, gsync);
                pre = true;
            }
            nbar_sync(BAR_E, 2 * G);
            tm_fence_after();
        }
        NB_TR(tr_e1)
        epi_half(ucb, ucnt);
        NB_TR(tr_e2)
        if (has_next) {
            init_half(cb, cnt);
            tm_wait_st();
            tm_fence_before();
            NB_TR(tr_e3)
            nbar_sync(BAR_U, 2 * G);  // next unit's samples set up by both groups
            tm_fence_after();
        }
        NB_TR(tr_e4)
#ifdef NB_P2_TRACE
        ++tr_units;
#endif
        S0 += nt;
    }
#ifdef NB_P2_TRACE
    NB_TR(tr_edge)
    if (blockIdx.x == 3 && (tid == 0 || tid == 200))
        printf("pass2 trace grp %d tid %d: steps %lld, per step: fft %lld wait %lld update %lld; units %lld, per unit edge: first-fft/wait %lld epilogue %lld init %lld wait %lld other %lld; total %lld cycles\n",
               grp, tid, tr_n, tr_fft / tr_n, tr_wait / tr_n, tr_upd / tr_n, tr_units, tr_e1 / tr_units, tr_e2 / tr_units,
               tr_e3 / tr_units, tr_e4 / tr_units, tr_edge / tr_units, tr_t - tr_begin);
#endif
    tm_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc(tmem_base, 512u);
}

// ------------------------------------------------------------------ launch
// Kernel choice per size (measured at N = 2^24, K = 20):
//   pass 1: L1 = 4096 (non-uniform) k2_pass1_tma; L1 = 4096 uniform and
//           L1 = 2048 k2_pass1_tm (two column workers, TMEM state; two-level
//           FFT at 4096); L1 < 2048 k2_pass1.
//   pass 2: L2 = 4096 (non-uniform) k2_pass2_fs; L2 = 4096 uniform and
//           L2 = 2048 k2_pass2_g2 (two FFT groups + a sample warpgroup);
//           L2 = 1024 k2_pass2_ws; L2 < 1024 k2_pass2_small.
// (A uniform plan — K = 1, e.g. the size-2N FFTs of the inverse — has one
// step per row, so the fused-sample kernel would be all unit boundary: 2.39
// vs 1.23 ms per CG iteration; the warp-specialized kernel overlaps those.)
template <int L>
constexpr size_t pass1_smem() {
    return sizeof(double2) * (L + 2 * padded_len(L) + 16 + FftShapeX<L>::TW_LEN);
}
template <int L>
constexpr size_t pass2_small_smem() {
    return sizeof(double2) * (2 * padded_len(L) + FftShapeX<L>::TW_LEN) +
           (sizeof(double) + sizeof(int)) * kMaxSamplesPerThread * (L / 16);
}
template <int L>
constexpr size_t pass2_ws_smem() {
    return sizeof(double2) * (2 * padded_len(L) + FftShapeX<L>::TW_LEN) +
           (sizeof(double) + sizeof(int)) * WsShape<L>::CAP;
}

template <class F>
void set_smem(F* fn, size_t bytes) {
    NB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

int occupancy(const void* fn, int threads, size_t smem) {
    int n = 0;
    NB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem));
    return std::max(1, n);
}

template <int L1>
void launch_pass1(const double2* c, double2* Y, const CorePlan& pl, int r0, int r1,
                  cudaStream_t s) {
    const DeviceCtx& ctx = DeviceCtx::get(pl.device);
    Pass1Params p{(long long)pl.n, pl.bk.log_n1, pl.bk.log_n2, r0, r1};
    const long long n2 = 1ll << pl.bk.log_n2;
    if constexpr (L1 >= 2048) {
        constexpr size_t SMT = P1TmShape<L1>::SMEM;
        const int grid = (int)std::min<long long>((n2 + 1) / 2, (long long)ctx.sms);
        if constexpr (L1 == 4096) {
            if (!pl.uniform) {
                CUtensorMap map;
                if (!make_y_tensor_map(&map, Y, pl.bk.log_n2, r1 - r0))
                    throw Error(kCudaError, "cuTensorMapEncodeTiled failed for the pass-1 Y map");
                constexpr size_t SMA = sizeof(double2) * (2 * padded_len(4096) + 32 + 2048 + 512);
                set_smem(k2_pass1_tma, SMA);
                k2_pass1_tma<<<grid, 512, SMA, s>>>(c, map, p);
                NB_LAUNCH();
                return;
            }
        }
        constexpr bool F2L = L1 == 4096;
        auto fn = pl.uniform ? k2_pass1_tm<L1, true, F2L> : k2_pass1_tm<L1, false, F2L>;
        set_smem(fn, SMT);
        fn<<<grid, P1TmShape<L1>::THREADS, SMT, s>>>(c, Y, p);
        NB_LAUNCH();
        return;
    }
    constexpr size_t SM = pass1_smem<L1>();
    auto fn = pl.uniform ? k2_pass1<L1, true> : k2_pass1<L1, false>;
    set_smem(fn, SM);
    const int grid = (int)std::min<long long>(n2, (long long)ctx.sms * occupancy((const void*)fn, L1 / 16, SM));
    fn<<<grid, L1 / 16, SM, s>>>(c, Y, p);
    NB_LAUNCH();
}

template <int L2, bool UNIFORM>
void launch_ws(const double2* Y, double2* f, const Pass2Params& p, long long n1, int sms, cudaStream_t s) {
    constexpr size_t SM = pass2_ws_smem<L2>();
    constexpr int threads = WsShape<L2>::ALL;
    auto fn = k2_pass2_ws<L2, UNIFORM>;
    set_smem(fn, SM);
    const int grid = (int)std::min<long long>(n1, (long long)sms * occupancy((const void*)fn, threads, SM));
    fn<<<grid, threads, SM, s>>>(Y, f, p);
    NB_LAUNCH();
}

template <int L2, bool UNIFORM>
void launch_g2(const double2* Y, double2* f, const Pass2Params& p, long long n1, int sms, cudaStream_t s) {
    constexpr size_t SM = G2Shape<L2>::SMEM;
    constexpr int threads = G2Shape<L2>::ALL;
    constexpr bool F2L = L2 == 4096;
    auto fn = p.ds ? k2_pass2_g2<L2, UNIFORM, true, 1, F2L> : k2_pass2_g2<L2, UNIFORM, false, 1, F2L>;
    set_smem(fn, SM);
    const int grid = (int)std::min<long long>(n1, (long long)sms);
    fn<<<grid, threads, SM, s>>>(Y, f, p);
    NB_LAUNCH();
}

void launch_fs(const double2* Y, double2* f, const Pass2Params& p, long long n1, int sms, cudaStream_t s) {
    auto fn = p.ds ? k2_pass2_fs<false, true> : k2_pass2_fs<false, false>;
    set_smem(fn, FsShape::SMEM);
    const int grid = (int)std::min<long long>(n1, (long long)sms);
    fn<<<grid, 2 * FsShape::G, FsShape::SMEM, s>>>(Y, f, p);
    NB_LAUNCH();
}

template <int L2>
void launch_pass2(const double2* Y, double2* f, const CorePlan& pl, int r0, int r1, long long row0,
                  long long row1, bool sorted_out, cudaStream_t s) {
    const DeviceCtx& ctx = DeviceCtx::get(pl.device);
    Pass2Params p{};
    p.n = (long long)pl.n;
    p.log_n1 = pl.bk.log_n1;
    p.log_n2 = pl.bk.log_n2;
    p.r0 = r0;
    p.r1 = r1;
    p.xs = pl.bk.xs.as<double>();
    p.ds = pl.delta_from_freq ? pl.bk.ds.as<double>() : nullptr;
    p.skey = pl.delta_from_freq ? pl.bk.skey.as<unsigned>() : nullptr;
    p.perm = sorted_out ? nullptr : pl.bk.perm.as<int>();
    p.rowoff = pl.bk.rowoff.as<int>();
    p.row0 = row0;
    p.row1 = row1;
    for (size_t r = 0; r < pl.series_deg.size() && r < (size_t)kRankCap; ++r) p.deg[r] = pl.series_deg[r];
    p.deg_rel0 = bessel_series_degree_rel(pl.gamma_factors, r1 - 1);
    p.deg_rel1 = bessel_series_degree_rel(pl.gamma_factors, r1);
    const long long n1 = row1 - row0;  // rows of this launch (grid size)
    const bool u = pl.uniform;
    if constexpr (L2 == 4096) {
        if (!u) return launch_fs(Y, f, p, n1, ctx.sms, s);
    }
    if constexpr (L2 >= 2048) {
        u ? launch_g2<L2, true>(Y, f, p, n1, ctx.sms, s) : launch_g2<L2, false>(Y, f, p, n1, ctx.sms, s);
    } else if constexpr (L2 == 1024) {
        u ? launch_ws<L2, true>(Y, f, p, n1, ctx.sms, s) : launch_ws<L2, false>(Y, f, p, n1, ctx.sms, s);
    } else {
        constexpr size_t SM = pass2_small_smem<L2>();
        constexpr int threads = L2 / 16;
        auto fn = u ? k2_pass2_small<L2, true> : k2_pass2_small<L2, false>;
        set_smem(fn, SM);
        const int grid = (int)std::min<long long>(n1, (long long)ctx.sms * occupancy((const void*)fn, threads, SM));
        fn<<<grid, threads, SM, s>>>(Y, f, p);
        NB_LAUNCH();
    }
}

void dispatch_pass1(int L, const double2* c, double2* Y, const CorePlan& pl, int r0, int r1,
                    cudaStream_t s) {
    switch (L) {
        case 16: return launch_pass1<16>(c, Y, pl, r0, r1, s);
        case 32: return launch_pass1<32>(c, Y, pl, r0, r1, s);
        case 64: return launch_pass1<64>(c, Y, pl, r0, r1, s);
        case 128: return launch_pass1<128>(c, Y, pl, r0, r1, s);
        case 256: return launch_pass1<256>(c, Y, pl, r0, r1, s);
        case 512: return launch_pass1<512>(c, Y, pl, r0, r1, s);
        case 1024: return launch_pass1<1024>(c, Y, pl, r0, r1, s);
        case 2048: return launch_pass1<2048>(c, Y, pl, r0, r1, s);
        case 4096: return launch_pass1<4096>(c, Y, pl, r0, r1, s);
        default: throw Error(kInternal, "pass1 size");
    }
}
void dispatch_pass2(int L, const double2* Y, double2* f, const CorePlan& pl, int r0, int r1,
                    cudaStream_t s, long long row0 = 0, long long row1 = -1, bool sorted_out = false) {
    if (row1 < 0) row1 = 1ll << pl.bk.log_n1;
    switch (L) {
        case 16: return launch_pass2<16>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 32: return launch_pass2<32>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 64: return launch_pass2<64>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 128: return launch_pass2<128>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 256: return launch_pass2<256>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 512: return launch_pass2<512>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 1024: return launch_pass2<1024>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 2048: return launch_pass2<2048>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        case 4096: return launch_pass2<4096>(Y, f, pl, r0, r1, row0, row1, sorted_out, s);
        default: throw Error(kInternal, "pass2 size");
    }
}

// ------------------------------------------------------------------ generic
__global__ void k2g_scale(const double2* __restrict__ c, double2* __restrict__ w, long long n,
                          int r) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double vr = v_factor_from_s(grid_s(k, n), r);
    const double2 cv = c[k];
    w[k] = make_double2(cv.x * vr, cv.y * vr);
}

__global__ void k2g_accum(const double2* __restrict__ X, double2* __restrict__ f,
                          const double* __restrict__ delta, const long long* __restrict__ t,
                          long long n, int r, int deg, int first, int uniform) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double2 x = X[t[j]];
    double2 term;
    if (uniform) {
        term = x;
    } else {
        term = cmul(u_factor(delta[j], r, deg), x);
    }
    f[j] = first ? term : cadd(f[j], term);
}

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace {
// f[j] = fs[invperm[j]]: coalesced f stores and invperm loads, 16-byte gathers from fs
// (random loads stay in flight; scattered 16-byte stores would be partial-sector
// read-modify-writes in L2)
__global__ void k_unpermute(const double2* __restrict__ fs, const int* __restrict__ invperm, long long n,
                            double2* __restrict__ f) {
    const long long j0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (j0 + 3 < n) {
        const int4 ix = __ldcs(reinterpret_cast<const int4*>(invperm + j0));
        const double2 a = __ldg(fs + ix.x), b = __ldg(fs + ix.y), c = __ldg(fs + ix.z), d = __ldg(fs + ix.w);
        __stcs(f + j0, a);
        __stcs(f + j0 + 1, b);
        __stcs(f + j0 + 2, c);
        __stcs(f + j0 + 3, d);
    } else {
        for (long long j = j0; j < n; ++j) f[j] = fs[invperm[j]];
    }
}
}  // namespace

void exec_type2_pass1(const CorePlan& pl, const double2* c, double2* Y, size_t r0, size_t r1,
                      cudaStream_t s) {
    if (!pl.fused || pl.bk.log_n1 == 0) throw Error(kInternal, "exec_type2_pass1: fused plan with N1 > 1 only");
    ensure_bessel_constants(pl.device);
    dispatch_pass1(1 << pl.bk.log_n1, c, Y, pl, (int)r0, (int)r1, s);
}
void exec_type2_pass2_rows(const CorePlan& pl, const double2* Y, double2* f, size_t r0, size_t r1,
                           long long row0, long long row1, bool sorted_out, cudaStream_t s) {
    if (!pl.fused || pl.bk.log_n1 == 0) throw Error(kInternal, "exec_type2_pass2_rows: fused plan with N1 > 1 only");
    if (row1 <= row0) return;
    dispatch_pass2(1 << pl.bk.log_n2, Y, f, pl, (int)r0, (int)r1, s, row0, row1, sorted_out);
}
void unpermute(const CorePlan& pl, const double2* fs, double2* f, size_t batch, cudaStream_t s) {
    for (size_t b = 0; b < batch; ++b) {
        k_unpermute<<<blocks((pl.n + 3) / 4), 256, 0, s>>>(fs + b * pl.n, pl.bk.invperm.as<int>(), (long long)pl.n,
                                                           f + b * pl.n);
        NB_LAUNCH();
    }
}

void exec_type2(const CorePlan& pl, const double2* c, double2* f, size_t batch, size_t r0,
                size_t r1, cudaStream_t s, cudaEvent_t* ev) {
    ensure_bessel_constants(pl.device);
    const size_t N = pl.n;
    if (r1 > pl.K) r1 = pl.K;
    if (r0 >= r1) {
        NB_CUDA(cudaMemsetAsync(f, 0, sizeof(double2) * N * batch, s));
        return;
    }
    if (pl.fused) {
        const size_t nt = r1 - r0;
        DevBuf Y(sizeof(double2) * N * nt, s);
        const int L1 = 1 << pl.bk.log_n1, L2 = 1 << pl.bk.log_n2;
        for (size_t b = 0; b < batch; ++b) {
            const double2* cb = c + b * N;
            double2* fb = f + b * N;
            if (ev && b == 0) NB_CUDA(cudaEventRecord(ev[0], s));
            if (pl.bk.log_n1 == 0) {
                k2_scale<<<blocks(N), 256, 0, s>>>(cb, Y.as<double2>(), (long long)N, (int)r0,
                                                   (int)r1, pl.uniform ? 1 : 0);
                NB_LAUNCH();
            } else {
                dispatch_pass1(L1, cb, Y.as<double2>(), pl, (int)r0, (int)r1, s);
            }
            if (ev && b == 0) NB_CUDA(cudaEventRecord(ev[1], s));
            dispatch_pass2(L2, Y.as<double2>(), fb, pl, (int)r0, (int)r1, s);
            if (ev && b == 0) NB_CUDA(cudaEventRecord(ev[2], s));
        }
        return;
    }
    // generic path: per-term scale -> FFT -> gather/accumulate (ascending r)
    DevBuf w(sizeof(double2) * N, s);
    for (size_t b = 0; b < batch; ++b) {
        const double2* cb = c + b * N;
        double2* fb = f + b * N;
        for (size_t r = r0; r < r1; ++r) {
            if (pl.uniform) {
                NB_CUDA(cudaMemcpyAsync(w.get(), cb, sizeof(double2) * N, cudaMemcpyDeviceToDevice, s));
            } else {
                k2g_scale<<<blocks(N), 256, 0, s>>>(cb, w.as<double2>(), (long long)N, (int)r);
                NB_LAUNCH();
            }
            fft_exec(w.as<double2>(), w.as<double2>(), N, 1, -1, s, pl.device);
            k2g_accum<<<blocks(N), 256, 0, s>>>(w.as<double2>(), fb, pl.ax.delta.as<double>(),
                                                pl.ax.t.as<long long>(), (long long)N, (int)r,
                                                pl.series_deg.empty() ? 15 : pl.series_deg[r],
                                                r == r0 ? 1 : 0, pl.uniform ? 1 : 0);
            NB_LAUNCH();
        }
    }
}

}  // namespace nb
