// Fused transpose core (type I, the type-II adjoint, type-III inner stage).
//
// Reference: exec_transpose_core transforms.hpp:206-221
//   F2~^T g = sum_r v_r .* F scatter_t(u_r .* g)     (F symmetric: F^T = F)
// evaluated by the reference as K passes of {scale, scatter, FFTW, scale-add}
// over HBM-sized vectors.  Here the K terms run in two passes of a four-step
// FFT, N = N1*N2, bins t = t1 + N1 t2, outputs k = k1 N2 + k2 — the mirror
// image of the type-II kernels (nufft2.cu):
//
//  pass A (CTA per row t1, persistent): the samples bucketed on the row
//    (plan-time sort by (t1, t2), ascending j inside a bin) are staged once
//    per row in shared memory as G_j = 2 exp(2 i h_j) g_j and h_j.  For every
//    r, a term phase (each thread owns 17 samples: balanced, branch-free,
//    17 independent Horner chains per Bessel coefficient) writes
//        T_j = (h_j^r g_r(h_j^2)) G_j            (= i^-r u_r[j] g_j, bessel.cuh)
//    into the idle FFT exchange buffer; a bin phase sums each of the thread's
//    16 bins in ascending j (the reference's order; no atomics); then the
//    N2-point row FFT runs in registers + shared memory, i^r is applied and
//    Z_r[t1][k2] is written (row-major, full-sector stores).
//  pass B (CTA per column k2, persistent): for r = 0..K-1 the column
//    Z_r[:][k2] is read, multiplied by the inter-pass twiddle w_N^{t1 k2},
//    transformed (N1-point FFT) and accumulated into registers as
//    acc[k] += v_r(k) X_r[k] with the Chebyshev recurrence for v_r; f is
//    written once.
//
// HBM bytes per point (batch 1): g 16 (gathered) + f 16 + delta/key/perm 16
// + 32 K (Z written and read once).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "bessel.cuh"
#include "fft_block.cuh"
#include "plans.hpp"
#include "tmem.cuh"

// second-level twiddle mode of block_fft_2l (fft_block.cuh) per kernel
#ifndef NB_PA_TW2
#define NB_PA_TW2 2
#endif
#ifndef NB_PB_TW2
#define NB_PB_TW2 2
#endif
#ifndef NB_PB_PF
#define NB_PB_PF 0  // next-term register prefetch at L1 = 2048: measured slower (cfg4 22.9 -> 24.1 ms)
#endif
#ifndef NB_PB_TMA2048
#define NB_PB_TMA2048 1
#endif
#ifndef NB_PB_QL
#define NB_PB_QL 0  // inputs per thread loaded through the LSU instead of the TMA box (even, 0..8): cfg4 19.07 / 19.40 / 19.98 / 20.49 ms at 0 / 2 / 4 / 6
#endif
#ifndef NB_PA_BINS
#define NB_PA_BINS 1
#endif
#ifndef NB_PA_SPLIT_TERM
#define NB_PA_SPLIT_TERM 1
#endif


namespace nb {

namespace {

constexpr size_t kSmemLimit = 227 * 1024;

struct PassAParams {
    long long n;
    int log_n1, log_n2;
    int r0, r1;
    const double* ds;
    const unsigned* skey;
    const int* perm;
    const int* rowoff;
    int deg[kRankCap];
    int conj;  // transform conj(g) (the adjoints: F2~* f = conj(F2~^T conj(f)), transforms.hpp:226-232)
    // stacked launch (k1_passA_tm without TMA): nb input vectors g + b * gstride share the plan
    // and write Z + b * zstride; the work units are the (vector, row) pairs
    int nb;
    long long gstride, zstride;
};

struct PassBParams {
    long long n;
    int log_n1, log_n2;
    int r0, r1;
    int conj;  // write conj(f)
};

// multiply by i^r
__device__ __forceinline__ double2 rot_ipow(double2 z, int r) {
    switch (r & 3) {
        case 1: return make_double2(-z.y, z.x);
        case 2: return make_double2(-z.x, -z.y);
        case 3: return make_double2(z.y, -z.x);
        default: return z;
    }
}

// samples per chunk of a row in pass A and the shared-memory footprint.  The
// per-term sample products are staged in the FFT exchange buffer (it is idle
// between two transforms), so a chunk holds at most padded_len(L2) = 17 G
// samples: QA = 17 per thread, a fixed, fully unrolled count.
template <int L2>
struct PassAShape {
    static constexpr int G = L2 / 16;
    static constexpr int QA = 17;
    static constexpr int CAP = QA * G;  // == padded_len(L2)
    static constexpr size_t SMEM = sizeof(double2) * (padded_len(L2) + FftShapeX<L2>::TW_LEN) +
                                   (sizeof(double2) + sizeof(double)) * CAP + sizeof(unsigned) * L2;
    static_assert(CAP == padded_len(L2) && CAP <= 65535, "pass A capacity");
    static_assert(SMEM <= kSmemLimit, "pass A shared memory");
};

template <int L2, bool UNIFORM>
__global__ void __launch_bounds__(L2 / 16, 1)
    k1_passA(const double2* __restrict__ g, double2* __restrict__ Z, PassAParams p) {
    using S = PassAShape<L2>;
    constexpr int G = S::G;
    constexpr int QA = S::QA;
    constexpr int CAP = S::CAP;
    extern __shared__ double2 smem[];
    double2* buf = smem;  // FFT exchange buffer; holds the sample terms between transforms
    double2* tw = buf + padded_len(L2);
    double2* gs = tw + FftShapeX<L2>::TW_LEN;
    double* hs = reinterpret_cast<double*>(gs + CAP);
    unsigned* bo = reinterpret_cast<unsigned*>(hs + CAP);  // bin b: [lo16, hi16) of the chunk
    unsigned short* bo16 = reinterpret_cast<unsigned short*>(bo);
    const int tid = threadIdx.x;
    twiddle_table_build<L2>(tw, tid, G);
    Twiddles<L2> T;
    twiddle_init<L2>(T, tw, tid);
    __syncthreads();
    const long long N = p.n;
    const long long n1 = 1ll << p.log_n1;
    const unsigned mask = (1u << p.log_n2) - 1u;
    for (long long row = blockIdx.x; row < n1; row += gridDim.x) {
        const int beg = p.rowoff[row], end = p.rowoff[row + 1];
        if (beg == end) {  // empty row: Z_r[row][:] = 0
            for (int r = p.r0; r < p.r1; ++r) {
                double2* out = Z + (long long)(r - p.r0) * N + (row << p.log_n2);
#pragma unroll
                for (int q = 0; q < 16; ++q) out[tid + q * G] = make_double2(0.0, 0.0);
            }
            continue;
        }
        for (int cb = beg, chunk = 0; cb < end; cb += CAP, ++chunk) {
            const int cnt = min(CAP, end - cb);
            for (int i = tid; i < L2; i += G) bo[i] = 0u;
            __syncthreads();
            for (int i = tid; i < cnt; i += G) {
                const unsigned t2 = p.skey[cb + i] & mask;
                if (i == 0 || (p.skey[cb + i - 1] & mask) != t2) bo16[2 * t2] = (unsigned short)i;
                if (i == cnt - 1 || (p.skey[cb + i + 1] & mask) != t2) bo16[2 * t2 + 1] = (unsigned short)(i + 1);
                double2 gv = __ldg(g + p.perm[cb + i]);
                if (p.conj) gv.y = -gv.y;
                if constexpr (UNIFORM) {
                    gs[i] = gv;
                } else {
                    const double h = half_phase(p.ds[cb + i]);
                    double sn, cs;
                    sincos(2.0 * h, &sn, &cs);
                    hs[i] = h;
                    gs[i] = cmul(make_double2(2.0 * cs, 2.0 * sn), gv);
                }
            }
            for (int i = cnt + tid; i < CAP; i += G) {  // tail slots: zero terms
                gs[i] = make_double2(0.0, 0.0);
                if constexpr (!UNIFORM) hs[i] = 0.0;
            }
            double hr[QA];  // h^r of the thread's samples tid + u G (fixed ownership)
#pragma unroll
            for (int u = 0; u < QA; ++u) hr[u] = 1.0;
            __syncthreads();
            if constexpr (!UNIFORM) {
                for (int r = 0; r < p.r0; ++r) {
#pragma unroll
                    for (int u = 0; u < QA; ++u) hr[u] *= hs[tid + u * G];
                }
            }
            for (int r = p.r0; r < p.r1; ++r) {
                __syncthreads();  // previous term's last-stage reads of buf are done
                const double2* src = gs;
                if constexpr (!UNIFORM) {
                    // term phase: buf[i] = h_i^r g_r(h_i^2) G_i (every thread QA samples)
                    const double* a = kBes + r * kSeriesTerms;
                    const int deg = p.deg[r];
                    double w[QA], gr[QA];
#pragma unroll
                    for (int u = 0; u < QA; ++u) {
                        const double h = hs[tid + u * G];
                        w[u] = h * h;
                        gr[u] = 0.0;
                    }
                    for (int m = deg; m >= 0; --m) {
                        const double am = a[m];
#pragma unroll
                        for (int u = 0; u < QA; ++u) gr[u] = __fma_rn(gr[u], w[u], am);
                    }
#pragma unroll
                    for (int u = 0; u < QA; ++u) {
                        const int i = tid + u * G;
                        const double m = hr[u] * gr[u];
                        buf[i] = cscale(gs[i], m);
                        hr[u] *= hs[i];
                    }
                    src = buf;
                    __syncthreads();
                }
                // bin phase: the thread's 16 bins, duplicates summed in ascending j
                double2 v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const unsigned rb = bo[tid + q * G];
                    const int i0 = rb & 0xffffu, i1 = rb >> 16;
                    double2 acc = make_double2(0.0, 0.0);
                    if (i0 < i1) {
                        acc = src[i0];
                        for (int i = i0 + 1; i < i1; ++i) acc = cadd(acc, src[i]);
                    }
                    v[q] = acc;
                }
                if constexpr (!UNIFORM) __syncthreads();  // terms read before stage 1 reuses buf
                block_fft_1buf<L2, -1>(v, buf, tid, T, [] { __syncthreads(); });
                double2* out = Z + (long long)(r - p.r0) * N + (row << p.log_n2);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const double2 z = UNIFORM ? v[q] : rot_ipow(v[q], r);
                    const int k2 = tid + q * G;
                    out[k2] = chunk == 0 ? z : cadd(out[k2], z);
                }
            }
            __syncthreads();  // gs / hs / bins free for the next chunk
        }
    }
}

// Two-worker pass A (L2 = 2048, 4096): each CTA runs two independent row
// workers (rows 2*blockIdx + g, stride 2*gridDim), so one worker's term/bin
// phases overlap the other's FFT.  The per-sample state moves from shared
// memory to tensor memory (tmem.cuh): per owned sample Q_j = h_j^r G_j
// (4 columns, advanced by one multiply by h_j per term) and h_j (2 columns),
// 17 samples x 6 = 102 columns per thread; each worker keeps one padded
// buffer (terms, then FFT exchange) and its bin table in shared memory.
template <int L2, int NW = 2>
struct PassATmShape {
    static constexpr int G = L2 / 16;
    static constexpr int QA = 17;
    static constexpr int CAP = QA * G;
    static constexpr int COL_Q = 0, COL_H = 4 * QA;  // 68 + 34 = 102 columns
    static constexpr size_t SMEM = sizeof(double2) * (NW * padded_len(L2) + FftShapeX<L2>::TW_LEN) +
                                   NW * sizeof(unsigned) * L2;
    static_assert(SMEM <= kSmemLimit, "pass A (row workers) shared memory");
    static_assert((NW * G + 127) / 128 * 6 * QA <= 512, "TMEM columns");
};

// F2L (L2 = 4096): the row FFT is block_fft_2l; output k2 of register q is
// fft2l_out_index(tid, q) (lanes 2i, 2i+1 write adjacent k2: full 32-byte sectors).
// TMA (with F2L): a single-chunk row term leaves through the tensor-memory-access
// engine — the z values are staged conflict-free in the exchange buffer in the
// order (b, warp, u, e) and one 5-D cp.async.bulk.tensor store writes the 64 KiB
// Z row (dims: e pair = 4 doubles, u, warp, b, rr N1 + row), as in k2_pass1_tma.
// BD: terms per bin summed as batches of independent loads before the residual loop — 2 when
// no bin of the plan holds more than two samples (jittered grids: cfg3 4.01 vs 4.09 ms), 4
// otherwise (iid samples: the adjoint 5.47 -> 5.24 ms, cfg4 22.9 -> 22.1 ms)
template <int L2, bool UNIFORM, bool F2L = false, bool TMA = false, int NW = 2, int BD = 2>
__global__ void __launch_bounds__(NW * (L2 / 16), 1)
    k1_passA_tm(const double2* __restrict__ g_all, double2* __restrict__ Z_all, PassAParams p,
                const __grid_constant__ CUtensorMap zmap) {
    static_assert(!F2L || L2 == 4096, "two-level FFT is 4096-point");
    static_assert(!TMA || F2L, "TMA store needs the two-level output order");
    using S = PassATmShape<L2, NW>;
    constexpr int G = S::G;
    constexpr int QA = S::QA;
    constexpr int CAP = S::CAP;
    extern __shared__ __align__(1024) double2 smem[];  // TMA box source: 128-byte aligned
    __shared__ unsigned tmem_base;
    const int grp = threadIdx.x / G;
    const int tid = threadIdx.x - grp * G;
    double2* buf = smem + grp * padded_len(L2);
    double2* tw = smem + NW * padded_len(L2);
    unsigned* bo = reinterpret_cast<unsigned*>(tw + FftShapeX<L2>::TW_LEN) + grp * L2;
    unsigned short* bo16 = reinterpret_cast<unsigned short*>(bo);
    twiddle_table_build<L2>(tw, threadIdx.x, NW * G);
    Twiddles<L2> T;
    twiddle_init<L2>(T, tw, tid);
    if (threadIdx.x < 32) tm_alloc(&tmem_base, 512u);
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const unsigned tcol = tm_lane_base(tmem_base) + (unsigned)((threadIdx.x >> 7) * 6 * QA);
    const int bar = 1 + grp;
    auto gsync = [bar] { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G) : "memory"); };
    const long long N = p.n;
    const long long n1 = 1ll << p.log_n1;
    const unsigned mask = (1u << p.log_n2) - 1u;
    const long long units = TMA ? n1 : n1 * max(p.nb, 1);  // (vector, row) pairs; TMA rows: one vector
    for (long long unit = (long long)NW * blockIdx.x + grp; unit < units; unit += (long long)NW * gridDim.x) {
        const long long row = unit & (n1 - 1), vec = unit >> p.log_n1;
        const double2* __restrict__ g = g_all + vec * p.gstride;
        double2* __restrict__ Z = Z_all + vec * p.zstride;
        const int beg = p.rowoff[row], end = p.rowoff[row + 1];
        if (beg == end) {  // empty row: Z_r[row][:] = 0
            for (int r = p.r0; r < p.r1; ++r) {
                double2* out = Z + (long long)(r - p.r0) * N + (row << p.log_n2);
#pragma unroll
                for (int q = 0; q < 16; ++q) out[tid + q * G] = make_double2(0.0, 0.0);
            }
            continue;
        }
        for (int cb = beg, chunk = 0; cb < end; cb += CAP, ++chunk) {
            const int cnt = min(CAP, end - cb);
            // (the gather indices are requested before the bin table is built: their DRAM round
            // trip overlaps the key loads below instead of following them)
            int pidx[QA];
#pragma unroll
            for (int uu = 0; uu < QA; ++uu) {
                const int i = tid + uu * G;
                pidx[uu] = i < cnt ? p.perm[cb + i] : -1;
            }
            if (TMA && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            gsync();  // previous chunk's readers of bo / buf are done
            for (int i = tid; i < L2; i += G) bo[i] = 0u;
            gsync();
            if constexpr (L2 != 2048) {
                for (int i = tid; i < cnt; i += G) {
                    const unsigned t2 = p.skey[cb + i] & mask;
                    if (i == 0 || (p.skey[cb + i - 1] & mask) != t2) bo16[2 * t2] = (unsigned short)i;
                    if (i == cnt - 1 || (p.skey[cb + i + 1] & mask) != t2) bo16[2 * t2 + 1] = (unsigned short)(i + 1);
                }
            } else {
                // bin table, N = 2^22: all the keys first instead of one round trip per iteration
                // of the rolled loop (cfg4 16.63 -> 16.44 ms; at 4096 the unrolled form measured
                // slower: adjoint 4.80 -> 4.95 ms)
                unsigned kc[QA], kp[QA], kn[QA];
#pragma unroll
                for (int uu = 0; uu < QA; ++uu) {
                    const int i = tid + uu * G;
                    kc[uu] = kp[uu] = kn[uu] = 0u;
                    if (i < cnt) {
                        kc[uu] = p.skey[cb + i] & mask;
                        kp[uu] = i > 0 ? (p.skey[cb + i - 1] & mask) : ~0u;
                        kn[uu] = i < cnt - 1 ? (p.skey[cb + i + 1] & mask) : ~0u;
                    }
                }
#pragma unroll
                for (int uu = 0; uu < QA; ++uu) {
                    const int i = tid + uu * G;
                    if (i < cnt) {
                        if (kp[uu] != kc[uu]) bo16[2 * kc[uu]] = (unsigned short)i;
                        if (kn[uu] != kc[uu]) bo16[2 * kc[uu] + 1] = (unsigned short)(i + 1);
                    }
                }
            }
            // owned samples i = tid + u G: Q = h^r0 G_j (G_j = 2 exp(2ih) g_j), h.
            // Every index, then every gathered value and delta, is loaded before any of them
            // is used: the TMEM stores below are ordered asm statements, and with the loads
            // inside the chunk loop each chunk paid its own perm -> g DRAM round trips in turn
            // (long-scoreboard stalls were 15-17 % of this kernel)
            double2 Gin[QA];
            double din[QA];
#pragma unroll
            for (int uu = 0; uu < QA; ++uu) {
                const int i = tid + uu * G;
                Gin[uu] = make_double2(0.0, 0.0);
                din[uu] = 0.0;
                if (pidx[uu] >= 0) {
                    Gin[uu] = __ldg(g + pidx[uu]);
                    if constexpr (!UNIFORM) din[uu] = p.ds[cb + i];
                }
            }
#pragma unroll
            for (int k = 0; k < (QA + 3) / 4; ++k) {
                unsigned qv[16], hv[8];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int uu = 4 * k + u;
                    const int i = tid + uu * G;
                    double2 Gj = make_double2(0.0, 0.0);
                    double h = 0.0;
                    if (uu < QA && i < cnt) {
                        Gj = Gin[uu < QA ? uu : 0];
                        if (p.conj) Gj.y = -Gj.y;
                        if constexpr (!UNIFORM) {
                            const double dj = din[uu < QA ? uu : 0];
                            h = half_phase(dj);
                            double sn, cs;  // exp(2ih) = exp(-i pi delta), argument exact (and
                                            // sincospi inlines to far less code than sincos)
                            sincospi(-dj, &sn, &cs);
                            Gj = cmul(make_double2(2.0 * cs, 2.0 * sn), Gj);
#pragma unroll 1  // a partial term range (multi-GPU) only
                            for (int r = 0; r < p.r0; ++r) Gj = cscale(Gj, h);
                        }
                    }
                    qv[4 * u] = lo32(Gj.x);
                    qv[4 * u + 1] = hi32(Gj.x);
                    qv[4 * u + 2] = lo32(Gj.y);
                    qv[4 * u + 3] = hi32(Gj.y);
                    hv[2 * u] = lo32(h);
                    hv[2 * u + 1] = hi32(h);
                }
                if (4 * k + 4 <= QA) {
                    tm_st16(tcol + S::COL_Q + 16 * k, qv);
                    tm_st8(tcol + S::COL_H + 8 * k, hv);
                } else {  // QA % 4 == 1: the last sample alone
                    tm_st4(tcol + S::COL_Q + 16 * k, qv[0], qv[1], qv[2], qv[3]);
                    unsigned h2[8] = {hv[0], hv[1], 0, 0, 0, 0, 0, 0};
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(tcol + S::COL_H + 8 * k),
                                 "r"(h2[0]), "r"(h2[1])
                                 : "memory");
                }
            }
            tm_wait_st();
            for (int r = p.r0; r < p.r1; ++r) {
                // (the wait for the previous term's last-stage reads of buf — and for the TMA
                // engine to have read its box — sits at the first write of buf below, after the
                // first eight samples' series: that work overlaps the drain)
                // term phase: buf[i] = g_r(h_i^2) Q_i, then Q_i <- h_i Q_i.  Two TMEM chunks
                // (8 samples) share one Horner loop (8 independent FMA chains per coefficient)
                const double* a = kBes + r * kSeriesTerms;
                const int deg = p.deg[r];
                constexpr int NCHK = (QA + 3) / 4;
#if NB_PA_SPLIT_TERM
                // T1: the series g_r(h^2) of every owned sample (TMEM and registers only) ...
                double grv[4 * NCHK];
#pragma unroll
                for (int k0 = 0; k0 < NCHK; k0 += 2) {
                    double w[8], gr[8];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int k = k0 + c;
                        unsigned hv[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) hv[e] = 0u;
                        if (k < NCHK) {
                            if (4 * k + 4 <= QA) {
                                tm_ld8(tcol + S::COL_H + 8 * k, hv);
                            } else {
                                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                                             : "=r"(hv[0]), "=r"(hv[1])
                                             : "r"(tcol + S::COL_H + 8 * k)
                                             : "memory");
                            }
                        }
                        tm_wait_ld();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const double hh = mk64(hv[2 * u], hv[2 * u + 1]);
                            w[4 * c + u] = hh * hh;
                        }
                    }
                    if constexpr (UNIFORM) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) gr[u] = 1.0;
                    } else {
#pragma unroll
                        for (int u = 0; u < 8; ++u) gr[u] = a[deg];
#pragma unroll 1
                        for (int m = deg - 1; m >= 0; --m) {
                            const double am = a[m];
#pragma unroll
                            for (int u = 0; u < 8; ++u) gr[u] = __fma_rn(gr[u], w[u], am);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (4 * k0 + u < 4 * NCHK) grv[4 * k0 + u] = gr[u];
                }
                // ... then the wait for buf (previous term's last-stage reads, the TMA drain) ...
                if (TMA && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                gsync();
                // ... T2: buf[i] = g_r Q_i, Q_i <- h_i Q_i
#pragma unroll
                for (int k = 0; k < NCHK; ++k) {
                    const bool full = 4 * k + 4 <= QA;
                    unsigned qv[16], hv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) hv[e] = 0u;
                    if (full) {
                        tm_ld16(tcol + S::COL_Q + 16 * k, qv);
                        if constexpr (!UNIFORM) tm_ld8(tcol + S::COL_H + 8 * k, hv);
                    } else {
                        tm_ld4(tcol + S::COL_Q + 16 * k, qv[0], qv[1], qv[2], qv[3]);
                        if constexpr (!UNIFORM) tm_ld2(tcol + S::COL_H + 8 * k, hv[0], hv[1]);
#pragma unroll
                        for (int e = 4; e < 16; ++e) qv[e] = 0u;
                    }
                    tm_wait_ld();
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int uu = 4 * k + u;
                        if (uu >= QA) break;
                        const double2 Qv = make_double2(mk64(qv[4 * u], qv[4 * u + 1]), mk64(qv[4 * u + 2], qv[4 * u + 3]));
                        buf[tid + uu * G] = cscale(Qv, grv[uu]);
                        const double2 Qn = UNIFORM ? Qv : cscale(Qv, mk64(hv[2 * u], hv[2 * u + 1]));
                        qv[4 * u] = lo32(Qn.x);
                        qv[4 * u + 1] = hi32(Qn.x);
                        qv[4 * u + 2] = lo32(Qn.y);
                        qv[4 * u + 3] = hi32(Qn.y);
                    }
                    if constexpr (!UNIFORM) {
                        if (full) tm_st16(tcol + S::COL_Q + 16 * k, qv);
                        else tm_st4(tcol + S::COL_Q + 16 * k, qv[0], qv[1], qv[2], qv[3]);
                    }
                }
#else
#pragma unroll
                for (int k0 = 0; k0 < NCHK; k0 += 2) {
                    double h[8], w[8], gr[8];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int k = k0 + c;
                        unsigned hv[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) hv[e] = 0u;
                        if (k < NCHK) {
                            if (4 * k + 4 <= QA) {
                                tm_ld8(tcol + S::COL_H + 8 * k, hv);
                            } else {
                                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                                             : "=r"(hv[0]), "=r"(hv[1])
                                             : "r"(tcol + S::COL_H + 8 * k)
                                             : "memory");
                            }
                        }
                        tm_wait_ld();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            h[4 * c + u] = mk64(hv[2 * u], hv[2 * u + 1]);
                            w[4 * c + u] = h[4 * c + u] * h[4 * c + u];
                        }
                    }
                    if constexpr (UNIFORM) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) gr[u] = 1.0;
                    } else {
                        // rolled Horner (uniform degree; the same operations as series_fixed):
                        // the switch-unrolled form multiplied the kernel's code size
#pragma unroll
                        for (int u = 0; u < 8; ++u) gr[u] = a[deg];
#pragma unroll 1
                        for (int m = deg - 1; m >= 0; --m) {
                            const double am = a[m];
#pragma unroll
                            for (int u = 0; u < 8; ++u) gr[u] = __fma_rn(gr[u], w[u], am);
                        }
                    }
                    if (k0 == 0) {
                        if (TMA && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        gsync();  // previous term's last-stage reads of buf (and the TMA's) are done
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int k = k0 + c;
                        if (k >= NCHK) break;
                        const bool full = 4 * k + 4 <= QA;
                        unsigned qv[16];
                        if (full) {
                            tm_ld16(tcol + S::COL_Q + 16 * k, qv);
                        } else {
                            tm_ld4(tcol + S::COL_Q + 16 * k, qv[0], qv[1], qv[2], qv[3]);
#pragma unroll
                            for (int e = 4; e < 16; ++e) qv[e] = 0u;
                        }
                        tm_wait_ld();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int uu = 4 * k + u;
                            if (uu >= QA) break;
                            const double2 Qv =
                                make_double2(mk64(qv[4 * u], qv[4 * u + 1]), mk64(qv[4 * u + 2], qv[4 * u + 3]));
                            buf[tid + uu * G] = cscale(Qv, gr[4 * c + u]);
                            const double2 Qn = UNIFORM ? Qv : cscale(Qv, h[4 * c + u]);
                            qv[4 * u] = lo32(Qn.x);
                            qv[4 * u + 1] = hi32(Qn.x);
                            qv[4 * u + 2] = lo32(Qn.y);
                            qv[4 * u + 3] = hi32(Qn.y);
                        }
                        if constexpr (!UNIFORM) {
                            if (full) tm_st16(tcol + S::COL_Q + 16 * k, qv);
                            else tm_st4(tcol + S::COL_Q + 16 * k, qv[0], qv[1], qv[2], qv[3]);
                        }
                    }
                }
#endif
                gsync();  // terms visible
                // bin sums in ascending j.  Sixteen bins per thread, about one sample per bin:
                // all bin ranges first, then every bin's first and second term as two batches
                // of independent (predicated) loads, and a loop only for bins with three or
                // more samples — sixteen dependent range -> term -> branch chains in sequence
                // were 22 % of this kernel's stall samples at cfg4 (r2_ncu_type3_s5.txt)
                double2 v[16];
#if !NB_PA_BINS
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const unsigned rb = bo[tid + q * G];
                    const int i0 = rb & 0xffffu, i1 = rb >> 16;
                    double2 acc = make_double2(0.0, 0.0);
                    if (i0 < i1) {
                        acc = buf[i0];
                        for (int i = i0 + 1; i < i1; ++i) acc = cadd(acc, buf[i]);
                    }
                    v[q] = acc;
                }
#else
                unsigned rbv[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) rbv[q] = bo[tid + q * G];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int i0 = rbv[q] & 0xffffu, i1 = rbv[q] >> 16;
                    v[q] = i0 < i1 ? buf[i0] : make_double2(0.0, 0.0);
                }
                bool more = false;
#pragma unroll
                for (int d = 1; d < BD; ++d) {  // the d-th term of every bin, one batch per d
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int i0 = rbv[q] & 0xffffu, i1 = rbv[q] >> 16;
                        if (i0 + d < i1) v[q] = cadd(v[q], buf[i0 + d]);
                        if (d == BD - 1) more |= i0 + BD < i1;
                    }
                }
                if (more) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int i0 = rbv[q] & 0xffffu, i1 = rbv[q] >> 16;
#pragma unroll 1  // rare: keep it small (unrolled, these 16 loops were a quarter of the kernel's code
                  // and the kernel stalled 19 % of the time on instruction fetch at N = 2^22)
                        for (int i = i0 + BD; i < i1; ++i) v[q] = cadd(v[q], buf[i]);
                    }
                }
#endif
                if constexpr (F2L) {
                    // the terms must have been read by every bin sum before the exchange
                    // first writes buf: wait there, after the first-level DFT
                    block_fft_2l<-1, false, NB_PA_TW2>(v, buf, tid, T, gsync, [&] { gsync(); });
                } else {
                    gsync();  // terms read before stage 1 reuses buf
                    block_fft_1buf<L2, -1>(v, buf, tid, T, gsync);
                }
                double2* out = Z + (long long)(r - p.r0) * N + (row << p.log_n2);
                if (TMA && chunk == 0) {
                    gsync();  // exchange reads done: buf becomes the staging box
                    double2* stg = buf + (((tid >> 5) * 16 + ((tid >> 1) & 15)) * 2 + (tid & 1));
#pragma unroll
                    for (int q = 0; q < 16; ++q) stg[256 * q] = UNIFORM ? v[q] : rot_ipow(v[q], r);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    gsync();  // box complete
                    if (tid == 0) {
                        const int z4 = (int)(((long long)(r - p.r0) << p.log_n1) + row);
                        asm volatile(
                            "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                                &zmap),
                            "r"(0), "r"(0), "r"(0), "r"(0), "r"(z4), "r"((unsigned)__cvta_generic_to_shared(buf))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const double2 z = UNIFORM ? v[q] : rot_ipow(v[q], r);
                        const int k2 = F2L ? fft2l_out_index(tid, q) : tid + q * G;
                        out[k2] = chunk == 0 ? z : cadd(out[k2], z);
                    }
                }
            }
            tm_wait_st();
        }
    }
    if (TMA && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    tm_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc(tmem_base, 512u);
}

// pass B: column k2 of every Z_r, inter-pass twiddle, N1-point FFT, v_r accumulate
template <int L1, bool UNIFORM>
__global__ void __launch_bounds__(L1 / 16, 1)
    k1_passB(const double2* __restrict__ Z, double2* __restrict__ f, PassBParams p) {
    constexpr int G = L1 / 16;
    extern __shared__ double2 smem[];
    double2* buf0 = smem;
    double2* buf1 = buf0 + padded_len(L1);
    double2* step = buf1 + padded_len(L1);
    double2* tw = step + 16;
    const int tid = threadIdx.x;
    twiddle_table_build<L1>(tw, tid, G);
    Twiddles<L1> T;
    twiddle_init<L1>(T, tw, tid);
    const long long n2 = 1ll << p.log_n2;
    const long long N = p.n;
    for (long long k2 = blockIdx.x; k2 < n2; k2 += gridDim.x) {
        __syncthreads();  // previous column's readers of step are done
        for (int q = tid; q < 16; q += G) step[q] = unit_root(k2 * q * G, N);  // w_N^{k2 q G}
        const double2 base = unit_root(k2 * tid, N);                          // w_N^{k2 tid}
        const double two_s0 = (double)(4 * ((((long long)tid) << p.log_n2) + k2)) / (double)N - 2.0;
        double tcur[16], tprev[16];
        double2 acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            acc[q] = make_double2(0.0, 0.0);
            tprev[q] = 1.0;
            tcur[q] = 0.5 * (two_s0 + 0.25 * q);
        }
        if constexpr (!UNIFORM) {
            for (int r = 1; r < p.r0; ++r) {
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
            const double2* col = Z + (long long)(r - p.r0) * N + k2;
            double2 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const long long t1 = tid + q * G;
                v[q] = cmul(__ldcg(col + (t1 << p.log_n2)), cmul(base, step[q]));
            }
            block_fft<L1, -1>(v, buf0, buf1, tid, T, [] { __syncthreads(); });
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                if constexpr (UNIFORM) {
                    acc[q] = cadd(acc[q], v[q]);
                } else {
                    const double vr = (r == 0) ? 0.5 : tcur[q];
                    acc[q].x = __fma_rn(vr, v[q].x, acc[q].x);
                    acc[q].y = __fma_rn(vr, v[q].y, acc[q].y);
                }
            }
            if constexpr (!UNIFORM) {
                if (r > 0) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const double tn = __fma_rn(two_s0 + 0.25 * q, tcur[q], -tprev[q]);
                        tprev[q] = tcur[q];
                        tcur[q] = tn;
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const long long k1 = tid + q * G;
            f[(k1 << p.log_n2) + k2] = p.conj ? cconj(acc[q]) : acc[q];
        }
    }
}

// Two-worker pass B (L1 = 2048, 4096): two independent column workers per CTA
// (columns 2*blockIdx + g, stride 2*gridDim) for twice the warps in flight;
// the accumulator and the Chebyshev state of each thread's 16 points live in
// tensor memory (tmem.cuh: 128 columns per thread, [acc re/im lo/hi x 16]
// [T_{r-1}, T_r lo/hi x 16]) instead of 128 registers, and each worker
// exchanges through one padded buffer of its own (as k2_pass1_tm, nufft2.cu).
// F2L (L1 = 4096): the column FFT is block_fft_2l (two group barriers per term
// instead of four); the thread's outputs are then k1 = k1_0 + 256 q with
// k1_0 = fft2l_out_index(tid, 0), so the accumulator slots, the Chebyshev
// arguments and the final f rows follow k1_0.
// TMA (with F2L): the Z column of each term is loaded by one 5-D
// cp.async.bulk.tensor load (4096 x 16 B, natural t1 order) into the worker's
// exchange buffer, issued as soon as the previous term's FFT has released the
// buffer so it overlaps the accumulator update; the FFT inputs then come from
// contiguous shared memory instead of 16 scattered global loads per thread.
template <int L1, bool UNIFORM, bool F2L = false, bool TMA = false>
__global__ void __launch_bounds__(2 * (L1 / 16), 1)
    k1_passB_tm(const double2* __restrict__ Z, double2* __restrict__ f, PassBParams p,
                const __grid_constant__ CUtensorMap zmap) {
    static_assert(!F2L || L1 == 4096, "two-level FFT is 4096-point");
    static_assert(!TMA || F2L || L1 == 2048, "TMA load path: the two-level kernel, or whole 2048-point columns");
    constexpr int G = L1 / 16;
    extern __shared__ __align__(1024) double2 smem[];
    __shared__ unsigned tmem_base;
    __shared__ __align__(8) unsigned long long colbar[4];  // per worker: [2 grp] first half, [2 grp + 1] second half
    const int grp = threadIdx.x / G;
    const int tid = threadIdx.x - grp * G;
    double2* buf = smem + grp * padded_len(L1);
    double2* step = smem + 2 * padded_len(L1) + grp * 16;
    double2* tw = smem + 2 * padded_len(L1) + 32;
    twiddle_table_build<L1>(tw, threadIdx.x, 2 * G);
    Twiddles<L1> T;
    twiddle_init<L1>(T, tw, tid);
    if (threadIdx.x < 32) tm_alloc(&tmem_base, 512u);
    if (TMA && tid == 0) {
        for (int h = 0; h < 2; ++h)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                             (unsigned)__cvta_generic_to_shared(&colbar[2 * grp + h]))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    const unsigned tcol = tm_lane_base(tmem_base) + (unsigned)((threadIdx.x >> 7) * 128);
    const unsigned tc_a = tcol, tc_s = tcol + 64;
    // the column of a term arrives in two 32 KiB halves: t1 < 2048 into a dedicated
    // buffer `pre` (issued a whole term ahead), t1 >= 2048 into the exchange buffer
    // (issued once the previous FFT has released it)
    // TMA without F2L (L1 = 2048): the whole 32 KiB column lands in `pre`, a term ahead; the
    // 16-byte loads at a 32 KiB stride it replaces cost the LSU one tag lookup per element
    // (2048 cycles per column-term and worker, 40 % of this kernel at cfg4)
    double2* pre = smem + 2 * padded_len(L1) + 32 + FftShapeX<L1>::TW_LEN + grp * 2048;
    const unsigned bar_s0 = (unsigned)__cvta_generic_to_shared(&colbar[2 * grp]);
    const unsigned bar_s1 = (unsigned)__cvta_generic_to_shared(&colbar[2 * grp + 1]);
    const unsigned buf_s = (unsigned)__cvta_generic_to_shared(smem + grp * padded_len(L1));
    const unsigned pre_s = (unsigned)__cvta_generic_to_shared(pre);
    int col_phase = 0;
    // TMA without F2L: the engine moves 0.61 pieces per clock per SM (scripts/microbench_tma_load.cu),
    // which made a whole 2048-piece column per term the kernel's bound; the last QL of the
    // thread's 16 inputs (t1 >= 2048 - 128 QL) come through the LSU instead, a term ahead
    constexpr int QL = (TMA && !F2L) ? NB_PB_QL : 0;
    constexpr unsigned kBoxBytes = (TMA && !F2L) ? (16 - QL) * 128 * 16 : 32768;
    auto col_load = [&](int half, int rr, long long kk2) {  // thread 0 of the worker
        const unsigned bs = half ? bar_s1 : bar_s0;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bs), "r"(kBoxBytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
            "%6}], [%7];" ::"r"(half ? buf_s : pre_s),
            "l"(&zmap), "r"(0), "r"(0), "r"(8 * half), "r"(rr), "r"((int)kk2), "r"(bs)
            : "memory");
    };
    auto col_wait = [&](unsigned bs, int ph) {
        asm volatile(
            "{\n\t.reg .pred P;\n"
            "CBW_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
            "@!P bra CBW_%=;\n}" ::"r"(bs),
            "r"(ph)
            : "memory");
    };
    const int bar = 1 + grp;
    auto gsync = [bar] {
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G) : "memory");
    };
    const long long n2 = 1ll << p.log_n2;
    const long long N = p.n;
    for (long long k2 = 2ll * blockIdx.x + grp; k2 < n2; k2 += 2ll * gridDim.x) {
        gsync();  // previous column's readers of step are done
        for (int q = tid; q < 16; q += G) step[q] = unit_root(k2 * q * G, N);  // w_N^{k2 q G}
        const double2 base = unit_root(k2 * tid, N);                          // w_N^{k2 tid}
        const int k1_0 = F2L ? fft2l_out_index(tid, 0) : tid;                 // first output row
        const double two_s0 = (double)(4 * ((((long long)k1_0) << p.log_n2) + k2)) / (double)N - 2.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // acc = 0, state (T_{r0-1}, T_r0)
            unsigned av[16], sv[16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double ts = two_s0 + 0.25 * (4 * j + u);
                double tprev = 1.0, tcur = 0.5 * ts;
                for (int r = 1; r < p.r0; ++r) {
                    const double tn = __fma_rn(ts, tcur, -tprev);
                    tprev = tcur;
                    tcur = tn;
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) av[4 * u + c] = 0u;
                sv[4 * u] = lo32(tprev);
                sv[4 * u + 1] = hi32(tprev);
                sv[4 * u + 2] = lo32(tcur);
                sv[4 * u + 3] = hi32(tcur);
            }
            tm_st16(tc_a + 16 * j, av);
            if constexpr (!UNIFORM) tm_st16(tc_s + 16 * j, sv);
        }
        tm_wait_st();
        if constexpr (TMA) {
            gsync();  // the previous column's last exchange reads of buf / pre are done
            if (tid == 0) {
                col_load(0, 0, k2);
                if constexpr (F2L) col_load(1, 0, k2);
            }
        }
        gsync();  // step visible
        // L1 = 2048 runs 256 threads per CTA (registers to spare): the next term's column is
        // loaded into nx while this term transforms, instead of 16 exposed strided loads per
        // term (long-scoreboard stalls were 30 % of this kernel at cfg4)
        constexpr bool PF = NB_PB_PF && !TMA && L1 == 2048;
        double2 nx[PF ? 16 : 1];
        if constexpr (PF) {
            const double2* col = Z + k2;
#pragma unroll
            for (int q = 0; q < 16; ++q) nx[q] = __ldcg(col + ((long long)(tid + q * G) << p.log_n2));
        }
        double2 nl[QL > 0 ? QL : 1];
        if constexpr (QL > 0) {
            const double2* col = Z + k2;
#pragma unroll
            for (int q = 16 - QL; q < 16; ++q) nl[q - (16 - QL)] = __ldcg(col + ((long long)(tid + q * G) << p.log_n2));
        }
        for (int r = p.r0; r < p.r1; ++r) {
            double2 v[16];
            if constexpr (TMA && F2L) {
                col_wait(bar_s0, col_phase);
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = q == 0 ? pre[tid] : cmul(pre[tid + q * G], step[q]);
                col_wait(bar_s1, col_phase);
                col_phase ^= 1;
#pragma unroll
                for (int q = 8; q < 16; ++q) v[q] = cmul(buf[tid + (q - 8) * G], step[q]);
            } else if constexpr (TMA) {
                col_wait(bar_s0, col_phase);
                col_phase ^= 1;
#pragma unroll
                for (int q = 0; q < 16 - QL; ++q) v[q] = cmul(pre[tid + q * G], cmul(base, step[q]));
                if constexpr (QL > 0) {
#pragma unroll
                    for (int q = 16 - QL; q < 16; ++q) v[q] = cmul(nl[q - (16 - QL)], cmul(base, step[q]));
                    if (r + 1 < p.r1) {
                        const double2* col = Z + (long long)(r + 1 - p.r0) * N + k2;
#pragma unroll
                        for (int q = 16 - QL; q < 16; ++q)
                            nl[q - (16 - QL)] = __ldcg(col + ((long long)(tid + q * G) << p.log_n2));
                    }
                }
            } else if constexpr (PF) {
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] = cmul(nx[q], cmul(base, step[q]));
                if (r + 1 < p.r1) {
                    const double2* col = Z + (long long)(r + 1 - p.r0) * N + k2;
#pragma unroll
                    for (int q = 0; q < 16; ++q) nx[q] = __ldcg(col + ((long long)(tid + q * G) << p.log_n2));
                }
            } else {
                const double2* col = Z + (long long)(r - p.r0) * N + k2;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const long long t1 = tid + q * G;
                    v[q] = cmul(__ldcg(col + (t1 << p.log_n2)), cmul(base, step[q]));
                }
            }
            gsync();  // previous term's last-stage reads of buf (and this term's inputs) are done
            if constexpr (TMA) {
                if (tid == 0 && r + 1 < p.r1) col_load(0, r + 1 - p.r0, k2);  // pre is free: a whole term ahead
            }
            if constexpr (TMA && F2L) {
                // the inter-pass twiddle w_N^{k2 (tid + 256 q)} = base * step[q]: step[q] on
                // the inputs above, the thread constant base with the first-level twiddles
                block_fft_2l<-1, true, NB_PB_TW2>(v, buf, tid, T, gsync, NoHook(), base);
            } else if constexpr (F2L) {
                block_fft_2l<-1, false, NB_PB_TW2>(v, buf, tid, T, gsync);
            } else {
                block_fft_1buf<L1, -1>(v, buf, tid, T, gsync);
            }
            if constexpr (TMA && F2L) {
                if (r + 1 < p.r1) {
                    gsync();  // exchange reads done: the next term's second half may land in buf
                    if (tid == 0) col_load(1, r + 1 - p.r0, k2);
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                unsigned av[16], sv[16];
                tm_ld16(tc_a + 16 * j, av);
                if constexpr (!UNIFORM) tm_ld16(tc_s + 16 * j, sv);
                tm_wait_ld();
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = 4 * j + u;
                    double2 a = make_double2(mk64(av[4 * u], av[4 * u + 1]), mk64(av[4 * u + 2], av[4 * u + 3]));
                    if constexpr (UNIFORM) {
                        a = cadd(a, v[q]);
                    } else {
                        const double tprev = mk64(sv[4 * u], sv[4 * u + 1]);
                        const double tcur = mk64(sv[4 * u + 2], sv[4 * u + 3]);
                        const double vr = (r == 0) ? 0.5 : tcur;
                        a.x = __fma_rn(vr, v[q].x, a.x);
                        a.y = __fma_rn(vr, v[q].y, a.y);
                        if (r > 0) {
                            const double tn = __fma_rn(two_s0 + 0.25 * q, tcur, -tprev);
                            sv[4 * u] = sv[4 * u + 2];
                            sv[4 * u + 1] = sv[4 * u + 3];
                            sv[4 * u + 2] = lo32(tn);
                            sv[4 * u + 3] = hi32(tn);
                        }
                    }
                    av[4 * u] = lo32(a.x);
                    av[4 * u + 1] = hi32(a.x);
                    av[4 * u + 2] = lo32(a.y);
                    av[4 * u + 3] = hi32(a.y);
                }
                tm_st16(tc_a + 16 * j, av);
                if constexpr (!UNIFORM) {
                    if (r > 0) tm_st16(tc_s + 16 * j, sv);
                }
            }
        }
        tm_wait_st();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            unsigned av[16];
            tm_ld16(tc_a + 16 * j, av);
            tm_wait_ld();
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long k1 = k1_0 + (4 * j + u) * G;
                const double2 fv = make_double2(mk64(av[4 * u], av[4 * u + 1]), mk64(av[4 * u + 2], av[4 * u + 3]));
                f[(k1 << p.log_n2) + k2] = p.conj ? cconj(fv) : fv;
            }
        }
    }
    tm_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc(tmem_base, 512u);
}

// N1 == 1: f[k] = sum_r v_r(k) Z_r[k]
__global__ void k1_combine(const double2* __restrict__ Z, double2* __restrict__ f, long long N,
                           int r0, int r1, int uniform, int conj) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const double s = __dsub_rn(__dmul_rn(2.0, (double)k / (double)N), 1.0);
    double tprev = 1.0, tcur = s;
    double2 acc = make_double2(0.0, 0.0);
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
        if (r < r0) continue;
        const double2 z = Z[(long long)(r - r0) * N + k];
        if (uniform) {
            acc = cadd(acc, z);
        } else {
            acc.x = __fma_rn(vr, z.x, acc.x);
            acc.y = __fma_rn(vr, z.y, acc.y);
        }
    }
    f[k] = conj ? cconj(acc) : acc;
}

// Z columns (rr*N + t1*4096 + k2, N1 = 2^log_n1 rows) as the 5-D tensor k1_passB_tm<.., TMA>
// loads from: (re/im, t1 & 255, t1 >> 8, rr, k2), box = half a column of one term
bool make_zcol_tensor_map(CUtensorMap* map, const double2* Z, int log_n1, int log_n2, int nterms, int box_hi = 8) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }();
    if (!encode || (log_n1 != 12 && log_n1 != 11)) return false;
    const cuuint64_t n1 = 1ull << log_n1, n2 = 1ull << log_n2;
    const cuuint64_t row = n2 * 16ull;  // bytes per t1
    // a box is 2048 pieces of 16 B (32 KiB): half a column at N1 = 4096, a whole one at 2048
    cuuint64_t dims[5] = {2, 256, n1 / 256, (cuuint64_t)nterms, n2};
    cuuint64_t strides[4] = {row, 256 * row, n1 * row, 16};
    cuuint32_t box[5] = {2, 256, (cuuint32_t)box_hi, 1, 1};  // box_hi * 256 pieces
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)Z, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Z (row-major rr*N + row*4096 + k2) as the 5-D tensor k1_passA_tm<.., TMA> stores into
bool make_z_tensor_map(CUtensorMap* map, double2* Z, int log_n1, int nterms) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }();
    if (!encode) return false;
    const cuuint64_t rows = (cuuint64_t)nterms << log_n1;
    cuuint64_t dims[5] = {4, 16, 8, 16, rows};
    cuuint64_t strides[4] = {256, 32, 4096, 65536};  // bytes: u, warp, b, (rr, row)
    cuuint32_t box[5] = {4, 16, 8, 16, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)Z, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

// nb > 1 (L2 = 2048 only, passA_stackable): nb vectors g + b N -> Z + b (r1 - r0) N in one launch
template <int L2>
void launch_passA(const double2* g, double2* Z, const CorePlan& pl, int r0, int r1, bool conj, cudaStream_t s,
                  int nb = 1) {
    const DeviceCtx& ctx = DeviceCtx::get(pl.device);
    constexpr size_t SM = PassAShape<L2>::SMEM;
    if (nb > 1 && L2 != 2048) throw Error(kInternal, "stacked pass A");
    PassAParams p{};
    p.nb = nb;
    p.gstride = (long long)pl.n;
    p.zstride = (long long)pl.n * (r1 - r0);
    p.conj = conj ? 1 : 0;
    p.n = (long long)pl.n;
    p.log_n1 = pl.bk.log_n1;
    p.log_n2 = pl.bk.log_n2;
    p.r0 = r0;
    p.r1 = r1;
    p.ds = pl.bk.ds.as<double>();
    p.skey = pl.bk.skey.as<unsigned>();
    p.perm = pl.bk.perm.as<int>();
    p.rowoff = pl.bk.rowoff.as<int>();
    for (size_t r = 0; r < pl.series_deg.size() && r < (size_t)kRankCap; ++r) p.deg[r] = pl.series_deg[r];
    if constexpr (L2 == 4096) {
        constexpr size_t SMT = PassATmShape<L2>::SMEM;
        // two-level row FFT; Z rows stored by TMA (LSU stores when the tensor map
        // cannot describe Z)
        const bool crowded = pl.bk.crowded.empty() || pl.bk.crowded[0] != 0;
        auto fnt = pl.uniform ? k1_passA_tm<L2, true, true> : k1_passA_tm<L2, false, true>;
        CUtensorMap zmap{};
        if (make_z_tensor_map(&zmap, Z, pl.bk.log_n1, r1 - r0)) {
            fnt = pl.uniform ? k1_passA_tm<L2, true, true, true> : k1_passA_tm<L2, false, true, true>;
            if (crowded && !pl.uniform) fnt = k1_passA_tm<L2, false, true, true, 2, 4>;
        } else if (crowded && !pl.uniform) {
            fnt = k1_passA_tm<L2, false, true, false, 2, 4>;
        }
        set_smem(fnt, SMT);
        const long long rows = 1ll << pl.bk.log_n1;
        const int gridt = (int)std::min<long long>((rows + 1) / 2, (long long)ctx.sms);
        fnt<<<gridt, 2 * (L2 / 16), SMT, s>>>(g, Z, p, zmap);
        NB_LAUNCH();
        return;
    }
    if constexpr (L2 == 2048) {
        // four row workers of 128 threads (16 warps/SM) with the per-sample state in TMEM:
        // the cfg4 inner type-I transforms 30.3 -> 27.1 ms per type-III exec (a jittered
        // type I at 2^22: 1.44 -> 1.47 ms); two workers measured 1.63 ms
        using S4 = PassATmShape<L2, 4>;
        const bool crowded = pl.bk.crowded.empty() || pl.bk.crowded[0] != 0;
        auto f4 = pl.uniform ? k1_passA_tm<L2, true, false, false, 4> : k1_passA_tm<L2, false, false, false, 4>;
        if (crowded && !pl.uniform) f4 = k1_passA_tm<L2, false, false, false, 4, 4>;
        CUtensorMap zmap{};
        set_smem(f4, S4::SMEM);
        const long long rows = (1ll << pl.bk.log_n1) * nb;
        const int grid4 = (int)std::min<long long>((rows + 3) / 4, (long long)ctx.sms);
        f4<<<grid4, 4 * (L2 / 16), S4::SMEM, s>>>(g, Z, p, zmap);
        NB_LAUNCH();
        return;
    }
    auto fn = pl.uniform ? k1_passA<L2, true> : k1_passA<L2, false>;
    set_smem(fn, SM);
    const long long n1 = 1ll << pl.bk.log_n1;
    const int grid = (int)std::min<long long>(n1, (long long)ctx.sms * occupancy((const void*)fn, L2 / 16, SM));
    fn<<<grid, L2 / 16, SM, s>>>(g, Z, p);
    NB_LAUNCH();
}

template <int L1>
void launch_passB(const double2* Z, double2* f, const CorePlan& pl, int r0, int r1, bool conj, cudaStream_t s) {
    const DeviceCtx& ctx = DeviceCtx::get(pl.device);
    if constexpr (L1 >= 2048) {
        size_t SMT = sizeof(double2) * (2 * padded_len(L1) + 32 + FftShapeX<L1>::TW_LEN);
        PassBParams p{(long long)pl.n, pl.bk.log_n1, pl.bk.log_n2, r0, r1, conj ? 1 : 0};
        auto fn = pl.uniform ? k1_passB_tm<L1, true> : k1_passB_tm<L1, false>;
        CUtensorMap zmap{};
        if constexpr (L1 == 2048) {
            // Z columns (32 KiB) loaded by TMA a term ahead
            if (NB_PB_TMA2048 && make_zcol_tensor_map(&zmap, Z, pl.bk.log_n1, pl.bk.log_n2, r1 - r0, (16 - NB_PB_QL) / 2)) {
                fn = pl.uniform ? k1_passB_tm<L1, true, false, true> : k1_passB_tm<L1, false, false, true>;
                SMT += sizeof(double2) * 2 * 2048;  // the two `pre` column buffers
            }
        }
        if constexpr (L1 == 4096) {
            // two-level column FFT; Z columns loaded by TMA when N2 = 4096
            fn = pl.uniform ? k1_passB_tm<L1, true, true> : k1_passB_tm<L1, false, true>;
            if (pl.bk.log_n2 == 12 && make_zcol_tensor_map(&zmap, Z, pl.bk.log_n1, pl.bk.log_n2, r1 - r0)) {
                fn = pl.uniform ? k1_passB_tm<L1, true, true, true> : k1_passB_tm<L1, false, true, true>;
                SMT += sizeof(double2) * 2 * 2048;  // the two `pre` half-column buffers
            }
        }
        set_smem(fn, SMT);
        const long long n2 = 1ll << pl.bk.log_n2;
        const int grid = (int)std::min<long long>((n2 + 1) / 2, (long long)ctx.sms);
        fn<<<grid, 2 * (L1 / 16), SMT, s>>>(Z, f, p, zmap);
        NB_LAUNCH();
        return;
    }
    constexpr size_t SM = sizeof(double2) * (2 * padded_len(L1) + 16 + FftShapeX<L1>::TW_LEN);
    PassBParams p{(long long)pl.n, pl.bk.log_n1, pl.bk.log_n2, r0, r1, conj ? 1 : 0};
    auto fn = pl.uniform ? k1_passB<L1, true> : k1_passB<L1, false>;
    set_smem(fn, SM);
    const long long n2 = 1ll << pl.bk.log_n2;
    const int grid = (int)std::min<long long>(n2, (long long)ctx.sms * occupancy((const void*)fn, L1 / 16, SM));
    fn<<<grid, L1 / 16, SM, s>>>(Z, f, p);
    NB_LAUNCH();
}

void dispatch_passA(int L, const double2* g, double2* Z, const CorePlan& pl, int r0, int r1, bool conj, cudaStream_t s,
                    int nb = 1) {
    if (nb > 1) return launch_passA<2048>(g, Z, pl, r0, r1, conj, s, nb);
    switch (L) {
        case 16: return launch_passA<16>(g, Z, pl, r0, r1, conj, s);
        case 32: return launch_passA<32>(g, Z, pl, r0, r1, conj, s);
        case 64: return launch_passA<64>(g, Z, pl, r0, r1, conj, s);
        case 128: return launch_passA<128>(g, Z, pl, r0, r1, conj, s);
        case 256: return launch_passA<256>(g, Z, pl, r0, r1, conj, s);
        case 512: return launch_passA<512>(g, Z, pl, r0, r1, conj, s);
        case 1024: return launch_passA<1024>(g, Z, pl, r0, r1, conj, s);
        case 2048: return launch_passA<2048>(g, Z, pl, r0, r1, conj, s);
        case 4096: return launch_passA<4096>(g, Z, pl, r0, r1, conj, s);
        default: throw Error(kInternal, "pass A size");
    }
}

void dispatch_passB(int L, const double2* Z, double2* f, const CorePlan& pl, int r0, int r1, bool conj, cudaStream_t s) {
    switch (L) {
        case 16: return launch_passB<16>(Z, f, pl, r0, r1, conj, s);
        case 32: return launch_passB<32>(Z, f, pl, r0, r1, conj, s);
        case 64: return launch_passB<64>(Z, f, pl, r0, r1, conj, s);
        case 128: return launch_passB<128>(Z, f, pl, r0, r1, conj, s);
        case 256: return launch_passB<256>(Z, f, pl, r0, r1, conj, s);
        case 512: return launch_passB<512>(Z, f, pl, r0, r1, conj, s);
        case 1024: return launch_passB<1024>(Z, f, pl, r0, r1, conj, s);
        case 2048: return launch_passB<2048>(Z, f, pl, r0, r1, conj, s);
        case 4096: return launch_passB<4096>(Z, f, pl, r0, r1, conj, s);
        default: throw Error(kInternal, "pass B size");
    }
}

}  // namespace

void exec_transpose_fused(const CorePlan& pl, const double2* g, double2* f, size_t batch,
                          cudaStream_t s, cudaEvent_t* ev, size_t r_begin, size_t r_end, bool conj) {
    ensure_bessel_constants(pl.device);
    const size_t N = pl.n;
    const int r0 = (int)r_begin, r1 = (int)std::min(r_end, pl.K);
    if (r1 <= r0) {  // no terms: zero output
        NB_CUDA(cudaMemsetAsync(f, 0, sizeof(double2) * N * batch, s));
        return;
    }
    const int L1 = 1 << pl.bk.log_n1, L2 = 1 << pl.bk.log_n2;
    // L2 = 2048 (N = 2^22, 2^21): 2048 or 1024 rows over 4 x 148 row workers leave the last wave
    // of a launch half empty (3.46 rows per worker: 86 %); kStack vectors per pass-A launch
    // fill it (13.8 rows per worker: 99 %).  Type III runs its K inner transforms this way.
    constexpr size_t kStack = 4;
    const size_t stack = (L2 == 2048 && pl.bk.log_n1 > 0 && !ev) ? std::min(batch, kStack) : 1;
    const size_t zlen = N * (size_t)(r1 - r0);
    DevBuf Z(sizeof(double2) * zlen * stack, s);
    for (size_t b = 0; b < batch; ++b) {
        if (ev && b == 0) NB_CUDA(cudaEventRecord(ev[0], s));
        if (stack > 1) {
            if (b % stack == 0)
                dispatch_passA(L2, g + b * N, Z.as<double2>(), pl, r0, r1, conj, s, (int)std::min(stack, batch - b));
            dispatch_passB(L1, Z.as<double2>() + (b % stack) * zlen, f + b * N, pl, r0, r1, conj, s);
            continue;
        }
        dispatch_passA(L2, g + b * N, Z.as<double2>(), pl, r0, r1, conj, s);
        if (ev && b == 0) NB_CUDA(cudaEventRecord(ev[1], s));
        if (pl.bk.log_n1 == 0) {
            k1_combine<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(Z.as<double2>(), f + b * N, (long long)N,
                                                                 r0, r1, pl.uniform ? 1 : 0, conj ? 1 : 0);
            NB_LAUNCH();
        } else {
            dispatch_passB(L1, Z.as<double2>(), f + b * N, pl, r0, r1, conj, s);
        }
        if (ev && b == 0) NB_CUDA(cudaEventRecord(ev[2], s));
    }
}

}  // namespace nb
