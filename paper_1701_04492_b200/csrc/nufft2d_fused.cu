// Fused 2D type-II execution (power-of-two grids, 16 <= m, n <= 4096).
//
// Reference: exec_nufft2d2_impl transform2d.hpp:107-147
//   f_j = sum_{r1<Kx} sum_{r2<Ky} ux_r1[j] uy_r2[j] [F_m D_vy_r2 C D_vx_r1 F_n^T](ty_j, tx_j)
// evaluated by the reference as Kx row stages (m FFTs of size n, reused over
// r2) and Kx*Ky column stages (n FFTs of size m), each followed by a gather
// over all samples.  Here:
//
//  row kernel (CTA per row ky, persistent): the C row is read once into
//    shared memory; for every r1 it is scaled by vx_r1(kx) (Chebyshev state in
//    registers), transformed (n-point FFT) and R_r1[ky][tx] is written
//    (row-major, full sectors) — the only HBM round trip of the row stage.
//  column kernel (CTA per column tx, persistent): the samples with tx_j = tx
//    (plan-time stable sort) stay in shared memory/registers for all Kx*Ky
//    terms.  For r1 = Kx-1..0 the column R_r1[:][tx] is staged in shared
//    memory once; for r2 = Ky-1..0 the column is scaled by vy_r2 (a Ky x m
//    table, L2-resident), transformed (m-point FFT) and every sample updates
//        S_j <- S_j (i hy_j) + gy_r2(hy_j^2) X[ty_j]              (Horner in r2),
//    then A_j <- A_j (i hx_j) + gx_r1(hx_j^2) S_j                 (Horner in r1,
//    A_j in an HBM scratch in sorted order, coalesced), and finally
//    f_j = 4 exp(2i(hx_j + hy_j)) A_j — the Bessel form of the reference's
//    ux*uy (bessel.cuh) without materializing either factor.
//
// HBM bytes: C 16 mn + R 32 Kx mn + A 32 Kx count + f 16 count + sample data;
// the Kx*Ky column FFTs never leave the SM.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>

#include "bessel.cuh"
#include "fft_block.cuh"
#include "plans.hpp"
#include "tmem.cuh"

// second-level twiddle mode of block_fft_2l (fft_block.cuh) per kernel
#ifndef NB_2DR_TW2
#define NB_2DR_TW2 4
#endif
#ifndef NB_2DC_TW2
#define NB_2DC_TW2 4
#endif

namespace nb {

namespace {

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// z (i h)^r0: the Horner-in-r1 sum of a partial term range [r0, r1hi) (multi-GPU r1 split)
__device__ __forceinline__ double2 ipow_scale(double2 z, double h, int r0) {
    if (r0 == 0) return z;
    double hr = 1.0;
    for (int m = 0; m < r0; ++m) hr *= h;
    z = cscale(z, hr);
    switch (r0 & 3) {
        case 1: return make_double2(-z.y, z.x);
        case 2: return make_double2(-z.x, -z.y);
        case 3: return make_double2(z.y, -z.x);
        default: return z;
    }
}

constexpr int kQ2d = 20;  // samples per column-kernel thread (capacity 1.25 m per chunk)

struct RowParams {
    long long m, n;
    int log_n;
    int kx;
    int ux_uniform;
    int r1lo, r1hi;  // row-stage terms [r1lo, r1hi) (multi-GPU r1 split); R slice r1 - r1lo
};

struct ColParams {
    long long m, n;
    int log_n;
    int kx, ky;
    int ux_uniform, uy_uniform;
    const double* dxs;
    const double* dys;
    const unsigned short* tys;
    const int* perm;
    const int* coloff;
    const double* vyt;  // ky x m
    double2* A;         // sorted-order scratch
    int degx[kRankCap];
    int degy[kRankCap];
    int r1lo, r1hi;     // r1 terms [r1lo, r1hi) of this launch; R slice r1 - r1lo
};

// ---------------------------------------------------------------- row stage
template <int LN>
__global__ void __launch_bounds__(LN / 16, 1)
    k2d_rows(const double2* __restrict__ C, double2* __restrict__ R, RowParams p) {
    constexpr int G = LN / 16;
    extern __shared__ double2 smem[];
    double2* crow = smem;
    double2* buf0 = crow + LN;
    double2* buf1 = buf0 + padded_len(LN);
    double2* tw = buf1 + padded_len(LN);
    const int tid = threadIdx.x;
    twiddle_table_build<LN>(tw, tid, G);
    Twiddles<LN> T;
    twiddle_init<LN>(T, tw, tid);
    const long long mn = p.m * p.n;
    // 2 s_q = 4 kx / n - 2 with kx = tid + q G  ->  two_s0 + q/4 (exact)
    const double two_s0 = (double)(4 * tid) / (double)p.n - 2.0;
    for (long long ky = blockIdx.x; ky < p.m; ky += gridDim.x) {
        __syncthreads();  // previous row's readers of crow are done
#pragma unroll
        for (int q = 0; q < 16; ++q) crow[tid + q * G] = __ldcs(C + ky * p.n + tid + q * G);
        double tcur[16], tprev[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            tprev[q] = 1.0;
            tcur[q] = 0.5 * (two_s0 + 0.25 * q);
        }
        __syncthreads();
        for (int r = 0; r < p.r1hi; ++r) {
            if (r < p.r1lo) {  // advance the recurrence to the first term of the range
                if (r > 0) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const double tn = __fma_rn(two_s0 + 0.25 * q, tcur[q], -tprev[q]);
                        tprev[q] = tcur[q];
                        tcur[q] = tn;
                    }
                }
                continue;
            }
            if constexpr (FftShape<LN>::STAGES < 3) __syncthreads();
            double2 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 cv = crow[tid + q * G];
                const double vr = p.ux_uniform ? 1.0 : ((r == 0) ? 0.5 : tcur[q]);
                v[q] = make_double2(cv.x * vr, cv.y * vr);
            }
            block_fft<LN, -1>(v, buf0, buf1, tid, T, [] { __syncthreads(); });
            double2* out = R + (long long)(r - p.r1lo) * mn + ky * p.n;
#pragma unroll
            for (int q = 0; q < 16; ++q) out[tid + q * G] = v[q];
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
}

// ---------------------------------------------------------------- column stage
template <int LM>
struct ColShape {
    static constexpr int G = LM / 16;
    static constexpr int CAP = kQ2d * G;
    static constexpr size_t SMEM = sizeof(double2) * (LM + padded_len(LM) + FftShapeX<LM>::TW_LEN) +
                                   (sizeof(double) + sizeof(unsigned short)) * CAP;
    static_assert(SMEM <= 227 * 1024, "column kernel shared memory");
};

template <int LM>
__global__ void __launch_bounds__(LM / 16, 1)
    k2d_cols(const double2* __restrict__ R, double2* __restrict__ f, ColParams p) {
    using S = ColShape<LM>;
    constexpr int G = S::G;
    constexpr int Q = kQ2d;
    constexpr int CAP = S::CAP;
    constexpr int CH = 4;  // Horner chunk (independent FMA chains per coefficient)
    extern __shared__ double2 smem[];
    double2* rcol = smem;
    double2* buf = rcol + LM;  // FFT exchange; holds X between the FFT and the gathers
    double2* tw = buf + padded_len(LM);
    double* shy = reinterpret_cast<double*>(tw + FftShapeX<LM>::TW_LEN);
    unsigned short* sty = reinterpret_cast<unsigned short*>(shy + CAP);
    const int tid = threadIdx.x;
    twiddle_table_build<LM>(tw, tid, G);
    Twiddles<LM> T;
    twiddle_init<LM>(T, tw, tid);
    __syncthreads();
    const long long mn = p.m * p.n;
    for (long long tx = blockIdx.x; tx < p.n; tx += gridDim.x) {
        const int beg = p.coloff[tx], end = p.coloff[tx + 1];
        for (int cb = beg; cb < end; cb += CAP) {
            const int cnt = min(CAP, end - cb);
            __syncthreads();  // previous chunk's readers of shy / sty are done
            for (int i = tid; i < CAP; i += G) {
                const bool ok = i < cnt;
                shy[i] = (ok && !p.uy_uniform) ? half_phase(p.dys[cb + i]) : 0.0;
                // gather slot of X[ty]: natural index, or its place after the two-level FFT
                sty[i] = ok ? (unsigned short)(LM == 4096 ? fft2l_slot_of(p.tys[cb + i]) : p.tys[cb + i])
                            : (unsigned short)0;
            }
            for (int r1 = p.r1hi - 1; r1 >= p.r1lo; --r1) {
                __syncthreads();  // previous term's gathers from buf / reads of rcol done
                const double2* col = R + (long long)(r1 - p.r1lo) * mn + tx;
#pragma unroll
                for (int q = 0; q < 16; ++q) rcol[tid + q * G] = __ldcs(col + (long long)(tid + q * G) * p.n);
                double2 acc[Q];
#pragma unroll
                for (int u = 0; u < Q; ++u) acc[u] = make_double2(0.0, 0.0);
                for (int r2 = p.ky - 1; r2 >= 0; --r2) {
                    double2 v[16];
                    const double* vy = p.vyt + (long long)r2 * p.m;
                    __syncthreads();  // rcol visible; previous gathers from buf done
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = cscale(rcol[tid + q * G], __ldg(vy + tid + q * G));
                    if constexpr (LM == 4096) {  // two-level FFT, X left in place (fft2l_slot)
                        block_fft_2l<-1, false, NB_2DR_TW2>(v, buf, tid, T, [] { __syncthreads(); });
#pragma unroll
                        for (int q = 0; q < 16; ++q) buf[fft2l_slot(tid, q)] = v[q];
                    } else {
                        block_fft_1buf<LM, -1>(v, buf, tid, T, [] { __syncthreads(); });
                        __syncthreads();  // last-stage reads of buf done
#pragma unroll
                        for (int q = 0; q < 16; ++q) buf[tid + q * G] = v[q];
                    }
                    __syncthreads();
                    // S <- S (i hy) + gy_r2(hy^2) X[ty]
                    const double* a = kBes + r2 * kSeriesTerms;
                    const int deg = p.degy[r2];
#pragma unroll
                    for (int u0 = 0; u0 < Q; u0 += CH) {
                        double h[CH], w[CH], g[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            h[c] = shy[tid + (u0 + c) * G];
                            w[c] = h[c] * h[c];
                            g[c] = 0.0;
                        }
                        if (p.uy_uniform) {
#pragma unroll
                            for (int c = 0; c < CH; ++c) g[c] = 1.0;
                        } else {
                            for (int m = deg; m >= 0; --m) {
                                const double am = a[m];
#pragma unroll
                                for (int c = 0; c < CH; ++c) g[c] = __fma_rn(g[c], w[c], am);
                            }
                        }
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            const int u = u0 + c;
                            const double2 X = buf[sty[tid + u * G]];
                            const double ax = acc[u].x;
                            acc[u].x = __fma_rn(g[c], X.x, -h[c] * acc[u].y);
                            acc[u].y = __fma_rn(g[c], X.y, h[c] * ax);
                        }
                    }
                }
                // A <- A (i hx) + gx_r1(hx^2) S ; the last term writes f
                const double* a = kBes + r1 * kSeriesTerms;
                const int deg = p.degx[r1];
#pragma unroll
                for (int u = 0; u < Q; ++u) {
                    const int i = tid + u * G;
                    if (i >= cnt) continue;
                    const double hx = p.ux_uniform ? 0.0 : half_phase(p.dxs[cb + i]);
                    double gx = 1.0;
                    if (!p.ux_uniform) {
                        const double w = hx * hx;
                        gx = 0.0;
                        for (int m = deg; m >= 0; --m) gx = __fma_rn(gx, w, a[m]);
                    }
                    double2 A = cscale(acc[u], gx);
                    if (r1 != p.r1hi - 1) {
                        const double2 prev = p.A[cb + i];
                        A.x = __fma_rn(-hx, prev.y, A.x);
                        A.y = __fma_rn(hx, prev.x, A.y);
                    }
                    if (r1 > p.r1lo) {
                        p.A[cb + i] = A;
                    } else {
                        A = ipow_scale(A, hx, p.r1lo);
                        double ph = 0.0, scale = 1.0;
                        if (!p.ux_uniform) {
                            ph += 2.0 * hx;
                            scale *= 2.0;
                        }
                        if (!p.uy_uniform) {
                            ph += 2.0 * shy[i];
                            scale *= 2.0;
                        }
                        double sn = 0.0, cs = 1.0;
                        if (ph != 0.0) sincos(ph, &sn, &cs);
                        __stcs(f + p.perm[cb + i], cmul(make_double2(scale * cs, scale * sn), A));
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------- column stage, m = 4096
// Two FFT groups of 256 threads alternate the Kx*Ky column steps of a unit
// (column tx, <= 4608 samples), the organization of the type-II fused pass 2
// (k2_pass2_fs, nufft2.cu) with one more loop level:
//   per r1 (outer, Kx-1 .. 0): the R_r1 column is staged in shared memory once;
//     per r2 (Ky-1 .. 0), group (step % 2): v = vy_r2 .* column, two-level FFT,
//     X left in place in the group's buffer; then, after the other group's
//     update of the previous step (named-barrier hand-off), every sample of the
//     unit: S <- S (i hy) + gy_r2 X[ty], gy_{r2-1} = r2 gy_r2 - hy^2 gy_{r2+1}
//     (backward Bessel recurrence) — state (S, gy pair, hy, slot, hx) in TMEM;
//   block end: A <- A (i hx) + gx_r1(hx^2) S with A in a sorted-order HBM
//     scratch (coalesced), and for r1 = 0 f[perm] = 4 exp(2i(hx + hy)) A.
// The FFT of one group overlaps the sample update of the other; each step
// moves no HBM bytes except the L2-resident vy row.
struct Col2Shape {
    static constexpr int G = 256;
    static constexpr int SLOTS = 18;  // CAP = 4608 = 1.125 x 4096 samples per unit
    static constexpr int CAP = SLOTS * G;
    static constexpr int CH = 2;
    static constexpr int COL_S = 0, COL_G = 4 * SLOTS, COL_HY = 8 * SLOTS, COL_T = 10 * SLOTS,
                         COL_HX = 11 * SLOTS, COLS = 13 * SLOTS;
    static constexpr size_t SMEM = sizeof(double2) * (3 * kBuf2l + FftShapeX<4096>::TW_LEN);
    static_assert(COLS <= 256 && SLOTS % CH == 0, "TMEM layout");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

struct Col2Params {
    long long m, n;
    int kx, ky;
    int ux_uniform, uy_uniform;
    const double* dxs;
    const double* dys;
    const unsigned short* tys;
    const int* perm;
    const int* coloff;
    const double* vyt;  // ky x m
    double2* A;         // sorted-order scratch
    int degx[kRankCap];
    int degy_top0, degy_top1;  // relative-accuracy degrees of gy_{Ky-1}, gy_{Ky}
    int r1lo, r1hi;            // r1 terms [r1lo, r1hi) of this launch; R slice r1 - r1lo
};

__device__ __forceinline__ void c2_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void c2_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__global__ void __launch_bounds__(512, 1)
    k2d_cols_fs(const double2* __restrict__ R, double2* __restrict__ f, Col2Params p) {
    using W = Col2Shape;
    constexpr int G = 256, CH = 2;
    constexpr int BAR_G = 1, BAR_H = 3;  // group barriers 1-2, hand-off 3-4 (by arriving group)
    constexpr int NCH = W::SLOTS / CH;   // chunks of a unit
    extern __shared__ double2 smem[];
    __shared__ unsigned tmem_base;
    const int grp = threadIdx.x >> 8;
    const int tid = threadIdx.x & (G - 1);
    double2* buf = smem + grp * kBuf2l;
    double2* rcol = smem + 2 * kBuf2l;
    double2* tw = smem + 3 * kBuf2l;
    twiddle_table_build<4096>(tw, threadIdx.x, 2 * G);
    Twiddles<4096> T;
    twiddle_init<4096>(T, tw, tid);
    if (threadIdx.x < 32) tm_alloc(&tmem_base, 512u);
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    // thread tid of both groups shares the TMEM state of its sample slots
    const unsigned tl = tm_lane_base(tmem_base) + (unsigned)(((tid >> 7) & 1) * 256);
    const int gbar = BAR_G + grp;
    auto gsync = [gbar] { c2_bar_sync(gbar, G); };
    const long long mn = p.m * p.n;
    const int nsteps = p.ky;
    const double sx = p.ux_uniform ? 1.0 : 2.0, sy = p.uy_uniform ? 1.0 : 2.0;
    int S0 = 0;  // global step index (group of step = index & 1)
    for (long long tx = blockIdx.x; tx < p.n; tx += gridDim.x) {
        const int beg = p.coloff[tx], end = p.coloff[tx + 1];
        for (int cb = beg; cb < end; cb += W::CAP) {
            const int cnt = min(W::CAP, end - cb);
            const int nch = ((cnt + G - 1) / G + CH - 1) / CH;  // occupied chunks (CTA-uniform)
            // unit setup (this group's chunks): hy, hx, gather slot of X[ty]
            for (int k = grp; k < nch; k += 2) {
                unsigned hy[2 * CH], hx[2 * CH], sl[CH];
#pragma unroll
                for (int u = 0; u < CH; ++u) {
                    const int i = tid + (CH * k + u) * G;
                    const bool ok = i < cnt;
                    const double y = (ok && !p.uy_uniform) ? half_phase(p.dys[cb + i]) : 0.0;
                    const double x = (ok && !p.ux_uniform) ? half_phase(p.dxs[cb + i]) : 0.0;
                    hy[2 * u] = lo32(y);
                    hy[2 * u + 1] = hi32(y);
                    hx[2 * u] = lo32(x);
                    hx[2 * u + 1] = hi32(x);
                    sl[u] = ok ? (unsigned)fft2l_slot_of(p.tys[cb + i]) : 0u;
                }
                tm_stn<2 * CH>(tl + W::COL_HY + 2 * CH * k, hy);
                tm_stn<2 * CH>(tl + W::COL_HX + 2 * CH * k, hx);
                tm_stn<CH>(tl + W::COL_T + CH * k, sl);
            }
            tm_wait_st();
            for (int r1 = p.r1hi - 1; r1 >= p.r1lo; --r1) {
                // block start: the R_r1 column (stride n) into shared memory; S = 0 and the
                // gy pair (gy_{Ky-1}, gy_Ky) by the series, this group's chunks
                const double2* col = R + (long long)(r1 - p.r1lo) * mn + tx;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    rcol[threadIdx.x + 512 * q] = __ldcg(col + (long long)(threadIdx.x + 512 * q) * p.n);
                for (int k = grp; k < nch; k += 2) {
                    unsigned hy[2 * CH], sv[4 * CH], gv[4 * CH];
                    tm_ldn<2 * CH>(tl + W::COL_HY + 2 * CH * k, hy);
                    tm_wait_ld();
                    double w[CH], ga[CH], gb[CH];
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const double h = mk64(hy[2 * u], hy[2 * u + 1]);
                        w[u] = h * h;
                    }
                    series_deg<CH>(ga, w, kBes + (nsteps - 1) * kSeriesTerms, p.degy_top0);
                    series_deg<CH>(gb, w, kBes + nsteps * kSeriesTerms, p.degy_top1);
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        gv[4 * u] = lo32(ga[u]);
                        gv[4 * u + 1] = hi32(ga[u]);
                        gv[4 * u + 2] = lo32(gb[u]);
                        gv[4 * u + 3] = hi32(gb[u]);
#pragma unroll
                        for (int c = 0; c < 4; ++c) sv[4 * u + c] = 0u;
                    }
                    tm_stn<4 * CH>(tl + W::COL_S + 4 * CH * k, sv);
                    tm_stn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
                }
                tm_wait_st();
                tm_fence_before();
                __syncthreads();  // column staged, block state set
                tm_fence_after();
                for (int i = (grp - S0) & 1; i < nsteps; i += 2) {
                    const int r2 = nsteps - 1 - i;
                    const double* vy = p.vyt + (long long)r2 * p.m;
                    double2 v[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = cscale(rcol[tid + q * G], __ldg(vy + tid + q * G));
                    gsync();  // this group's gathers from buf (its previous step) are done
                    block_fft_2l<-1, false, NB_2DC_TW2>(v, buf, tid, T, gsync);
#pragma unroll
                    for (int q = 0; q < 16; ++q) buf[fft2l_slot(tid, q)] = v[q];
                    gsync();  // X complete
                    if (i > 0) {  // the other group's update of step i-1 is done
                        c2_bar_sync(BAR_H + (grp ^ 1), 2 * G);
                        tm_fence_after();
                    }
                    const double rd = (double)r2;
#pragma unroll 1
                    for (int k = 0; k < nch; ++k) {
                        unsigned sv[4 * CH], gv[4 * CH], hv[2 * CH], t2v[CH];
                        tm_ldn<4 * CH>(tl + W::COL_S + 4 * CH * k, sv);
                        tm_ldn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
                        tm_ldn<2 * CH>(tl + W::COL_HY + 2 * CH * k, hv);
                        tm_ldn<CH>(tl + W::COL_T + CH * k, t2v);
                        tm_wait_ld();
#pragma unroll
                        for (int u = 0; u < CH; ++u) {
                            const double2 X = buf[t2v[u]];
                            const double h = mk64(hv[2 * u], hv[2 * u + 1]);
                            const double gr = mk64(gv[4 * u], gv[4 * u + 1]);
                            const double gr1 = mk64(gv[4 * u + 2], gv[4 * u + 3]);
                            const double ax = mk64(sv[4 * u], sv[4 * u + 1]);
                            const double ay = mk64(sv[4 * u + 2], sv[4 * u + 3]);
                            const double nx = __fma_rn(gr, X.x, -h * ay);
                            const double ny = __fma_rn(gr, X.y, h * ax);
                            const double gm1 = __fma_rn(rd, gr, -(h * h) * gr1);  // gy_{r2-1}
                            gv[4 * u] = lo32(gm1);
                            gv[4 * u + 1] = hi32(gm1);
                            gv[4 * u + 2] = lo32(gr);
                            gv[4 * u + 3] = hi32(gr);
                            sv[4 * u] = lo32(nx);
                            sv[4 * u + 1] = hi32(nx);
                            sv[4 * u + 2] = lo32(ny);
                            sv[4 * u + 3] = hi32(ny);
                        }
                        tm_stn<4 * CH>(tl + W::COL_S + 4 * CH * k, sv);
                        tm_stn<4 * CH>(tl + W::COL_G + 4 * CH * k, gv);
                    }
                    tm_wait_st();
                    tm_fence_before();
                    if (i < nsteps - 1) c2_bar_arrive(BAR_H + grp, 2 * G);  // hand off step i+1
                }
                tm_fence_before();
                __syncthreads();  // every update of the block done; rcol free
                tm_fence_after();
                // block end (this group's chunks): A <- A (i hx) + gx_r1(hx^2) S; r1 = 0 writes f
                const double* ax_c = kBes + r1 * kSeriesTerms;
                const int dgx = p.degx[r1];
                for (int k = grp; k < nch; k += 2) {
                    unsigned sv[4 * CH], hx[2 * CH], hy[2 * CH];
                    tm_ldn<4 * CH>(tl + W::COL_S + 4 * CH * k, sv);
                    tm_ldn<2 * CH>(tl + W::COL_HX + 2 * CH * k, hx);
                    if (r1 == p.r1lo) tm_ldn<2 * CH>(tl + W::COL_HY + 2 * CH * k, hy);
                    tm_wait_ld();
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const int i = tid + (CH * k + u) * G;
                        if (i >= cnt) continue;
                        const double h = mk64(hx[2 * u], hx[2 * u + 1]);
                        const double gx = p.ux_uniform ? 1.0 : bessel_g_rt(r1, dgx, h * h);
                        const double2 S = make_double2(mk64(sv[4 * u], sv[4 * u + 1]), mk64(sv[4 * u + 2], sv[4 * u + 3]));
                        double2 A = cscale(S, gx);
                        if (r1 != p.r1hi - 1) {
                            const double2 prev = p.A[cb + i];
                            A.x = __fma_rn(-h, prev.y, A.x);
                            A.y = __fma_rn(h, prev.x, A.y);
                        }
                        if (r1 > p.r1lo) {
                            p.A[cb + i] = A;
                        } else {
                            A = ipow_scale(A, h, p.r1lo);
                            const double hyv = mk64(hy[2 * u], hy[2 * u + 1]);
                            double sn, cs;
                            sincos(2.0 * (h + hyv), &sn, &cs);
                            const double sc = sx * sy;
                            __stcs(f + p.perm[cb + i], cmul(make_double2(sc * cs, sc * sn), A));
                        }
                    }
                }
                S0 += nsteps;
            }
            tm_fence_before();
            __syncthreads();  // unit done: slots and rcol free for the next unit
            tm_fence_after();
        }
    }
    tm_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tm_dealloc(tmem_base, 512u);
}

// sort key (tx, ty): samples of a column in ascending ty, so the X[ty] gathers of a
// warp (consecutive sorted samples) hit consecutive slots of the FFT buffer — spread
// over all banks by the fft2l swizzle — instead of random ones (about half the
// shared-memory wavefronts per gather).  The order inside a column does not change
// any result: every sample keeps its own accumulators.
__global__ void k2d_keys(const long long* __restrict__ tx, const long long* __restrict__ ty, int log_m,
                         long long count, unsigned* __restrict__ keys, int* __restrict__ idx) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= count) return;
    keys[j] = ((unsigned)tx[j] << log_m) | (unsigned)ty[j];
    idx[j] = (int)j;
}

__global__ void k2d_offsets(const unsigned* __restrict__ keys, int log_m, long long count, long long nb,
                            int* __restrict__ off) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > count) return;
    const long long cur = (i < count) ? (long long)(keys[i] >> log_m) : nb;
    const long long prev = (i > 0) ? (long long)(keys[i - 1] >> log_m) : -1;
    for (long long b = prev + 1; b <= cur; ++b) off[b] = (int)i;
}

__global__ void k2d_gather(const int* __restrict__ perm, long long count, const double* __restrict__ dx,
                           const double* __restrict__ dy, const long long* __restrict__ ty,
                           double* __restrict__ dxs, double* __restrict__ dys,
                           unsigned short* __restrict__ tys) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int j = perm[i];
    dxs[i] = dx[j];
    dys[i] = dy[j];
    tys[i] = (unsigned short)ty[j];
}

__global__ void k2d_vtable(double* __restrict__ vt, long long m, int K, int uniform) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m * K) return;
    const int r = (int)(i / m);
    const long long k = i % m;
    vt[i] = uniform ? 1.0 : v_factor_from_s(grid_s(k, m), r);
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

template <int LN>
void launch_rows(const double2* C, double2* R, const Plan2DState& st, cudaStream_t s, int r1lo, int r1hi) {
    const DeviceCtx& ctx = DeviceCtx::get(st.device);
    constexpr size_t SM = sizeof(double2) * (LN + 2 * padded_len(LN) + FftShapeX<LN>::TW_LEN);
    RowParams p{(long long)st.m, (long long)st.n, ilog2(st.n), (int)st.kx, st.ux_uniform ? 1 : 0, r1lo, r1hi};
    set_smem(k2d_rows<LN>, SM);
    const int grid = (int)std::min<long long>((long long)st.m,
                                              (long long)ctx.sms * occupancy((const void*)k2d_rows<LN>, LN / 16, SM));
    k2d_rows<LN><<<grid, LN / 16, SM, s>>>(C, R, p);
    NB_LAUNCH();
}

void launch_cols_fs(const double2* R, double2* f, double2* A, const Plan2DState& st, cudaStream_t s, int r1lo,
                    int r1hi) {
    const DeviceCtx& ctx = DeviceCtx::get(st.device);
    Col2Params p{};
    p.m = (long long)st.m;
    p.n = (long long)st.n;
    p.kx = (int)st.kx;
    p.ky = (int)st.ky;
    p.ux_uniform = st.ux_uniform ? 1 : 0;
    p.uy_uniform = st.uy_uniform ? 1 : 0;
    p.dxs = st.fz.dxs.as<double>();
    p.dys = st.fz.dys.as<double>();
    p.tys = st.fz.tys.as<unsigned short>();
    p.perm = st.fz.perm.as<int>();
    p.coloff = st.fz.coloff.as<int>();
    p.vyt = st.fz.vyt.as<double>();
    p.A = A;
    p.r1lo = r1lo;
    p.r1hi = r1hi;
    for (size_t r = 0; r < st.deg_x.size() && r < (size_t)kRankCap; ++r) p.degx[r] = st.deg_x[r];
    p.degy_top0 = bessel_series_degree_rel(st.uy_uniform ? 0.0 : st.ay.gamma, (int)st.ky - 1);
    p.degy_top1 = bessel_series_degree_rel(st.uy_uniform ? 0.0 : st.ay.gamma, (int)st.ky);
    set_smem(k2d_cols_fs, Col2Shape::SMEM);
    const int grid = (int)std::min<long long>((long long)st.n, (long long)ctx.sms);
    k2d_cols_fs<<<grid, 512, Col2Shape::SMEM, s>>>(R, f, p);
    NB_LAUNCH();
}

template <int LM>
void launch_cols(const double2* R, double2* f, double2* A, const Plan2DState& st, cudaStream_t s, int r1lo,
                 int r1hi) {
    if constexpr (LM == 4096) return launch_cols_fs(R, f, A, st, s, r1lo, r1hi);
    const DeviceCtx& ctx = DeviceCtx::get(st.device);
    constexpr size_t SM = ColShape<LM>::SMEM;
    ColParams p{};
    p.m = (long long)st.m;
    p.n = (long long)st.n;
    p.log_n = ilog2(st.n);
    p.kx = (int)st.kx;
    p.ky = (int)st.ky;
    p.ux_uniform = st.ux_uniform ? 1 : 0;
    p.uy_uniform = st.uy_uniform ? 1 : 0;
    p.dxs = st.fz.dxs.as<double>();
    p.dys = st.fz.dys.as<double>();
    p.tys = st.fz.tys.as<unsigned short>();
    p.perm = st.fz.perm.as<int>();
    p.coloff = st.fz.coloff.as<int>();
    p.vyt = st.fz.vyt.as<double>();
    p.A = A;
    p.r1lo = r1lo;
    p.r1hi = r1hi;
    for (size_t r = 0; r < st.deg_x.size() && r < (size_t)kRankCap; ++r) p.degx[r] = st.deg_x[r];
    for (size_t r = 0; r < st.deg_y.size() && r < (size_t)kRankCap; ++r) p.degy[r] = st.deg_y[r];
    set_smem(k2d_cols<LM>, SM);
    const int grid = (int)std::min<long long>((long long)st.n,
                                              (long long)ctx.sms * occupancy((const void*)k2d_cols<LM>, LM / 16, SM));
    k2d_cols<LM><<<grid, LM / 16, SM, s>>>(R, f, p);
    NB_LAUNCH();
}

#define NB_SIZE_SWITCH(L, CALL)                 \
    switch (L) {                                \
        case 16: { constexpr int LL = 16; CALL; break; }     \
        case 32: { constexpr int LL = 32; CALL; break; }     \
        case 64: { constexpr int LL = 64; CALL; break; }     \
        case 128: { constexpr int LL = 128; CALL; break; }   \
        case 256: { constexpr int LL = 256; CALL; break; }   \
        case 512: { constexpr int LL = 512; CALL; break; }   \
        case 1024: { constexpr int LL = 1024; CALL; break; } \
        case 2048: { constexpr int LL = 2048; CALL; break; } \
        case 4096: { constexpr int LL = 4096; CALL; break; } \
        default: throw Error(kInternal, "2D fused size");    \
    }

}  // namespace

bool fused_2d_eligible(size_t m, size_t n, size_t count) {
    if (!is_pow2(m) || !is_pow2(n) || m < 16 || n < 16 || m > 4096 || n > 4096) return false;
    // the column kernel re-runs all terms per chunk of kQ2d*m/16 samples of a
    // column: take it only while the average column fits about one chunk
    const double per_col = (double)count / (double)n;
    return per_col <= 1.1 * (double)(kQ2d * (m / 16)) && count < (size_t(1) << 31);
}

void build_2d_fused(Plan2DState& st, cudaStream_t s) {
    const size_t count = st.count, n = st.n, m = st.m;
    DevBuf keys(4 * count, s), keys_out(4 * count, s), idx(4 * count, s);
    st.fz.perm.alloc(4 * count);
    const int log_m = ilog2(m);
    k2d_keys<<<blocks(count), 256, 0, s>>>(st.ax.t.as<long long>(), st.ay.t.as<long long>(), log_m,
                                          (long long)count, keys.as<unsigned>(), idx.as<int>());
    NB_LAUNCH();
    const int bits = std::max(1, ilog2(n) + log_m);
    size_t temp = 0;
    NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.as<unsigned>(), keys_out.as<unsigned>(),
                                            idx.as<int>(), st.fz.perm.as<int>(), (int)count, 0, bits, s));
    DevBuf tb(temp, s);
    NB_CUDA(cub::DeviceRadixSort::SortPairs(tb.get(), temp, keys.as<unsigned>(), keys_out.as<unsigned>(),
                                            idx.as<int>(), st.fz.perm.as<int>(), (int)count, 0, bits, s));
    st.fz.coloff.alloc(4 * (n + 1));
    k2d_offsets<<<blocks(count + 1), 256, 0, s>>>(keys_out.as<unsigned>(), log_m, (long long)count, (long long)n,
                                                 st.fz.coloff.as<int>());
    NB_LAUNCH();
    st.fz.dxs.alloc(8 * count);
    st.fz.dys.alloc(8 * count);
    st.fz.tys.alloc(2 * count);
    k2d_gather<<<blocks(count), 256, 0, s>>>(st.fz.perm.as<int>(), (long long)count, st.ax.delta.as<double>(),
                                            st.ay.delta.as<double>(), st.ay.t.as<long long>(),
                                            st.fz.dxs.as<double>(), st.fz.dys.as<double>(),
                                            st.fz.tys.as<unsigned short>());
    NB_LAUNCH();
    st.fz.vyt.alloc(8 * m * st.ky);
    k2d_vtable<<<blocks(m * st.ky), 256, 0, s>>>(st.fz.vyt.as<double>(), (long long)m, (int)st.ky,
                                                st.uy_uniform ? 1 : 0);
    NB_LAUNCH();
    st.fused = true;
}

void exec_2d_fused(const Plan2DState& st, const double2* C, double2* f, size_t batch, cudaStream_t s, size_t r1_begin,
                   size_t r1_end) {
    ensure_bessel_constants(st.device);
    const size_t mn = st.m * st.n;
    const int r1lo = (int)r1_begin, r1hi = (int)std::min(r1_end, st.kx);
    if (r1hi <= r1lo) {
        NB_CUDA(cudaMemsetAsync(f, 0, sizeof(double2) * st.count * batch, s));
        return;
    }
    DevBuf R(sizeof(double2) * mn * (size_t)(r1hi - r1lo), s);
    DevBuf A(sizeof(double2) * std::max<size_t>(st.count, 1), s);
    const int LN = (int)st.n, LM = (int)st.m;
    for (size_t b = 0; b < batch; ++b) {
        NB_SIZE_SWITCH(LN, launch_rows<LL>(C + b * mn, R.as<double2>(), st, s, r1lo, r1hi));
        NB_SIZE_SWITCH(LM, launch_cols<LL>(R.as<double2>(), f + b * st.count, A.as<double2>(), st, s, r1lo, r1hi));
    }
}

}  // namespace nb
