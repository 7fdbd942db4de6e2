// In-register radix butterflies and the shared-memory Stockham block FFT.
//
// This is the uniform-FFT building block that replaces the reference's FFTW
// calls (proj/include/nufft/fft.hpp:97-109).  Convention (fft.hpp:2-5):
//   forward  (SIGN = -1): X_k = sum_j x_j exp(-2*pi*i*j*k/L), unnormalized
//   backward (SIGN = +1): X_k = sum_j x_j exp(+2*pi*i*j*k/L), unnormalized
//
// A group of G = L/16 threads computes one L-point transform (L = 16..4096,
// power of two).  Thread `tid` holds v[q] = x[tid + q*G] (q < 16) on entry and
// v[q] = X[tid + q*G] on exit — coalesced with unit stride across the group
// on both sides, so prologues (loads + diagonal scaling) and epilogues fuse
// directly onto the register arrays.  Stages are Stockham autosort with
// radix 16 (and one final radix 8/4/2 stage when log2 L is not a multiple of
// 4); between stages the data crosses shared memory once (write + read) in
// a ping-pong pair of padded buffers, one barrier per exchange.
#pragma once

#include "common.cuh"

namespace nb {

// exp(SIGN*2*pi*i*Q/16) multiply, special-casing the quarter turns
template <int Q, int SIGN>
__device__ __forceinline__ double2 mul_w16(double2 a) {
    constexpr int q = ((Q % 16) + 16) % 16;
    if constexpr (q == 0) {
        return a;
    } else if constexpr (q == 8) {
        return make_double2(-a.x, -a.y);
    } else if constexpr (q == 4 || q == 12) {
        // multiply by SIGN*i (q==4) or -SIGN*i (q==12)
        constexpr int s = (q == 4) ? SIGN : -SIGN;
        return s > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
    } else {
        constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173,
                         C2 = 0.70710678118654752440;
        // cos/sin of 2*pi*q/16
        constexpr double ctab[16] = {1, C1, C2, S1, 0, -S1, -C2, -C1, -1, -C1, -C2, -S1, 0, S1, C2, C1};
        constexpr double stab[16] = {0, S1, C2, C1, 1, C1, C2, S1, 0, -S1, -C2, -C1, -1, -C1, -C2, -S1};
        constexpr double c = ctab[q], s = SIGN * stab[q];
        return make_double2(__fma_rn(a.x, c, -a.y * s), __fma_rn(a.x, s, a.y * c));
    }
}

template <int SIGN>
__device__ __forceinline__ void dft2(double2& a0, double2& a1) {
    const double2 t = a0;
    a0 = cadd(t, a1);
    a1 = csub(t, a1);
}

template <int SIGN>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const double2 s13 = cadd(a1, a3), d13 = csub(a1, a3);
    const double2 w = mul_w16<4, SIGN>(d13);
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = cadd(d02, w);
    a3 = csub(d02, w);
}

// In-place R-point DFT of a[0..R-1] (natural order in and out), R in {2,4,8,16}.
template <int R, int SIGN>
__device__ __forceinline__ void dft(double2* a) {
    if constexpr (R == 1) {
    } else if constexpr (R == 2) {
        dft2<SIGN>(a[0], a[1]);
    } else if constexpr (R == 4) {
        dft4<SIGN>(a[0], a[1], a[2], a[3]);
    } else if constexpr (R == 8) {
        // t = t1 + 2*t2, k = k2 + 4*k1
        dft4<SIGN>(a[0], a[2], a[4], a[6]);
        dft4<SIGN>(a[1], a[3], a[5], a[7]);
        a[3] = mul_w16<2, SIGN>(a[3]);
        a[5] = mul_w16<4, SIGN>(a[5]);
        a[7] = mul_w16<6, SIGN>(a[7]);
        double2 o[8];
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
            double2 x0 = a[2 * k2], x1 = a[2 * k2 + 1];
            dft2<SIGN>(x0, x1);
            o[k2] = x0;
            o[k2 + 4] = x1;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = o[i];
    } else {
        static_assert(R == 16, "radix");
        // t = t1 + 4*t2 ; inner DFT4 over t2 for each t1 -> b[t1][k2] stored at a[t1 + 4*k2]
        dft4<SIGN>(a[0], a[4], a[8], a[12]);
        dft4<SIGN>(a[1], a[5], a[9], a[13]);
        dft4<SIGN>(a[2], a[6], a[10], a[14]);
        dft4<SIGN>(a[3], a[7], a[11], a[15]);
        // twiddle w16^(t1*k2)
        a[5] = mul_w16<1, SIGN>(a[5]);
        a[9] = mul_w16<2, SIGN>(a[9]);
        a[13] = mul_w16<3, SIGN>(a[13]);
        a[6] = mul_w16<2, SIGN>(a[6]);
        a[10] = mul_w16<4, SIGN>(a[10]);
        a[14] = mul_w16<6, SIGN>(a[14]);
        a[7] = mul_w16<3, SIGN>(a[7]);
        a[11] = mul_w16<6, SIGN>(a[11]);
        a[15] = mul_w16<9, SIGN>(a[15]);
        // outer DFT4 over t1 for each k2 -> out[k2 + 4*k1]
        dft4<SIGN>(a[0], a[1], a[2], a[3]);
        dft4<SIGN>(a[4], a[5], a[6], a[7]);
        dft4<SIGN>(a[8], a[9], a[10], a[11]);
        dft4<SIGN>(a[12], a[13], a[14], a[15]);
        // now a[4*k2 + k1] holds out[k2 + 4*k1]: transpose 4x4
        double2 o[16];
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2)
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) o[k2 + 4 * k1] = a[4 * k2 + k1];
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = o[i];
    }
}

// padded shared-memory index: one 16-byte pad per 16 elements (bank spread)
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int L) { return L + L / 16; }

// number of radix-16 stages and the remainder radix of an L-point FFT
template <int L>
struct FftShape {
    static constexpr int LOG = ilog2_c(L);
    static constexpr int N16 = LOG / 4;
    static constexpr int REM = 1 << (LOG % 4);
    static constexpr int STAGES = N16 + (REM > 1 ? 1 : 0);
    static constexpr int G = L / 16;  // threads per transform
    static_assert(L >= 16 && L <= 4096 && (1 << LOG) == L, "block FFT size");
};

// ---------------------------------------------------------------- twiddles
// Stage twiddles without table gathers (a scattered 16-byte L1 gather per
// twiddle cost more than the whole DFT arithmetic in microbenchmarks):
//  * the Ns = 16 stage uses w_{16 R2}^{k t}, k = j mod 16: a 16 x R2 table in
//    shared memory laid out [t][k] (one warp load touches 16 consecutive
//    entries: 2 wavefronts, no conflicts);
//  * the Ns = 256 stage (L >= 512) uses w_L^{k t} with k = j < 256: bases
//    w^k, w^{2k}, w^{4k}, w^{8k} live in a [4][256] shared table (evaluated
//    once per CTA with sincospi, correctly rounded argument; each thread reads
//    its own column, conflict-free) and the other powers are products of at
//    most three of them (<= ~3 ulp).
template <int L>
struct FftShapeX : FftShape<L> {
    static constexpr int R_LAST = (FftShape<L>::REM > 1) ? FftShape<L>::REM : 16;
    static constexpr int R2 = (FftShape<L>::STAGES == 2) ? R_LAST : 16;  // radix of the Ns=16 stage
    static constexpr int R3 = (FftShape<L>::STAGES == 3) ? R_LAST : 1;   // radix of the Ns=256 stage
    static constexpr int B3 = 16 / R3;                                    // its butterflies per thread
    static constexpr int T16_LEN = (FftShape<L>::STAGES >= 2) ? 16 * R2 : 16;
    // stage-3 bases w^(k 2^e), one 256-row per e < log2(R3): apply_pow_twiddles<R3> reads
    // rows 0 .. log2(R3)-1 only (4 rows at L = 4096, 3 at 2048: 4 KiB less shared memory
    // lets two k1_passA<2048> CTAs share an SM)
    static constexpr int TB_LEN = (FftShape<L>::STAGES == 3) ? ilog2_c(R3) * 256 : 0;
    static constexpr int TW_LEN = T16_LEN + TB_LEN;  // shared twiddle storage (double2)
};

template <int L>
struct Twiddles {
    // shared: t16[t*16 + k] = w_{16 R2}^{k t};  tb[e*256 + k] = w_L^{(k 2^e) mod L}, k < 256
    const double2* t16;
    const double2* tb;
};

// fill the shared twiddle storage tw (TW_LEN entries; all threads of the
// CTA, barrier before use)
template <int L>
__device__ __forceinline__ void twiddle_table_build(double2* tw, int tid, int nthreads) {
    using X = FftShapeX<L>;
    for (int i = tid; i < X::T16_LEN; i += nthreads) {
        const int t = i >> 4, k = i & 15;
        tw[i] = unit_root((long long)k * t, 16 * X::R2);
    }
    for (int i = tid; i < X::TB_LEN; i += nthreads) {
        const long long e = i >> 8, k = i & 255;
        tw[X::T16_LEN + i] = unit_root((k << e) % L, L);
    }
}

template <int L>
__device__ __forceinline__ void twiddle_init(Twiddles<L>& T, const double2* tw, int tid) {
    (void)tid;
    T.t16 = tw;
    T.tb = tw + FftShapeX<L>::T16_LEN;
}

template <int SIGN>
__device__ __forceinline__ double2 tw_sign(double2 w) {
    return SIGN < 0 ? w : make_double2(w.x, -w.y);
}

// a[t] *= w^t (t = 1..R-1) for the Ns = 256 stage, powers from the bases
// bs[e*256] = w^(k 2^e) (shared, per-thread column k)
template <int R, int SIGN>
__device__ __forceinline__ void apply_pow_twiddles(double2* a, const double2* bs) {
    const double2 p1 = tw_sign<SIGN>(bs[0]);
    if constexpr (R == 2) {
        a[1] = cmul(a[1], p1);
    } else {
        const double2 p2 = tw_sign<SIGN>(bs[256]);
        const double2 p3 = cmul(p1, p2);
        a[1] = cmul(a[1], p1);
        a[2] = cmul(a[2], p2);
        a[3] = cmul(a[3], p3);
        if constexpr (R >= 8) {
            const double2 p4 = tw_sign<SIGN>(bs[512]);
            const double2 p5 = cmul(p1, p4), p6 = cmul(p2, p4), p7 = cmul(p3, p4);
            a[4] = cmul(a[4], p4);
            a[5] = cmul(a[5], p5);
            a[6] = cmul(a[6], p6);
            a[7] = cmul(a[7], p7);
            if constexpr (R == 16) {
                const double2 p8 = tw_sign<SIGN>(bs[768]);
                a[8] = cmul(a[8], p8);
                a[9] = cmul(a[9], cmul(p1, p8));
                a[10] = cmul(a[10], cmul(p2, p8));
                a[11] = cmul(a[11], cmul(p3, p8));
                a[12] = cmul(a[12], cmul(p4, p8));
                a[13] = cmul(a[13], cmul(p5, p8));
                a[14] = cmul(a[14], cmul(p6, p8));
                a[15] = cmul(a[15], cmul(p7, p8));
            }
        }
    }
}

// One Stockham stage: radix R, Ns = product of the radices already applied.
// Reads v (layout x[tid + q*G]); if !LAST writes the stage output to `out`
// (padded, natural Stockham order); if LAST leaves it in v (same layout).
template <int L, int R, int NS, bool LAST, int SIGN>
__device__ __forceinline__ void stockham_stage(double2 (&v)[16], double2* out, int tid,
                                               const Twiddles<L>& T) {
    constexpr int G = L / 16;
    constexpr int B = 16 / R;  // butterflies per thread
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const int j = tid + b * G;
        const int k = j & (NS - 1);
        double2 a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = v[b + t * B];
        if constexpr (NS == 16) {
#pragma unroll
            for (int t = 1; t < R; ++t) a[t] = cmul(a[t], tw_sign<SIGN>(T.t16[t * 16 + k]));
        } else if constexpr (NS == 256) {
            apply_pow_twiddles<R, SIGN>(a, T.tb + k);
        } else {
            static_assert(NS == 1, "stage");
        }
        dft<R, SIGN>(a);
        if constexpr (LAST) {
#pragma unroll
            for (int t = 0; t < R; ++t) v[b + t * B] = a[t];
        } else {
            const int base = (j - k) * R + k;  // (j/Ns)*Ns*R + k
#pragma unroll
            for (int t = 0; t < R; ++t) out[pad16(base + t * NS)] = a[t];
        }
    }
}

template <int L>
__device__ __forceinline__ void load_stage_input(double2 (&v)[16], const double2* in, int tid) {
    constexpr int G = L / 16;
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = in[pad16(tid + q * G)];
}

// Full L-point FFT on the register array v (layout above).  buf0/buf1: two
// padded shared buffers of padded_len(L) double2 owned by this group; `bar`
// is the group barrier.  On exit the last-written buffer is
// buf[(STAGES-2)&1]; the other one is free.
template <int L, int SIGN, class Bar>
__device__ __forceinline__ void block_fft(double2 (&v)[16], double2* buf0, double2* buf1, int tid,
                                          const Twiddles<L>& T, Bar bar) {
    using S = FftShapeX<L>;
    if constexpr (S::STAGES == 1) {
        stockham_stage<L, 16, 1, true, SIGN>(v, nullptr, tid, T);
    } else if constexpr (S::STAGES == 2) {
        stockham_stage<L, 16, 1, false, SIGN>(v, buf0, tid, T);
        bar();
        load_stage_input<L>(v, buf0, tid);
        stockham_stage<L, S::R_LAST, 16, true, SIGN>(v, nullptr, tid, T);
    } else {
        static_assert(S::STAGES == 3, "L <= 4096");
        stockham_stage<L, 16, 1, false, SIGN>(v, buf0, tid, T);
        bar();
        load_stage_input<L>(v, buf0, tid);
        stockham_stage<L, 16, 16, false, SIGN>(v, buf1, tid, T);
        bar();
        load_stage_input<L>(v, buf1, tid);
        stockham_stage<L, S::R_LAST, 256, true, SIGN>(v, nullptr, tid, T);
    }
}

// Single-buffer variant (half the shared memory of block_fft): each exchange
// is write -> barrier -> read -> barrier.  The caller guarantees `buf` is free
// on entry; on exit other threads may still be reading it for the final stage,
// so the caller must barrier before writing `buf` again.
template <int L, int SIGN, class Bar>
__device__ __forceinline__ void block_fft_1buf(double2 (&v)[16], double2* buf, int tid,
                                               const Twiddles<L>& T, Bar bar) {
    using S = FftShapeX<L>;
    if constexpr (S::STAGES == 1) {
        stockham_stage<L, 16, 1, true, SIGN>(v, nullptr, tid, T);
    } else if constexpr (S::STAGES == 2) {
        stockham_stage<L, 16, 1, false, SIGN>(v, buf, tid, T);
        bar();
        load_stage_input<L>(v, buf, tid);
        stockham_stage<L, S::R_LAST, 16, true, SIGN>(v, nullptr, tid, T);
    } else {
        static_assert(S::STAGES == 3, "L <= 4096");
        stockham_stage<L, 16, 1, false, SIGN>(v, buf, tid, T);
        bar();
        load_stage_input<L>(v, buf, tid);
        bar();
        stockham_stage<L, 16, 16, false, SIGN>(v, buf, tid, T);
        bar();
        load_stage_input<L>(v, buf, tid);
        stockham_stage<L, S::R_LAST, 256, true, SIGN>(v, nullptr, tid, T);
    }
}

// ------------------------------------------------------------ two-level 4096
// 4096 = 16 x 256 with one group-wide exchange.  j = j0 + 256 j1, k = k1 + 16 k0:
//   A[j0, k1] = w_4096^{j0 k1} sum_j1 x[j0 + 256 j1] w_16^{j1 k1}   (thread j0, registers)
//   X[k1 + 16 k0] = sum_j0 A[j0, k1] w_256^{j0 k0}                  (16 independent 256-pt DFTs)
// The transpose A -> (k1-major) is the only exchange every thread of the group
// takes part in (write, barrier, read).  Each 256-point DFT then belongs to a
// sub-group of 16 threads of one warp (g = k1): radix 16 over j0 = u + 16 m,
// twiddle w_256^{u a}, and a 16 x 16 transpose inside the sub-group's own
// 256-element region of the same buffer that needs only __syncwarp.  Two
// group barriers per transform instead of four for block_fft_1buf; same FP64
// work; no padding (4096 slots).
//
// Sub-groups interleave in the warp (lane = 2u + (g & 1)), so lanes 2i, 2i+1
// hold outputs t and t + 1 — both halves of a 32-byte sector sit in one
// quarter-warp of a 16-byte store.  Slots are XOR-swizzled inside aligned
// 8-slot blocks (16-byte slots, 8 per 128-byte bank row): region g uses
// swz(g) = 4 (g & 1) | ((g >> 1) & 3), so the two sub-groups of a quarter-warp
// always touch complementary bank halves (every exchange access conflict-free),
// and the exchange-2 slots are further XORed with (a & 7) so a column read
// of the 16 x 16 tile is conflict-free.  X[t] of the thread's outputs ends in
// the slots it read last (fft2l_slot); since swz(g) is a bijection on every 8
// consecutive g, gathers of consecutive t (sorted samples) spread over all banks.
//
// In:  v[q] = x[tid + 256 q].   Out: v[b] = X[g + 16 u + 256 b] (fft2l_out_index).
// The thread may overwrite exactly its 16 slots fft2l_slot(tid, b) (e.g. with
// X) without a barrier; anything else needs a group barrier first.
constexpr int kBuf2l = 4096;  // buffer slots (double2)

__device__ __forceinline__ int fft2l_g(int tid) { return ((tid >> 5) << 1) | (tid & 1); }
__device__ __forceinline__ int fft2l_u(int tid) { return (tid >> 1) & 15; }
__host__ __device__ __forceinline__ int fft2l_swz(int g) { return ((g & 1) << 2) | ((g >> 1) & 3); }
__device__ __forceinline__ int fft2l_out_index(int tid, int b) { return fft2l_g(tid) + 16 * fft2l_u(tid) + 256 * b; }
// slot of X[t] after block_fft_2l when every owner writes its outputs in place
__host__ __device__ __forceinline__ int fft2l_slot_of(int t) {
    const int g = t & 15, a = (t >> 4) & 15, b = t >> 8;
    return g * 256 + 16 * a + (b ^ fft2l_swz(g) ^ (a & 7));
}
__device__ __forceinline__ int fft2l_slot(int tid, int b) {
    const int g = fft2l_g(tid), u = fft2l_u(tid);
    return g * 256 + 16 * u + (b ^ fft2l_swz(g) ^ (u & 7));
}

// a[t] *= p1^t (t = 1..15) given p1, p2 = p1^2, p4, p8 in registers
__device__ __forceinline__ void apply_pow_twiddles_regs(double2* a, double2 p1, double2 p2, double2 p4, double2 p8) {
    const double2 p3 = cmul(p1, p2);
    a[1] = cmul(a[1], p1);
    a[2] = cmul(a[2], p2);
    a[3] = cmul(a[3], p3);
    const double2 p5 = cmul(p1, p4), p6 = cmul(p2, p4), p7 = cmul(p3, p4);
    a[4] = cmul(a[4], p4);
    a[5] = cmul(a[5], p5);
    a[6] = cmul(a[6], p6);
    a[7] = cmul(a[7], p7);
    a[8] = cmul(a[8], p8);
    a[9] = cmul(a[9], cmul(p1, p8));
    a[10] = cmul(a[10], cmul(p2, p8));
    a[11] = cmul(a[11], cmul(p3, p8));
    a[12] = cmul(a[12], cmul(p4, p8));
    a[13] = cmul(a[13], cmul(p5, p8));
    a[14] = cmul(a[14], cmul(p6, p8));
    a[15] = cmul(a[15], cmul(p7, p8));
}

// the same products with at most five factors live at a time (p1, p2, p4, p8 and one of p3, p5,
// p6, p7), for kernels at the register limit
__device__ __forceinline__ void apply_pow_twiddles_lowreg(double2* a, double2 p1, double2 p2, double2 p4, double2 p8) {
    a[8] = cmul(a[8], p8);
    a[1] = cmul(a[1], p1);
    a[9] = cmul(a[9], cmul(p1, p8));
    a[2] = cmul(a[2], p2);
    a[10] = cmul(a[10], cmul(p2, p8));
    a[4] = cmul(a[4], p4);
    a[12] = cmul(a[12], cmul(p4, p8));
    {
        const double2 p5 = cmul(p1, p4);
        a[5] = cmul(a[5], p5);
        a[13] = cmul(a[13], cmul(p5, p8));
    }
    {
        const double2 p6 = cmul(p2, p4);
        a[6] = cmul(a[6], p6);
        a[14] = cmul(a[14], cmul(p6, p8));
    }
    const double2 p3 = cmul(p1, p2);
    a[3] = cmul(a[3], p3);
    a[11] = cmul(a[11], cmul(p3, p8));
    const double2 p7 = cmul(p3, p4);
    a[7] = cmul(a[7], p7);
    a[15] = cmul(a[15], cmul(p7, p8));
}

// PreWrite: called once, after the first-level DFT and twiddles and before the
// first write to buf — the point by which buf must be free (callers whose
// buf is still being read by the TMA engine wait there, not before the FFT).
struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};
// a[t] *= pre * w^t (t = 0..15): apply_pow_twiddles<16> with a thread-constant
// factor pre folded into the generated powers (pre * w^t = (pre * w^(t - 2^e)) * w^(2^e)):
// 15 products to form the factors instead of 11, 16 applications instead of 15 —
// cheaper than scaling the 16 inputs of the DFT by pre separately.
template <int SIGN>
__device__ __forceinline__ void apply_pow_twiddles_pre(double2* a, const double2* bs, double2 pre) {
    const double2 p1 = tw_sign<SIGN>(bs[0]), p2 = tw_sign<SIGN>(bs[256]);
    const double2 p4 = tw_sign<SIGN>(bs[512]), p8 = tw_sign<SIGN>(bs[768]);
    const double2 q1 = cmul(pre, p1), q2 = cmul(pre, p2), q3 = cmul(q1, p2);
    const double2 q4 = cmul(pre, p4), q5 = cmul(q1, p4), q6 = cmul(q2, p4), q7 = cmul(q3, p4);
    a[0] = cmul(a[0], pre);
    a[1] = cmul(a[1], q1);
    a[2] = cmul(a[2], q2);
    a[3] = cmul(a[3], q3);
    a[4] = cmul(a[4], q4);
    a[5] = cmul(a[5], q5);
    a[6] = cmul(a[6], q6);
    a[7] = cmul(a[7], q7);
    a[8] = cmul(a[8], cmul(pre, p8));
    a[9] = cmul(a[9], cmul(q1, p8));
    a[10] = cmul(a[10], cmul(q2, p8));
    a[11] = cmul(a[11], cmul(q3, p8));
    a[12] = cmul(a[12], cmul(q4, p8));
    a[13] = cmul(a[13], cmul(q5, p8));
    a[14] = cmul(a[14], cmul(q6, p8));
    a[15] = cmul(a[15], cmul(q7, p8));
}

// PRE: the 16 inputs of the thread carry a common factor `pre` that is applied
// with the first-level twiddles instead (the first-level DFT is linear).
// TW2: how the second-level twiddles w^{u a} reach the registers —
//   0: 15 loads from the [a][u] table t16 after the second DFT;
//   1: the four bases (rows a = 1, 2, 4, 8 of t16) loaded after the exchange reads, powers generated
//      (11 more complex products per thread);
//   2: the same bases loaded ahead of the exchange (16 registers carried across it).
// Table loads issued between the second DFT and the transpose queue behind the other worker's
// exchange traffic in the shared-memory pipe: 3997 (0) / 3800 (1) / 3650 (2) cycles per FFT per SM
// with two free-running workers (scripts/microbench_fft9.cu).  Kernels with no registers to spare
// keep mode 0 or 1.
template <int SIGN, bool PRE = false, int TW2 = 2, class Bar, class PreWrite = NoHook>
__device__ __forceinline__ void block_fft_2l(double2 (&v)[16], double2* buf, int tid, const Twiddles<4096>& T,
                                             Bar bar, PreWrite pre_write = PreWrite(),
                                             double2 pre = make_double2(1.0, 0.0)) {
    dft<16, SIGN>(v);
    if constexpr (PRE) {
        apply_pow_twiddles_pre<SIGN>(v, T.tb + tid, pre);
    } else {
        apply_pow_twiddles<16, SIGN>(v, T.tb + tid);
    }
    const int g = fft2l_g(tid), u = fft2l_u(tid), sw = fft2l_swz(g);
    double2 q1, q2, q4, q8;
    if constexpr (TW2 == 2 || TW2 == 4) {
        q1 = tw_sign<SIGN>(T.t16[16 + u]), q2 = tw_sign<SIGN>(T.t16[32 + u]);
        q4 = tw_sign<SIGN>(T.t16[64 + u]), q8 = tw_sign<SIGN>(T.t16[128 + u]);
    }
    pre_write();
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 256 + (tid ^ fft2l_swz(k1))] = v[k1];
    bar();
    double2* reg = buf + g * 256;
    const double2* rd1 = reg + (u ^ sw);
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = rd1[16 * m];
    if constexpr (TW2 == 1) {
        q1 = tw_sign<SIGN>(T.t16[16 + u]), q2 = tw_sign<SIGN>(T.t16[32 + u]);
        q4 = tw_sign<SIGN>(T.t16[64 + u]), q8 = tw_sign<SIGN>(T.t16[128 + u]);
    }
    dft<16, SIGN>(v);
    if constexpr (TW2 == 0) {
#pragma unroll
        for (int a = 1; a < 16; ++a) v[a] = cmul(v[a], tw_sign<SIGN>(T.t16[a * 16 + u]));
    } else if constexpr (TW2 == 3) {
        // the four bases loaded only now, applied in an order that keeps five factors live
        const double2 b8 = tw_sign<SIGN>(T.t16[128 + u]), b1 = tw_sign<SIGN>(T.t16[16 + u]);
        const double2 b2 = tw_sign<SIGN>(T.t16[32 + u]), b4 = tw_sign<SIGN>(T.t16[64 + u]);
        apply_pow_twiddles_lowreg(v, b1, b2, b4, b8);
    } else if constexpr (TW2 == 4) {
        apply_pow_twiddles_lowreg(v, q1, q2, q4, q8);
    } else {
        apply_pow_twiddles_regs(v, q1, q2, q4, q8);
    }
    __syncwarp();
    const int U = u ^ sw;
#pragma unroll
    for (int a = 0; a < 16; ++a) reg[16 * a + (U ^ (a & 7))] = v[a];
    __syncwarp();
    double2* rd2 = reg + 16 * u;
    const int A = sw ^ (u & 7);
#pragma unroll
    for (int w = 0; w < 16; ++w) v[w] = rd2[w ^ A];
    dft<16, SIGN>(v);
}

// the buffer that is NOT read by the final stage (safe to overwrite after
// block_fft returns, once every thread of the group has passed the last barrier)
template <int L>
__device__ __forceinline__ double2* block_fft_free_buf(double2* buf0, double2* buf1) {
    return (FftShape<L>::STAGES == 3) ? buf0 : buf1;
}

}  // namespace nb
