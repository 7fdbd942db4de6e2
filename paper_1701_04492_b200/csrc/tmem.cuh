// Tensor memory (TMEM) as per-thread scratch for the FP64 kernels.
//
// Each SM has 256 KB of TMEM (128 lanes x 512 columns x 32 bit) that the
// FP64 FFT path never uses for MMA.  tcgen05.st / tcgen05.ld with the
// 32x32b shape move whole 32-bit columns of the executing thread's own lane
// (warp w reaches lanes 32*(w%4) .. +31), at ~460 B/cycle/SM (ld) and
// ~340 B/cycle/SM (st) measured on B200 (scripts/microbench_tmem.cu) — more
// than three times the shared-memory crossbar — so per-thread state that
// would otherwise cost registers (Chebyshev recurrences, cached inputs,
// per-sample metadata) can live there.  Addresses: (lane << 16) | column.
#pragma once

#include "common.cuh"

namespace nb {

// warp-collective (all 32 lanes): allocate `cols` (power of two >= 32) columns,
// base address written to the shared-memory slot
__device__ __forceinline__ void tm_alloc(unsigned* slot, unsigned cols) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tm_dealloc(unsigned base, unsigned cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols) : "memory");
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// the executing warp's lane window
__device__ __forceinline__ unsigned tm_lane_base(unsigned tbase) {
    const unsigned warp = threadIdx.x >> 5;
    return tbase + ((32u * (warp & 3u)) << 16);
}

__device__ __forceinline__ void tm_st4(unsigned taddr, unsigned a, unsigned b, unsigned c, unsigned d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void tm_ld4(unsigned taddr, unsigned& a, unsigned& b, unsigned& c, unsigned& d) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tm_st8(unsigned taddr, const unsigned (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tm_ld8(unsigned taddr, unsigned (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
// 16 consecutive columns
__device__ __forceinline__ void tm_st16(unsigned taddr, const unsigned (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tm_ld16(unsigned taddr, unsigned (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tm_st2(unsigned taddr, unsigned a, unsigned b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tm_ld2(unsigned taddr, unsigned& a, unsigned& b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr) : "memory");
}
// N consecutive columns, N in {2, 4, 8, 16}
template <int N>
__device__ __forceinline__ void tm_stn(unsigned taddr, const unsigned (&v)[N]) {
    if constexpr (N == 2) {
        tm_st2(taddr, v[0], v[1]);
    } else if constexpr (N == 4) {
        tm_st4(taddr, v[0], v[1], v[2], v[3]);
    } else if constexpr (N == 8) {
        tm_st8(taddr, v);
    } else {
        static_assert(N == 16, "tm_stn");
        tm_st16(taddr, v);
    }
}
template <int N>
__device__ __forceinline__ void tm_ldn(unsigned taddr, unsigned (&v)[N]) {
    if constexpr (N == 2) {
        tm_ld2(taddr, v[0], v[1]);
    } else if constexpr (N == 4) {
        tm_ld4(taddr, v[0], v[1], v[2], v[3]);
    } else if constexpr (N == 8) {
        tm_ld8(taddr, v);
    } else {
        static_assert(N == 16, "tm_ldn");
        tm_ld16(taddr, v);
    }
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ unsigned lo32(double v) { return (unsigned)(__double_as_longlong(v) & 0xffffffffull); }
__device__ __forceinline__ unsigned hi32(double v) {
    return (unsigned)((unsigned long long)__double_as_longlong(v) >> 32);
}
__device__ __forceinline__ double mk64(unsigned lo, unsigned hi) {
    return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

}  // namespace nb
