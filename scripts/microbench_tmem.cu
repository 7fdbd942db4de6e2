// Microbenchmark (design tool): TMEM as per-thread scratch — tcgen05.ld / st
// throughput per SM for the 32x32b shape (each thread moves its own lane's
// columns), with W warps per CTA, one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int NW, bool STORE>
__global__ void __launch_bounds__(NW * 32, 1) k_tmem(unsigned* out, int iters) {
    __shared__ unsigned base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        const unsigned a = (unsigned)__cvta_generic_to_shared(&base);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(512u) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned t = base + ((32u * (warp & 3u)) << 16) + (unsigned)((warp >> 2) * 32) % 512u;
    unsigned acc = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
        unsigned r[32];
        if constexpr (STORE) {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = acc + i;
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(t),
                "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            acc += 1;
        } else {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                  "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                  "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                  "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                : "r"(t)
                : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i) acc ^= r[i];
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512u) : "memory");
}

template <int NW, bool STORE>
void run(unsigned* out, int sms) {
    const int iters = 20000;
    k_tmem<NW, STORE><<<sms, NW * 32>>>(out, 10);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_tmem<NW, STORE><<<sms, NW * 32>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes_per_sm = (double)iters * NW * 32 * 32 * 4;
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("%s warps=%2d: %.1f B/cycle/SM (%.2f TB/s/SM) %s\n", STORE ? "st" : "ld", NW, bytes_per_sm / cyc,
           bytes_per_sm / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* out;
    cudaMalloc(&out, sizeof(unsigned) * sms * 1024);
    run<4, false>(out, sms);
    run<8, false>(out, sms);
    run<16, false>(out, sms);
    run<4, true>(out, sms);
    run<8, true>(out, sms);
    run<16, true>(out, sms);
    return 0;
}
