// Microbenchmark (design tool): production block FFT (fft_block.cuh, radix 16,
// smem twiddles) with W independent 256-thread workers per SM, each on its own
// padded single buffer (the pass-1 / pass-2 organization), vs one worker with
// ping-pong buffers.  Reports SM-throughput cycles per 4096-point FFT.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

template <int W, bool PINGPONG>
__global__ void __launch_bounds__(W * 256, 1) k_bench(double2* out, int iters) {
    constexpr int L = 4096, G = 256;
    extern __shared__ double2 sm[];
    const int grp = threadIdx.x / G, tid = threadIdx.x % G;
    double2* tw = sm + (PINGPONG ? 2 : W) * padded_len(L);
    double2* b0 = sm + grp * padded_len(L);
    double2* b1 = sm + padded_len(L);
    twiddle_table_build<L>(tw, threadIdx.x, W * G);
    Twiddles<L> T;
    twiddle_init<L>(T, tw, tid);
    __syncthreads();
    const int bar = 1 + grp;
    auto gsync = [bar] { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G) : "memory"); };
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
    for (int it = 0; it < iters; ++it) {
        if constexpr (PINGPONG) {
            block_fft<L, -1>(v, b0, b1, tid, T, gsync);
        } else {
            gsync();
            block_fft_1buf<L, -1>(v, b0, tid, T, gsync);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int W, bool PP>
void run(double2* out, int sms) {
    constexpr int L = 4096;
    const size_t smem = sizeof(double2) * ((PP ? 2 : W) * padded_len(L) + FftShapeX<L>::TW_LEN);
    cudaFuncSetAttribute(k_bench<W, PP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<W, PP><<<sms, W * 256, smem>>>(out, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k_bench<W, PP><<<sms, W * 256, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms * 1e6 / ((double)W * iters);
    printf("workers=%d %s: %.0f ns = %.0f cycles per FFT per SM %s\n", W, PP ? "ping-pong" : "1buf", per,
           per * 1.965, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    run<1, true>(out, sms);
    run<1, false>(out, sms);
    run<2, false>(out, sms);
    run<3, false>(out, sms);
    return 0;
}
