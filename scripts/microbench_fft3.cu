// Microbenchmark (design tool): 4096-pt fp64 block FFT per SM
//   A: radix-16, 256 thr, single buffer, production twiddles (fft_block.cuh)
//   B: radix-16, 256 thr, ping-pong,     production twiddles
//   C: radix-8,  512 thr, single buffer, twiddles = register constants (upper bound)
//   D: radix-8,  512 thr, ping-pong,     twiddles = register constants
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

template <int MODE>
__global__ void __launch_bounds__((MODE >= 2) ? 512 : 256, 1) k_bench(double2* out, int iters) {
    constexpr int L = 4096;
    extern __shared__ double2 sm[];
    const int tid = threadIdx.x;
    if constexpr (MODE < 2) {
        constexpr int G = 256;
        double2* b0 = sm;
        double2* b1 = sm + padded_len(L);
        double2* tw = sm + 2 * padded_len(L);
        twiddle_table_build<L>(tw, tid, G);
        Twiddles<L> T;
        twiddle_init<L>(T, tw, tid);
        __syncthreads();
        double2 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
        for (int it = 0; it < iters; ++it) {
            if constexpr (MODE == 0) {
                __syncthreads();
                block_fft_1buf<L, -1>(v, b0, tid, T, [] { __syncthreads(); });
            } else {
                block_fft<L, -1>(v, b0, b1, tid, T, [] { __syncthreads(); });
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
        }
        double2 acc = make_double2(0, 0);
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
        out[blockIdx.x * blockDim.x + tid] = acc;
    } else {
        constexpr int G = 512;  // 8 points per thread, radix 8, stages NS = 1, 8, 64, 512
        double2* b0 = sm;
        double2* b1 = sm + padded_len(L);
        const double2 wc = make_double2(0.7 + tid * 1e-7, 0.3);
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
        auto stage = [&](auto NSc, double2* outb, bool last) {
            constexpr int NS = decltype(NSc)::value;
            const int j = tid;
            const int k = j & (NS - 1);
            double2 a[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) a[t] = v[t];
            if constexpr (NS > 1) {
#pragma unroll
                for (int t = 1; t < 8; ++t) a[t] = cmul(a[t], make_double2(wc.x + t, wc.y));
            }
            dft<8, -1>(a);
            if (last) {
#pragma unroll
                for (int t = 0; t < 8; ++t) v[t] = a[t];
            } else {
                const int base = (j - k) * 8 + k;
#pragma unroll
                for (int t = 0; t < 8; ++t) outb[pad16(base + t * NS)] = a[t];
            }
        };
        auto load = [&](const double2* in) {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = in[pad16(tid + q * G)];
        };
        for (int it = 0; it < iters; ++it) {
            if constexpr (MODE == 2) {
                __syncthreads();
                stage(std::integral_constant<int, 1>{}, b0, false);
                __syncthreads(); load(b0); __syncthreads();
                stage(std::integral_constant<int, 8>{}, b0, false);
                __syncthreads(); load(b0); __syncthreads();
                stage(std::integral_constant<int, 64>{}, b0, false);
                __syncthreads(); load(b0);
                stage(std::integral_constant<int, 512>{}, b0, true);
            } else {
                stage(std::integral_constant<int, 1>{}, b0, false);
                __syncthreads(); load(b0);
                stage(std::integral_constant<int, 8>{}, b1, false);
                __syncthreads(); load(b1);
                stage(std::integral_constant<int, 64>{}, b0, false);
                __syncthreads(); load(b0);
                stage(std::integral_constant<int, 512>{}, b0, true);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
        }
        double2 acc = make_double2(0, 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = cadd(acc, v[q]);
        out[blockIdx.x * blockDim.x + tid] = acc;
    }
}

template <int MODE>
void run(double2* out, int sms, int iters) {
    const int threads = MODE >= 2 ? 512 : 256;
    size_t smem = sizeof(double2) * (2 * padded_len(4096) + FftShapeX<4096>::TW_LEN);
    cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<MODE><<<sms, threads, smem>>>(out, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_bench<MODE><<<sms, threads, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms * 1e6 / iters;
    const char* names[] = {"A r16/256 1buf tw", "B r16/256 2buf tw", "C r8/512 1buf const", "D r8/512 2buf const"};
    printf("%s: %.1f ns per 4096-pt FFT per SM %s\n", names[MODE], per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    run<0>(out, sms, 400);
    run<1>(out, sms, 400);
    run<2>(out, sms, 400);
    run<3>(out, sms, 400);
    return 0;
}
