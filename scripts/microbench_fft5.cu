// Microbenchmark (design tool): the two-level 4096-point block FFT
// (block_fft_2l: one group-wide exchange + a half-warp 16x16 transpose) against
// the production three-stage single-buffer FFT (block_fft_1buf), with W
// independent 256-thread workers per SM.  Also checks block_fft_2l against
// block_fft on one random input.  Reports cycles per 4096-point FFT per SM.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

__global__ void __launch_bounds__(256, 1) k_check(const double2* in, double2* out_ref, double2* out_2l) {
    constexpr int L = 4096;
    extern __shared__ double2 sm[];
    double2* b0 = sm;
    double2* b1 = sm + padded_len(L);
    double2* tw = sm + 2 * padded_len(L);
    const int tid = threadIdx.x;
    twiddle_table_build<L>(tw, tid, 256);
    Twiddles<L> T;
    twiddle_init<L>(T, tw, tid);
    __syncthreads();
    double2 v[16];
    for (int q = 0; q < 16; ++q) v[q] = in[tid + 256 * q];
    block_fft<L, -1>(v, b0, b1, tid, T, [] { __syncthreads(); });
    for (int q = 0; q < 16; ++q) out_ref[tid + 256 * q] = v[q];
    __syncthreads();
    for (int q = 0; q < 16; ++q) v[q] = in[tid + 256 * q];
    block_fft_2l<-1>(v, b0, tid, T, [] { __syncthreads(); });
    for (int b = 0; b < 16; ++b) out_2l[fft2l_out_index(tid, b)] = v[b];
}

// MODE 0: block_fft_1buf; 1: block_fft_2l one buffer per worker (2 barriers);
// 2: block_fft_2l ping-pong pair per worker (1 barrier)
template <int W, int MODE>
__global__ void __launch_bounds__(W * 256, 1) k_bench(double2* out, int iters) {
    constexpr int L = 4096, G = 256;
    constexpr int NB = MODE == 2 ? 2 : 1;
    extern __shared__ double2 sm[];
    const int grp = threadIdx.x / G, tid = threadIdx.x % G;
    double2* tw = sm + W * NB * padded_len(L);
    double2* b0 = sm + grp * NB * padded_len(L);
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
        if constexpr (MODE == 0) {
            gsync();
            block_fft_1buf<L, -1>(v, b0, tid, T, gsync);
        } else if constexpr (MODE == 1) {
            gsync();
            block_fft_2l<-1>(v, b0, tid, T, gsync);
        } else {
            block_fft_2l<-1>(v, b0 + (it & 1) * padded_len(L), tid, T, gsync);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int W, int MODE>
void run(double2* out, int sms) {
    constexpr int L = 4096;
    const size_t smem = sizeof(double2) * (W * (MODE == 2 ? 2 : 1) * padded_len(L) + FftShapeX<L>::TW_LEN);
    if (smem > 227 * 1024) return;
    cudaFuncSetAttribute(k_bench<W, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<W, MODE><<<sms, W * 256, smem>>>(out, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k_bench<W, MODE><<<sms, W * 256, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms * 1e6 / ((double)W * iters);
    static const char* names[] = {"1buf (3 stages, 4 barriers)", "2l one buffer (2 barriers)", "2l ping-pong (1 barrier)"};
    printf("workers=%d %-30s: %.0f ns = %.0f cycles per FFT per SM  %s\n", W, names[MODE], per, per * 1.965,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    constexpr int L = 4096;
    double2 *in, *r1, *r2;
    cudaMallocManaged(&in, L * sizeof(double2));
    cudaMallocManaged(&r1, L * sizeof(double2));
    cudaMallocManaged(&r2, L * sizeof(double2));
    unsigned long long s = 12345;
    for (int i = 0; i < L; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        in[i].x = (double)(s >> 11) / 9007199254740992.0 - 0.5;
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        in[i].y = (double)(s >> 11) / 9007199254740992.0 - 0.5;
    }
    const size_t smc = sizeof(double2) * (2 * padded_len(L) + FftShapeX<L>::TW_LEN);
    cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    k_check<<<1, 256, smc>>>(in, r1, r2);
    cudaDeviceSynchronize();
    double num = 0, den = 0;
    for (int i = 0; i < L; ++i) {
        num += (r1[i].x - r2[i].x) * (r1[i].x - r2[i].x) + (r1[i].y - r2[i].y) * (r1[i].y - r2[i].y);
        den += r1[i].x * r1[i].x + r1[i].y * r1[i].y;
    }
    printf("check 2l vs block_fft: rel l2 %.3e (%s)\n", std::sqrt(num / den), cudaGetErrorString(cudaGetLastError()));
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    run<1, 0>(out, sms);
    run<2, 0>(out, sms);
    run<3, 0>(out, sms);
    run<1, 1>(out, sms);
    run<2, 1>(out, sms);
    run<3, 1>(out, sms);
    run<1, 2>(out, sms);
    return 0;
}
