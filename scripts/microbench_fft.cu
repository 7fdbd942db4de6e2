// Microbenchmark (design tool, not product): throughput of 4096-point fp64
// block FFTs per SM under different CTA organizations, to choose the pass
// structure.  Each CTA loops over `iters` FFTs on smem/register data (no HBM
// in the loop).  Variants:
//   0: 1 group of 256 threads, ping-pong buffers, twiddles from the global table
//   1: 2 independent groups of 256 threads (named barriers), 1 buffer each, global table
//   2: like 1, stage-3 twiddles computed per FFT from w^tid, w^(4 tid) (13 cmul)
//   3: 2 CTAs per SM of 256 threads, 1 buffer each, global table
//   4: 1 group, 1 buffer, global table
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void k_tw(double2* tw, int L) {
    int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < L) tw[m] = unit_root(m, L);
}

template <int VAR>
__global__ void __launch_bounds__(VAR == 1 || VAR == 2 ? 512 : 256, VAR == 3 ? 2 : 1)
    k_bench(double2* out, const double2* __restrict__ tw, int iters) {
    constexpr int L = 4096, G = 256;
    extern __shared__ double2 sm[];
    const int grp = (VAR == 1 || VAR == 2) ? threadIdx.x / G : 0;
    const int tid = threadIdx.x % G;
    double2* b0 = sm + grp * padded_len(L) * (VAR == 0 ? 2 : 1);
    double2* b1 = b0 + padded_len(L);
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
    for (int it = 0; it < iters; ++it) {
        if constexpr (VAR == 0) {
            block_fft<L, -1>(v, b0, b1, tid, tw, [] { __syncthreads(); });
        } else if constexpr (VAR == 3 || VAR == 4) {
            __syncthreads();
            block_fft_1buf<L, -1>(v, b0, tid, tw, [] { __syncthreads(); });
        } else {
            nbar(1 + grp, G);
            block_fft_1buf<L, -1>(v, b0, tid, tw, [grp] { nbar(1 + grp, G); });
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);  // keep magnitudes bounded
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int VAR>
void run(double2* out, const double2* tw, int sms, int iters) {
    const int threads = (VAR == 1 || VAR == 2) ? 512 : 256;
    const int ctas_per_sm = VAR == 3 ? 2 : 1;
    size_t smem = sizeof(double2) * padded_len(4096) * ((VAR == 0 || VAR == 1 || VAR == 2) ? 2 : 1);
    cudaFuncSetAttribute(k_bench<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms * ctas_per_sm;
    k_bench<VAR><<<grid, threads, smem>>>(out, tw, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_bench<VAR><<<grid, threads, smem>>>(out, tw, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const int groups = (VAR == 1 || VAR == 2) ? 2 : 1;
    const double ffts = (double)grid * groups * iters;
    const double pts = ffts * 4096;
    printf("variant %d: %.3f ms, %.1f ns per 4096-pt FFT per SM, %.2f Gpt/s (one r of a 2^24 pass: %.3f ms) err=%s\n",
           VAR, ms, ms * 1e6 / (ffts / sms), pts / ms / 1e6, (1 << 24) / (pts / ms / 1e3) * 1e3,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2 *out, *tw;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    cudaMalloc(&tw, sizeof(double2) * 4096);
    k_tw<<<16, 256>>>(tw, 4096);
    const int iters = 400;
    run<0>(out, tw, sms, iters);
    run<4>(out, tw, sms, iters);
    run<1>(out, tw, sms, iters);
    run<3>(out, tw, sms, iters);
    return 0;
}
