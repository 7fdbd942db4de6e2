// Microbenchmark (design tool): where does a 4096-pt block FFT spend its time?
// MODE bits:  1 = twiddles from the global table (else a register constant)
//             2 = smem exchange between stages (else stages run on registers only)
//             4 = two groups of 256 threads per CTA (named barriers)
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void k_tw(double2* tw, int L) {
    int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < L) tw[m] = unit_root(m, L);
}

template <int MODE, int NS, bool LAST>
__device__ __forceinline__ void stage(double2 (&v)[16], double2* out, int tid, const double2* __restrict__ tw,
                                      double2 wc) {
    constexpr int L = 4096, G = 256;
    const int j = tid;
    const int k = j & (NS - 1);
    double2 a[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) a[t] = v[t];
    if constexpr (NS > 1) {
        constexpr int STEP = L / (NS * 16);
#pragma unroll
        for (int t = 1; t < 16; ++t) {
            double2 w = (MODE & 1) ? __ldg(tw + k * t * STEP) : make_double2(wc.x + t, wc.y);
            a[t] = cmul(a[t], w);
        }
    }
    dft<16, -1>(a);
    if constexpr (LAST || !(MODE & 2)) {
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = a[t];
    } else {
        const int base = (j - k) * 16 + k;
#pragma unroll
        for (int t = 0; t < 16; ++t) out[pad16(base + t * NS)] = a[t];
    }
}

template <int MODE>
__global__ void __launch_bounds__((MODE & 4) ? 512 : 256, 1) k_bench(double2* out, const double2* __restrict__ tw, int iters) {
    constexpr int L = 4096, G = 256;
    extern __shared__ double2 sm[];
    const int grp = (MODE & 4) ? threadIdx.x / G : 0;
    const int tid = threadIdx.x % G;
    double2* buf = sm + grp * padded_len(L);
    double2 v[16];
    const double2 wc = make_double2(0.7 + tid * 1e-6, 0.3);
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
    auto bar = [&] {
        if (MODE & 4) nbar(1 + grp, G); else __syncthreads();
    };
    for (int it = 0; it < iters; ++it) {
        if (MODE & 2) bar();
        stage<MODE, 1, false>(v, buf, tid, tw, wc);
        if (MODE & 2) { bar(); load_stage_input<L>(v, buf, tid); bar(); }
        stage<MODE, 16, false>(v, buf, tid, tw, wc);
        if (MODE & 2) { bar(); load_stage_input<L>(v, buf, tid); }
        stage<MODE, 256, true>(v, buf, tid, tw, wc);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(double2* out, const double2* tw, int sms, int iters) {
    const int threads = (MODE & 4) ? 512 : 256;
    size_t smem = sizeof(double2) * padded_len(4096) * ((MODE & 4) ? 2 : 1);
    cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<MODE><<<sms, threads, smem>>>(out, tw, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_bench<MODE><<<sms, threads, smem>>>(out, tw, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const int groups = (MODE & 4) ? 2 : 1;
    const double per = ms * 1e6 / ((double)groups * iters);
    printf("mode %d (tw=%s, smem=%s, groups=%d): %.1f ns per 4096-pt FFT per SM (%.0f cycles @1.965GHz) %s\n", MODE,
           (MODE & 1) ? "table" : "const", (MODE & 2) ? "yes" : "no", groups, per, per * 1.965,
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
    run<1>(out, tw, sms, iters);
    run<2>(out, tw, sms, iters);
    run<3>(out, tw, sms, iters);
    run<4>(out, tw, sms, iters);
    run<5>(out, tw, sms, iters);
    run<6>(out, tw, sms, iters);
    run<7>(out, tw, sms, iters);
    return 0;
}
