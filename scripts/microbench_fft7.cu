// Microbenchmark (design tool): anti-phased workers.  The two-level 4096-point FFT
// alternates FP64 phases (three 16-point DFT levels + twiddles) and shared-memory
// phases (two exchanges).  One 256-thread worker alone saturates either pipe
// (microbench_fft6), so two free-running workers overlap only by chance.  Here a
// CTA-wide barrier at every phase boundary, with worker 1 started one phase late,
// forces "worker 0 in an FP64 phase while worker 1 is in an exchange" and back.
//   MODE 0: free-running workers (production block_fft_2l)
//   MODE 1: anti-phased, CTA-wide bar.sync at the 4 phase boundaries
//   MODE 2: anti-phased with arrive/sync pairs (a worker only waits for the OTHER
//           worker to have left the phase it is about to enter)
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_bench(double2* out, int iters) {
    constexpr int L = 4096, G = 256;
    extern __shared__ double2 sm[];
    const int grp = threadIdx.x / G, tid = threadIdx.x % G;
    double2* tw = sm + 2 * padded_len(L);
    double2* buf = sm + grp * padded_len(L);
    twiddle_table_build<L>(tw, threadIdx.x, 2 * G);
    Twiddles<L> T;
    twiddle_init<L>(T, tw, tid);
    __syncthreads();
    const int bar = 1 + grp;
    auto gsync = [bar] { bar_sync(bar, G); };
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
    if constexpr (MODE == 0) {
        for (int it = 0; it < iters; ++it) {
            gsync();
            block_fft_2l<-1>(v, buf, tid, T, gsync);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
        }
    } else {
        // phase boundary: MODE 1 = everyone meets; MODE 2 = token passing.  Tokens: barrier 3 =
        // "FP64 pipe free", barrier 4 = "smem pipe free"; a worker leaving an FP64 phase arrives
        // on 3 and syncs on 4 (the other worker has left its exchange), and vice versa.
        auto to_smem = [&] {
            if constexpr (MODE == 1) bar_sync(0, 512);
            else { bar_arrive(3 + 2 * grp, 512); bar_sync(4 + 2 * (grp ^ 1) - 1 + 1, 512); }
        };
        auto to_fp64 = [&] {
            if constexpr (MODE == 1) bar_sync(0, 512);
            else { bar_arrive(4 + 2 * grp, 512); bar_sync(3 + 2 * (grp ^ 1), 512); }
        };
        (void)to_fp64;
        if (grp == 1) {
            if constexpr (MODE == 1) bar_sync(0, 512);
        }
        const int g = fft2l_g(tid), u = fft2l_u(tid), sw = fft2l_swz(g);
        double2* reg = buf + g * 256;
        const double2* rd1 = reg + (u ^ sw);
        for (int it = 0; it < iters; ++it) {
            // F: (previous third level was below) first level
            dft<16, -1>(v);
            apply_pow_twiddles<16, -1>(v, T.tb + tid);
            to_smem();
#pragma unroll
            for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 256 + (tid ^ fft2l_swz(k1))] = v[k1];
            gsync();
#pragma unroll
            for (int m = 0; m < 16; ++m) v[m] = rd1[16 * m];
            to_fp64();
            dft<16, -1>(v);
#pragma unroll
            for (int a = 1; a < 16; ++a) v[a] = cmul(v[a], T.t16[a * 16 + u]);
            to_smem();
            __syncwarp();
            const int U = u ^ sw;
#pragma unroll
            for (int a = 0; a < 16; ++a) reg[16 * a + (U ^ (a & 7))] = v[a];
            __syncwarp();
            double2* rd2 = reg + 16 * u;
            const int A = sw ^ (u & 7);
#pragma unroll
            for (int w = 0; w < 16; ++w) v[w] = rd2[w ^ A];
            to_fp64();
            dft<16, -1>(v);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
        }
        if (grp == 0) {
            if constexpr (MODE == 1) bar_sync(0, 512);
        }
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(double2* out, int sms) {
    constexpr int L = 4096;
    const size_t smem = sizeof(double2) * (2 * padded_len(L) + FftShapeX<L>::TW_LEN);
    cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<MODE><<<sms, 512, smem>>>(out, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k_bench<MODE><<<sms, 512, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms * 1e6 / (2.0 * iters);
    printf("mode %d: %.0f cycles per FFT per SM  %s\n", MODE, per * 1.965, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    run<0>(out, sms);
    run<1>(out, sms);
    return 0;
}
