// Pipe-throughput microbenchmarks on this B200 (sm_100a): the FP64 roofline
// denominator (DFMA / DADD / DMUL issue rate per SM per clock) and the
// shared-memory crossbar alternatives the FFT exchanges could use (LDS.128,
// STS.128, SHFL.32), measured with clock64 inside the kernel and CUDA events
// outside.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_pipes scripts/microbench_pipes.cu
//   scripts/microbench_pipes  > profiles/r2_microbench_pipes.txt
// Prints one line per test and a JSON summary (fp64 peak in thread-ops/s at the
// clock measured under this load).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

constexpr int ITERS = 4096;

// 16 independent DFMA chains per thread: issue-bound, not latency-bound
__global__ void k_dfma(double* out, double a, double b, long long* cyc) {
    double r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_dadd(double* out, double a, long long* cyc) {
    double r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = r[i] + a;
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// LDS.128 / STS.128 conflict-free (consecutive 16-byte slots per lane)
// (4096 slots: with 2048 the q and q + 8 accesses aliased and the compiler merged them, which
// doubled the printed rates — 253 / 224 B/clk instead of the real 128 / 112)
__global__ void k_lds128(double* out, long long* cyc) {
    extern __shared__ double2 buf[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = make_double2(i, -i);
    __syncthreads();
    double2 acc = make_double2(0, 0);
    const int base = threadIdx.x & 255;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const double2 v = buf[(base + q * 256 + it) & 4095];
            acc.x += v.x;
            acc.y -= v.y;
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_sts128(double* out, long long* cyc) {
    extern __shared__ double2 buf[];
    const int base = threadIdx.x & 255;
    double2 v = make_double2(threadIdx.x, 1.0);
    const long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            buf[(base + q * 256 + it) & 4095] = v;
            v.x += 1.0;
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = buf[threadIdx.x].x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// SHFL.32 (xor pattern), 16 independent values per thread
__global__ void k_shfl(double* out, long long* cyc) {
    unsigned r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 17 + i;
    const long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = __shfl_xor_sync(0xffffffffu, r[i], (i & 15) + 1) + 1u;
    }
    const long long t1 = clock64();
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    const int threads = 512, blocks = sms;  // 16 warps / SM, as the NUFFT kernels run
    double* out;
    long long* cyc;
    CK(cudaMalloc(&out, sizeof(double) * threads * blocks));
    CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
    long long h[1024];
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaFuncSetAttribute(k_lds128, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_sts128, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    double fp64_ops_per_clk_sm = 0, fp64_ops_per_s = 0, sm_ghz = 0;
    for (int test = 0; test < 5; ++test) {
        const char* name = "";
        double thread_ops = 0, bytes = 0;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0));
            switch (test) {
                case 0: k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-9, cyc); name = "DFMA"; break;
                case 1: k_dadd<<<blocks, threads>>>(out, 1e-9, cyc); name = "DADD"; break;
                case 2: k_lds128<<<blocks, threads, 65536>>>(out, cyc); name = "LDS.128"; break;
                case 3: k_sts128<<<blocks, threads, 65536>>>(out, cyc); name = "STS.128"; break;
                case 4: k_shfl<<<blocks, threads>>>(out, cyc); name = "SHFL.32"; break;
            }
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
        }
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        CK(cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
        double cmax = 0;
        for (int b = 0; b < blocks; ++b) cmax = cmax > h[b] ? cmax : (double)h[b];
        const double per_thread = (test <= 1) ? 16.0 * ITERS : 16.0 * (ITERS / 4);
        thread_ops = per_thread * threads;                 // per SM (one block per SM)
        bytes = (test == 2 || test == 3) ? thread_ops * 16 : (test == 4 ? thread_ops * 4 : 0);
        const double per_clk = thread_ops / cmax;           // thread-ops per SM per clock
        const double ghz = cmax / (ms * 1e6);               // in-kernel cycles over the event time
        printf("%-8s %8.2f thread-ops/clk/SM  %6.2f warp-instr/clk/SM  %7.1f B/clk/SM  (%.3f ms, ~%.3f GHz)\n",
               name, per_clk, per_clk / 32, bytes / cmax, ms, ghz);
        if (test == 0) {
            fp64_ops_per_clk_sm = per_clk;
            sm_ghz = ghz;
            fp64_ops_per_s = per_clk * sms * ghz * 1e9;
        }
    }
    printf("{\"sms\": %d, \"dfma_thread_ops_per_clk_sm\": %.3f, \"sm_ghz_under_dfma\": %.4f, "
           "\"peak_fp64_thread_inst_per_s\": %.6e, \"peak_fp64_tflops_fma2\": %.3f, \"clock_rate_attr_khz\": %d}\n",
           sms, fp64_ops_per_clk_sm, sm_ghz, fp64_ops_per_s, 2 * fp64_ops_per_s / 1e12, clk_khz);
    return 0;
}
