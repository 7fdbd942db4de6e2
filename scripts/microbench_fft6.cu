// Microbenchmark (design tool): what bounds the two-level 4096-point block FFT
// (block_fft_2l, fft_block.cuh)?  The same instruction stream with parts removed:
//   FLAGS bit 0: keep the shared-memory exchanges (else registers stay where they are)
//         bit 1: keep the twiddle loads from shared memory (else register constants)
//         bit 2: keep the FP64 work (DFTs and twiddle products)
// plus a pipe-overlap test: warps that only issue DFMA next to warps that only
// issue LDS.128 in the same CTA (does the FP64 rate hold while the LSU is busy?).
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

template <int FLAGS, class Bar>
__device__ __forceinline__ void fft2l_variant(double2 (&v)[16], double2* buf, int tid, const Twiddles<4096>& T, Bar bar,
                                              double2 wc) {
    constexpr bool XCH = FLAGS & 1, TWL = FLAGS & 2, FP = FLAGS & 4;
    if (FP) dft<16, -1>(v);
    if (FP) {
        if (TWL) {
            apply_pow_twiddles<16, -1>(v, T.tb + tid);
        } else {
#pragma unroll
            for (int a = 1; a < 16; ++a) v[a] = cmul(v[a], make_double2(wc.x + a, wc.y));
        }
    }
    if (XCH) {
#pragma unroll
        for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 256 + (tid ^ fft2l_swz(k1))] = v[k1];
        bar();
    }
    const int g = fft2l_g(tid), u = fft2l_u(tid), sw = fft2l_swz(g);
    double2* reg = buf + g * 256;
    const double2* rd1 = reg + (u ^ sw);
    if (XCH) {
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = rd1[16 * m];
    }
    if (FP) dft<16, -1>(v);
    if (FP) {
#pragma unroll
        for (int a = 1; a < 16; ++a)
            v[a] = cmul(v[a], TWL ? T.t16[a * 16 + u] : make_double2(wc.x - a, wc.y));
    } else if (TWL) {
#pragma unroll
        for (int a = 1; a < 16; ++a) v[a].x += T.t16[a * 16 + u].x;
    }
    if (XCH) {
        __syncwarp();
        const int U = u ^ sw;
#pragma unroll
        for (int a = 0; a < 16; ++a) reg[16 * a + (U ^ (a & 7))] = v[a];
        __syncwarp();
        double2* rd2 = reg + 16 * u;
        const int A = sw ^ (u & 7);
#pragma unroll
        for (int w = 0; w < 16; ++w) v[w] = rd2[w ^ A];
    }
    if (FP) dft<16, -1>(v);
}

template <int W, int FLAGS>
__global__ void __launch_bounds__(W * 256, 1) k_bench(double2* out, int iters, double2 wc) {
    constexpr int L = 4096, G = 256;
    extern __shared__ double2 sm[];
    const int grp = threadIdx.x / G, tid = threadIdx.x % G;
    double2* tw = sm + W * padded_len(L);
    double2* b0 = sm + grp * padded_len(L);
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
        if (FLAGS & 1) gsync();
        fft2l_variant<FLAGS>(v, b0, tid, T, gsync, wc);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
    }
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int W, int FLAGS>
void run(double2* out, int sms) {
    constexpr int L = 4096;
    const size_t smem = sizeof(double2) * (W * padded_len(L) + FftShapeX<L>::TW_LEN);
    cudaFuncSetAttribute(k_bench<W, FLAGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const double2 wc = make_double2(0.999, 0.001);
    k_bench<W, FLAGS><<<sms, W * 256, smem>>>(out, 2, wc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k_bench<W, FLAGS><<<sms, W * 256, smem>>>(out, iters, wc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms * 1e6 / ((double)W * iters);
    printf("workers=%d exchange=%d twiddle-loads=%d fp64=%d : %.0f cycles per FFT per SM  %s\n", W, FLAGS & 1,
           (FLAGS >> 1) & 1, (FLAGS >> 2) & 1, per * 1.965, cudaGetErrorString(cudaGetLastError()));
}

// pipe overlap: NF warps of DFMA chains + NL warps of LDS.128 in one CTA
__global__ void __launch_bounds__(512, 1) k_overlap(double* out, int nf, int nl, int iters, long long* cyc) {
    __shared__ double2 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    const long long t0 = clock64();
    double s = 0;
    if (warp < nf) {
        double r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = fma(r[i], 0.999, 0.001);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) s += r[i];
    } else if (warp < nf + nl) {
        double2 acc = make_double2(0, 0);
        const int base = threadIdx.x & 255;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 v = buf[(base + q * 256 + it) & 2047];
                acc.x += v.x;
            }
        }
        s = acc.x;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    run<2, 7>(out, sms);
    run<2, 6>(out, sms);
    run<2, 4>(out, sms);
    run<2, 5>(out, sms);
    run<2, 3>(out, sms);
    run<2, 1>(out, sms);
    run<1, 7>(out, sms);
    run<1, 6>(out, sms);
    run<1, 4>(out, sms);
    run<1, 1>(out, sms);
    long long* cyc;
    cudaMallocManaged(&cyc, sizeof(long long) * sms * 16);
    const int iters = 2048;
    const int cfgs[][2] = {{8, 0}, {16, 0}, {0, 8}, {0, 16}, {8, 8}, {4, 4}, {12, 4}, {4, 12}};
    for (auto& c : cfgs) {
        k_overlap<<<sms, 512>>>((double*)out, c[0], c[1], iters, cyc);
        cudaDeviceSynchronize();
        long long fmax = 0, lmax = 0;
        for (int w = 0; w < 16; ++w) {
            if (w < c[0]) fmax = cyc[w] > fmax ? cyc[w] : fmax;
            else if (w < c[0] + c[1]) lmax = cyc[w] > lmax ? cyc[w] : lmax;
        }
        // DFMA thread-ops per clk per SM and LDS bytes per clk per SM, each over its own warps' duration
        const double f = fmax ? (double)c[0] * 32 * 16 * iters / fmax : 0.0;
        const double l = lmax ? (double)c[1] * 32 * 16 * 16 * iters / lmax : 0.0;
        printf("overlap: %2d DFMA warps + %2d LDS.128 warps: DFMA %.1f thread-ops/clk/SM (%lld cyc), LDS %.1f B/clk/SM (%lld cyc)\n",
               c[0], c[1], f, fmax, l, lmax);
    }
    return 0;
}
