// Microbenchmark (design tool): (1) FP64 / shared-memory pipe interference measured without
// the artefacts of microbench_pipes.cu (its LDS/STS loops let the compiler merge the q and
// q + 8 accesses, which alias mod 2048: the 253 / 224 B/clk it printed are twice the real
// rates); (2) per-phase clocks of the anti-phased two-worker FFT of microbench_fft7.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// NF warps of DFMA chains, NL warps of LDS.128 (integer consumer, distinct addresses),
// NS warps of STS.128
__global__ void __launch_bounds__(512, 1) k_overlap(double* out, int nf, int nl, int ns, int iters, long long* cyc) {
    extern __shared__ uint4 sbuf[];  // 4096 x 16 B
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sbuf[i] = make_uint4(i, i + 1, i + 2, i + 3);
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
        unsigned acc = 0;
        const int base = threadIdx.x & 255;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint4 v = sbuf[(base + q * 256 + it) & 4095];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
        }
        s = acc;
    } else if (warp < nf + nl + ns) {
        const int base = threadIdx.x & 255;
        uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                sbuf[(base + q * 256 + it) & 4095] = v;
                v.x += 1;
            }
        }
        s = v.x;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
}

__global__ void __launch_bounds__(512, 1) k_phase(double2* out, int iters, long long* ph) {
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
    if (grp == 1) bar_sync(0, 512);
    const int g = fft2l_g(tid), u = fft2l_u(tid), sw = fft2l_swz(g);
    double2* reg = buf + g * 256;
    const double2* rd1 = reg + (u ^ sw);
    long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t = clock64(), n;
#define TICK(i)        \
    n = clock64();     \
    acc[i] += n - t;   \
    t = n;
    for (int it = 0; it < iters; ++it) {
        dft<16, -1>(v);
        apply_pow_twiddles<16, -1>(v, T.tb + tid);
        TICK(0)
        bar_sync(0, 512);
        TICK(1)
#pragma unroll
        for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 256 + (tid ^ fft2l_swz(k1))] = v[k1];
        gsync();
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = rd1[16 * m];
        asm volatile("" ::"d"(v[15].x), "d"(v[0].x));
        TICK(2)
        bar_sync(0, 512);
        TICK(3)
        dft<16, -1>(v);
#pragma unroll
        for (int a = 1; a < 16; ++a) v[a] = cmul(v[a], T.t16[a * 16 + u]);
        TICK(4)
        bar_sync(0, 512);
        TICK(5)
        __syncwarp();
        const int U = u ^ sw;
#pragma unroll
        for (int a = 0; a < 16; ++a) reg[16 * a + (U ^ (a & 7))] = v[a];
        __syncwarp();
        double2* rd2 = reg + 16 * u;
        const int A = sw ^ (u & 7);
#pragma unroll
        for (int w = 0; w < 16; ++w) v[w] = rd2[w ^ A];
        asm volatile("" ::"d"(v[15].x), "d"(v[0].x));
        TICK(6)
        bar_sync(0, 512);
        TICK(7)
        dft<16, -1>(v);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
    }
    if (grp == 0) bar_sync(0, 512);
    double2 s = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) s = cadd(s, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && (tid == 0 || tid == 255))
        for (int i = 0; i < 8; ++i) ph[(grp * 2 + (tid == 255)) * 8 + i] = acc[i];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    long long* cyc;
    cudaMallocManaged(&cyc, sizeof(long long) * sms * 16);
    cudaFuncSetAttribute(k_overlap, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int iters = 2048;
    const int cfgs[][3] = {{8, 0, 0}, {0, 8, 0}, {0, 16, 0}, {0, 0, 8}, {0, 0, 16}, {0, 8, 8}, {8, 8, 0}, {8, 0, 8}, {8, 4, 4}, {4, 4, 4}};
    for (auto& c : cfgs) {
        k_overlap<<<sms, 512, 65536>>>((double*)out, c[0], c[1], c[2], iters, cyc);
        cudaDeviceSynchronize();
        long long fmax = 0, lmax = 0, smax = 0;
        for (int w = 0; w < 16; ++w) {
            if (w < c[0]) fmax = cyc[w] > fmax ? cyc[w] : fmax;
            else if (w < c[0] + c[1]) lmax = cyc[w] > lmax ? cyc[w] : lmax;
            else if (w < c[0] + c[1] + c[2]) smax = cyc[w] > smax ? cyc[w] : smax;
        }
        const double f = fmax ? (double)c[0] * 32 * 16 * iters / fmax : 0.0;
        const double l = lmax ? (double)c[1] * 32 * 16 * 16 * iters / lmax : 0.0;
        const double s = smax ? (double)c[2] * 32 * 16 * 16 * iters / smax : 0.0;
        printf("overlap: %2d DFMA + %2d LDS.128 + %2d STS.128 warps: DFMA %.1f thread-ops/clk/SM, LDS %.1f B/clk/SM, STS %.1f B/clk/SM  %s\n",
               c[0], c[1], c[2], f, l, s, cudaGetErrorString(cudaGetLastError()));
    }
    long long* ph;
    cudaMallocManaged(&ph, sizeof(long long) * 32);
    const size_t smem = sizeof(double2) * (2 * padded_len(4096) + FftShapeX<4096>::TW_LEN);
    cudaFuncSetAttribute(k_phase, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int it2 = 400;
    k_phase<<<sms, 512, smem>>>(out, it2, ph);
    cudaDeviceSynchronize();
    const char* names[8] = {"F3+F1", "bar", "S1", "bar", "F2", "bar", "S2", "bar"};
    for (int w = 0; w < 4; ++w) {
        printf("worker %d thread %3d:", w >> 1, (w & 1) ? 255 : 0);
        for (int i = 0; i < 8; ++i) printf(" %s %lld", names[i], ph[w * 8 + i] / it2);
        printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
