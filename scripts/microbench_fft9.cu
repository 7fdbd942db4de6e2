// Microbenchmark (design tool): second-level twiddles of block_fft_2l.
//   V0: production (15 LDS.128 from the [a][u] table between the DFT and the transpose)
//   V1: 4 base loads w_256^{u 2^e} + generated powers (apply_pow_twiddles, +44 FP64 / thread)
//   V2: V1 with the base loads issued before the first exchange (registers carry them)
// two free-running 256-thread workers per SM; cycles per FFT per SM
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1701_04492_b200/csrc/fft_block.cuh"

using namespace nb;

__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int SIGN>
__device__ __forceinline__ void pow_tw_regs(double2* a, double2 p1, double2 p2, double2 p4, double2 p8) {
    const double2 p3 = cmul(p1, p2);
    a[1] = cmul(a[1], p1);
    a[2] = cmul(a[2], p2);
    a[3] = cmul(a[3], p3);
    const double2 p5 = cmul(p1, p4), p6 = cmul(p2, p4), p7 = cmul(p3, p4);
    a[4] = cmul(a[4], p4);
    a[5] = cmul(a[5], p5);
    a[6] = cmul(a[6], p6);
    a[7] = cmul(a[7], p7);
    a[8] = cmul(a[8], p8);
    a[9] = cmul(a[9], cmul(p1, p8));
    a[10] = cmul(a[10], cmul(p2, p8));
    a[11] = cmul(a[11], cmul(p3, p8));
    a[12] = cmul(a[12], cmul(p4, p8));
    a[13] = cmul(a[13], cmul(p5, p8));
    a[14] = cmul(a[14], cmul(p6, p8));
    a[15] = cmul(a[15], cmul(p7, p8));
}

template <int V, class Bar, class Ph>
__device__ __forceinline__ void fft2l_v(double2 (&v)[16], double2* buf, int tid, const Twiddles<4096>& T,
                                        const double2* t2b, Bar bar, Ph ph) {
    dft<16, -1>(v);
    apply_pow_twiddles<16, -1>(v, T.tb + tid);
    const int g = fft2l_g(tid), u = fft2l_u(tid), sw = fft2l_swz(g);
    double2 q1, q2, q4, q8;
    if (V >= 2) {
        q1 = t2b[u]; q2 = t2b[16 + u]; q4 = t2b[32 + u]; q8 = t2b[48 + u];
    }
    ph();
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) buf[k1 * 256 + (tid ^ fft2l_swz(k1))] = v[k1];
    bar();
    double2* reg = buf + g * 256;
    const double2* rd1 = reg + (u ^ sw);
    if (V == 3) {
#pragma unroll
        for (int m0 = 0; m0 < 4; ++m0)
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) v[m0 + 4 * m1] = rd1[16 * (m0 + 4 * m1)];
    } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = rd1[16 * m];
    }
    if (V == 1) {
        q1 = t2b[u]; q2 = t2b[16 + u]; q4 = t2b[32 + u]; q8 = t2b[48 + u];
    }
    ph();
    dft<16, -1>(v);
    if (V == 0) {
#pragma unroll
        for (int a = 1; a < 16; ++a) v[a] = cmul(v[a], T.t16[a * 16 + u]);
    } else {
        pow_tw_regs<-1>(v, q1, q2, q4, q8);
    }
    ph();
    __syncwarp();
    const int U = u ^ sw;
#pragma unroll
    for (int a = 0; a < 16; ++a) reg[16 * a + (U ^ (a & 7))] = v[a];
    __syncwarp();
    double2* rd2 = reg + 16 * u;
    const int A = sw ^ (u & 7);
    if (V == 3) {
#pragma unroll
        for (int m0 = 0; m0 < 4; ++m0)
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) v[m0 + 4 * m1] = rd2[(m0 + 4 * m1) ^ A];
    } else {
#pragma unroll
        for (int w = 0; w < 16; ++w) v[w] = rd2[w ^ A];
    }
    ph();
    dft<16, -1>(v);
}

template <int V>
__global__ void __launch_bounds__(512, 1) k_bench(double2* out, int iters) {
    constexpr int L = 4096, G = 256;
    extern __shared__ double2 sm[];
    const int grp = threadIdx.x / G, tid = threadIdx.x % G;
    double2* tw = sm + 2 * padded_len(L);
    double2* t2b = tw + FftShapeX<L>::TW_LEN;
    double2* buf = sm + grp * padded_len(L);
    twiddle_table_build<L>(tw, threadIdx.x, 2 * G);
    if (threadIdx.x < 64) t2b[threadIdx.x] = unit_root((long long)(threadIdx.x & 15) << (threadIdx.x >> 4), 256);
    Twiddles<L> T;
    twiddle_init<L>(T, tw, tid);
    __syncthreads();
    const int bar = 1 + grp;
    auto gsync = [bar] { bar_sync(bar, G); };
    double2 v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = make_double2(tid * 1e-3 + q, blockIdx.x * 1e-3 - q);
    if (V == 4 && grp == 1) bar_sync(0, 512);
    for (int it = 0; it < iters; ++it) {
        if (V != 4) gsync();
        if (V == 4) fft2l_v<2>(v, buf, tid, T, t2b, gsync, [] { bar_sync(0, 512); });
        else fft2l_v<V>(v, buf, tid, T, t2b, gsync, [] {});
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = cscale(v[q], 1.0 / 64.0);
    }
    if (V == 4 && grp == 0) bar_sync(0, 512);
    double2 acc = make_double2(0, 0);
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = cadd(acc, v[q]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int V>
void run(double2* out, int sms) {
    constexpr int L = 4096;
    const size_t smem = sizeof(double2) * (2 * padded_len(L) + FftShapeX<L>::TW_LEN + 64);
    cudaFuncSetAttribute(k_bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<V><<<sms, 512, smem>>>(out, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 400;
    cudaEventRecord(a);
    k_bench<V><<<sms, 512, smem>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double per = ms * 1e6 / (2.0 * iters);
    printf("variant %d: %.0f cycles per FFT per SM  %s\n", V, per * 1.965, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    cudaMalloc(&out, sizeof(double2) * sms * 1024);
    run<0>(out, sms);
    run<1>(out, sms);
    run<2>(out, sms);
    run<3>(out, sms);
    run<4>(out, sms);
    return 0;
}
