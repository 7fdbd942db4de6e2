// Microbenchmark (design tool): TMA tensor-load rate for one Y row of pass 2 — 4096 pieces of
// 16 B at a 32-byte stride (rows t1, t1^1 interleaved) into a 64 KiB shared-memory box — with
// one or two loads in flight per SM.  For comparison: the same bytes as 2048 pieces of 32 B.
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

constexpr int kTerms = 20;
constexpr long long N2 = 4096, N1 = 4096, N = N1 * N2;

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

template <int NBUF>
__global__ void __launch_bounds__(32 * NBUF, 1) k_load(const __grid_constant__ CUtensorMap map, int nrows, int wide,
                                                       long long* cyc, double* sink) {
    extern __shared__ __align__(1024) double2 smem[];
    __shared__ __align__(8) unsigned long long bar[NBUF];
    const int w = threadIdx.x >> 5;
    double2* buf = smem + w * 4096;
    const unsigned bs = (unsigned)__cvta_generic_to_shared(buf);
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&bar[w]);
    if ((threadIdx.x & 31) == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    double acc = 0;
    int ph = 0;
    for (int i = 0; i < nrows; ++i) {
        const int row = (NBUF * (blockIdx.x + i * gridDim.x) + w) % (int)(N1 / 2 * kTerms);
        if ((threadIdx.x & 31) == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(65536) : "memory");
            if (wide)
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(bs),
                    "l"(&map), "r"(0), "r"(0), "r"(0), "r"(row), "r"(mb)
                    : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(bs),
                    "l"(&map), "r"(0), "r"(i & 1), "r"(0), "r"(0), "r"(row), "r"(mb)
                    : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred P;\n"
            "W_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
            "@!P bra W_%=;\n}" ::"r"(mb),
            "r"(ph)
            : "memory");
        ph ^= 1;
        acc += buf[threadIdx.x & 31].x;
        __syncwarp();
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* Y;
    if (cudaMalloc(&Y, sizeof(double2) * N * kTerms) != cudaSuccess) return 1;
    cudaMemset(Y, 0, sizeof(double2) * N * kTerms);
    long long* cyc;
    double* sink;
    cudaMallocManaged(&cyc, sizeof(long long) * sms);
    cudaMalloc(&sink, sizeof(double) * sms * 64);
    auto encode = get_encode();
    for (int wide = 0; wide < 2; ++wide) {
        CUtensorMap map;
        CUresult rc;
        const cuuint64_t rows = (cuuint64_t)(N1 / 2) * kTerms;  // pair rows of all terms
        if (!wide) {
            cuuint64_t dims[5] = {2, 2, 256, 16, rows};
            cuuint64_t strides[4] = {16, 32, 256 * 32, (cuuint64_t)N2 * 32};
            cuuint32_t box[5] = {2, 1, 256, 16, 1};
            cuuint32_t es[5] = {1, 1, 1, 1, 1};
            rc = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)Y, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {  // contiguous half of the pair row: 2048 pieces of 32 B = plain 64 KiB
            cuuint64_t dims[4] = {4, 256, 16, rows};
            cuuint64_t strides[3] = {32, 256 * 32, (cuuint64_t)N2 * 32};
            cuuint32_t box[4] = {4, 256, 8, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            rc = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)Y, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (rc != CUDA_SUCCESS) {
            printf("encode failed %d\n", (int)rc);
            continue;
        }
        for (int nbuf = 1; nbuf <= 2; ++nbuf) {
            const int nrows = 200;
            if (nbuf == 1) {
                cudaFuncSetAttribute(k_load<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
                k_load<1><<<sms, 32, 65536>>>(map, 4, wide, cyc, sink);
                k_load<1><<<sms, 32, 65536>>>(map, nrows, wide, cyc, sink);
            } else {
                cudaFuncSetAttribute(k_load<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
                k_load<2><<<sms, 64, 131072>>>(map, 4, wide, cyc, sink);
                k_load<2><<<sms, 64, 131072>>>(map, nrows, wide, cyc, sink);
            }
            cudaDeviceSynchronize();
            long long cmax = 0;
            for (int i = 0; i < sms; ++i) cmax = cyc[i] > cmax ? cyc[i] : cmax;
            printf("%s, %d in flight per SM: %.0f cycles per 64 KiB box per SM  %s\n",
                   wide ? "2048 pieces of 32 B" : "4096 pieces of 16 B at a 32-byte stride", nbuf,
                   (double)cmax / (nrows * nbuf), cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
