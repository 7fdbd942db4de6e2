// Microbenchmark (design tool): TMA store throughput for the Y column of pass 1 as a function
// of the contiguous piece size.  One 64 KiB shared-memory box (a 4096-point column of
// complex128) per store, two boxes in flight per SM (the two column workers), K = 20 terms:
//   A: the production layout — 2048 pieces of 32 B (rows t1, t1^1 interleaved), 5-D map
//   B: plain row-major Y[r][t1][k2] — 4096 pieces of 16 B at stride N2 * 16 B, 3-D map
//      (adjacent columns, stored by the other worker, complete each 32-byte sector)
// Prints cycles per box per SM and the achieved write bandwidth.
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

template <int MODE>
__global__ void __launch_bounds__(64, 1) k_store(const __grid_constant__ CUtensorMap map, int ncols, long long* cyc) {
    extern __shared__ __align__(1024) double2 smem[];
    const int w = threadIdx.x >> 5;  // worker = warp
    double2* buf = smem + w * 4096;
    for (int i = threadIdx.x & 31; i < 4096; i += 32) buf[i] = make_double2(i, blockIdx.x);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const unsigned bs = (unsigned)__cvta_generic_to_shared(buf);
    const long long t0 = clock64();
    if ((threadIdx.x & 31) == 0) {
        for (int c = 0; c < ncols; ++c) {
            const int k2 = (2 * (blockIdx.x + c * gridDim.x) + w) % (int)N2;
            for (int r = 0; r < kTerms; ++r) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                if (MODE == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&map),
                        "r"(0), "r"(0), "r"(0), "r"(16 * r), "r"(k2), "r"(bs)
                        : "memory");
                } else {
                    asm volatile(
                        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(&map),
                        "r"(0), "r"(k2), "r"(0), "r"(16 * r), "r"(bs)
                        : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* Y;
    if (cudaMalloc(&Y, sizeof(double2) * N * kTerms) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    long long* cyc;
    cudaMallocManaged(&cyc, sizeof(long long) * sms);
    auto encode = get_encode();
    for (int mode = 0; mode < 3; ++mode) {
        CUtensorMap map;
        CUresult rc;
        if (mode == 0) {
            const cuuint64_t row = N2 * 32ull;
            cuuint64_t dims[5] = {4, 16, 8, 16ull * kTerms, (cuuint64_t)N2};
            cuuint64_t strides[4] = {8 * row, row, 128 * row, 32};
            cuuint32_t box[5] = {4, 16, 8, 16, 1};
            cuuint32_t es[5] = {1, 1, 1, 1, 1};
            rc = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)Y, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            // 3-D {2 doubles, k2, t1 + 4096 r}; the box is a 4096-row column of 16-byte pieces.  mode 2: 128B swizzle
            cuuint64_t dims[3] = {2, (cuuint64_t)N2, (cuuint64_t)N1 * kTerms};
            cuuint64_t strides[2] = {16, (cuuint64_t)N2 * 16};
            cuuint32_t box[3] = {2, 1, 256};
            cuuint32_t es[3] = {1, 1, 1};
            // boxDim <= 256 per dimension: a 4096-row column is 16 boxes of 256 rows -> use a 4-D split instead
            cuuint64_t dims4[4] = {2, (cuuint64_t)N2, 256, 16ull * kTerms};
            cuuint64_t strides4[3] = {16, (cuuint64_t)N2 * 16, (cuuint64_t)N2 * 16 * 256};
            cuuint32_t box4[4] = {2, 1, 256, 16};
            cuuint32_t es4[4] = {1, 1, 1, 1};
            (void)dims; (void)strides; (void)box; (void)es;
            rc = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)Y, dims4, strides4, box4, es4,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, mode == 2 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (rc != CUDA_SUCCESS) {
            printf("mode %d: encode failed rc=%d\n", mode, (int)rc);
            continue;
        }
        const int ncols = 8;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms = 0;
        if (mode == 0) {
            cudaFuncSetAttribute(k_store<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
            k_store<0><<<sms, 64, 2 * 65536>>>(map, 1, cyc);
            cudaEventRecord(a);
            k_store<0><<<sms, 64, 2 * 65536>>>(map, ncols, cyc);
            cudaEventRecord(b);
        } else {
            cudaFuncSetAttribute(k_store<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536);
            k_store<1><<<sms, 64, 2 * 65536>>>(map, 1, cyc);
            cudaEventRecord(a);
            k_store<1><<<sms, 64, 2 * 65536>>>(map, ncols, cyc);
            cudaEventRecord(b);
        }
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        long long cmax = 0;
        for (int i = 0; i < sms; ++i) cmax = cyc[i] > cmax ? cyc[i] : cmax;
        const double boxes = 2.0 * ncols * kTerms;
        printf("mode %d (%s): %.0f cycles per 64 KiB box per SM (two in flight), %.2f TB/s written  %s\n", mode,
               mode == 0 ? "32-byte pieces, 5-D" : (mode == 1 ? "16-byte pieces, 4-D" : "16-byte pieces, 4-D, 128B swizzle"),
               cmax / boxes, boxes * sms * 65536.0 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
