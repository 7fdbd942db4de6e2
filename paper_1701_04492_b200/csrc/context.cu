// Per-device context, stream-ordered scratch, logical FFT counters.
#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>

#include "engine.cuh"

namespace nb {

namespace {
__global__ void k_twiddle_table(double2* tw, int L) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m < L) tw[m] = unit_root(m, L);
}

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DeviceCtx>> g_ctx;

std::mutex g_count_mu;
std::atomic<unsigned long long> g_launches{0};
std::map<size_t, uint64_t> g_counts;
}  // namespace

namespace {
cudaMemPool_t create_pool(int device) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    NB_CUDA(cudaMemPoolCreate(&pool, &props));
    uint64_t threshold = UINT64_MAX;
    NB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    return pool;
}
}  // namespace

void trim_scratch(int device) {
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lock(g_ctx_mu);
        auto it = g_ctx.find(device);
        if (it == g_ctx.end()) return;
        pool = it->second->pool;
    }
    cudaMemPoolTrimTo(pool, 0);  // unused blocks only; live allocations are untouched
}

DeviceCtx& DeviceCtx::get(int device) {
    std::lock_guard<std::mutex> lock(g_ctx_mu);
    auto it = g_ctx.find(device);
    if (it != g_ctx.end()) return *it->second;
    auto ctx = std::make_unique<DeviceCtx>();
    ctx->device = device;
    NB_CUDA(cudaSetDevice(device));
    ctx->sms = sm_count(device);
    ctx->pool = create_pool(device);
    for (int l = 1; l <= 12; ++l) {
        const int L = 1 << l;
        double2* p = nullptr;
        NB_CUDA(cudaMalloc(&p, sizeof(double2) * L));
        k_twiddle_table<<<(L + 255) / 256, 256>>>(p, L);
        NB_LAUNCH();
        ctx->tw[l] = p;
    }
    NB_CUDA(cudaDeviceSynchronize());
    auto& ref = *ctx;
    g_ctx.emplace(device, std::move(ctx));
    return ref;
}

void DevBuf::alloc(size_t bytes, cudaStream_t s) {
    release();
    s_ = s;
    if (bytes == 0) bytes = 16;
    int dev = 0;
    NB_CUDA(cudaGetDevice(&dev));
    NB_CUDA(cudaMallocFromPoolAsync(&p_, bytes, DeviceCtx::get(dev).pool, s));
}
void DevBuf::release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
}

DevArray::~DevArray() {
    if (p_) cudaFree(p_);
}
DevArray& DevArray::operator=(DevArray&& o) noexcept {
    if (this != &o) {
        if (p_) cudaFree(p_);
        p_ = o.p_;
        bytes_ = o.bytes_;
        o.p_ = nullptr;
        o.bytes_ = 0;
    }
    return *this;
}
void DevArray::alloc(size_t bytes) {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    bytes_ = bytes;
    NB_CUDA(cudaMalloc(&p_, bytes ? bytes : 16));
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(); }

void fft_count(size_t n, uint64_t times) {
    std::lock_guard<std::mutex> lock(g_count_mu);
    g_counts[n] += times;
}
uint64_t fft_exec_count(size_t n) {
    std::lock_guard<std::mutex> lock(g_count_mu);
    auto it = g_counts.find(n);
    return it == g_counts.end() ? 0 : it->second;
}
void fft_reset_exec_counts() {
    std::lock_guard<std::mutex> lock(g_count_mu);
    g_counts.clear();
}

}  // namespace nb
