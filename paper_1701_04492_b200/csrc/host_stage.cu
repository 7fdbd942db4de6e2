// Staged host <-> device copies for PAGEABLE host memory (the *_host entry
// points, i.e. what the drop-in C++ API passes from std::vector).
//
// cudaMemcpy from pageable memory is staged by the driver through its own small
// page-locked buffers, one copy engine at a time, and a device->host copy blocks
// the calling thread: at N = 2^24 (256 MiB each way) that ran at a fraction of
// the PCIe bandwidth.  Here every transfer moves in chunks through a ring of
// page-locked buffers owned by the library (per device, allocated once): a pool
// of host threads copies chunk i + 1 between the caller's memory and a ring
// slot while the copy engine moves chunk i, so PCIe and host memory bandwidth
// overlap.  Page-locked caller memory skips all of this (plain cudaMemcpyAsync).
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.cuh"

namespace nb {

namespace {

// persistent workers for parallel memcpy (created on first use)
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    // dst[0, n) = src[0, n), split across the workers and the calling thread
    void copy(void* dst, const void* src, size_t n) {
        const size_t parts = std::min<size_t>(workers_.size() + 1, std::max<size_t>(1, n >> 20));
        if (parts <= 1) {
            std::memcpy(dst, src, n);
            return;
        }
        const size_t step = ((n + parts - 1) / parts + 63) & ~size_t(63);
        {
            std::unique_lock<std::mutex> lk(mu_);
            for (size_t p = 1; p < parts; ++p) {
                const size_t a = std::min(n, p * step), b = std::min(n, a + step);
                if (b > a) {
                    jobs_.push_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
                    ++pending_;
                }
            }
        }
        cv_.notify_all();
        std::memcpy(dst, src, std::min(n, step));
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
        const unsigned nw = std::min(7u, hw - 1);
        for (unsigned i = 0; i < nw; ++i) workers_.emplace_back([this] { run(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void run() {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
                if (stop_ && jobs_.empty()) return;
                job = std::move(jobs_.back());
                jobs_.pop_back();
            }
            job();
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::vector<std::thread> workers_;
    std::vector<std::function<void()>> jobs_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    size_t pending_ = 0;
    bool stop_ = false;
};

constexpr size_t kChunk = size_t(16) << 20;  // bytes per ring slot
constexpr int kSlots = 4;                    // ring depth per direction

struct Ring {
    char* buf[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    bool used[kSlots] = {};
};

struct Stager {
    std::mutex mu;  // one staged transfer at a time per device
    Ring in, out;
    explicit Stager(int device) {
        NB_CUDA(cudaSetDevice(device));
        for (Ring* r : {&in, &out})
            for (int i = 0; i < kSlots; ++i) {
                NB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&r->buf[i]), kChunk, cudaHostAllocPortable));
                NB_CUDA(cudaEventCreateWithFlags(&r->ev[i], cudaEventDisableTiming));
            }
    }
};

Stager& stager(int device) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Stager>> m;
    std::lock_guard<std::mutex> lk(mu);
    auto& p = m[device];
    if (!p) p = std::make_unique<Stager>(device);
    return *p;
}

}  // namespace

bool host_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (!host_pageable(src) || bytes <= kChunk / 4) {
        NB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    int dev = 0;
    NB_CUDA(cudaGetDevice(&dev));
    Stager& st = stager(dev);
    std::lock_guard<std::mutex> lk(st.mu);
    Ring& r = st.in;
    size_t off = 0;
    for (int i = 0; off < bytes; ++i) {
        const int k = i % kSlots;
        const size_t len = std::min(kChunk, bytes - off);
        if (r.used[k]) NB_CUDA(cudaEventSynchronize(r.ev[k]));  // the engine has read the slot
        CopyPool::get().copy(r.buf[k], static_cast<const char*>(src) + off, len);
        NB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, r.buf[k], len, cudaMemcpyHostToDevice, s));
        NB_CUDA(cudaEventRecord(r.ev[k], s));
        r.used[k] = true;
        off += len;
    }
    // returns with the last chunks in flight: `src` is free to reuse, the slots are
    // guarded by their events, and the data is ordered on `s`
}

void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    if (!host_pageable(dst) || bytes <= kChunk / 4) {
        NB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    int dev = 0;
    NB_CUDA(cudaGetDevice(&dev));
    Stager& st = stager(dev);
    std::lock_guard<std::mutex> lk(st.mu);
    Ring& r = st.out;
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) {
        const int k = (int)(i % kSlots);
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        NB_CUDA(cudaMemcpyAsync(r.buf[k], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaEventRecord(r.ev[k], s));
    };
    for (size_t i = 0; i < std::min<size_t>(kSlots, nchunks); ++i) issue(i);
    for (size_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kSlots);
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        NB_CUDA(cudaEventSynchronize(r.ev[k]));
        CopyPool::get().copy(static_cast<char*>(dst) + off, r.buf[k], len);
        if (i + kSlots < nchunks) issue(i + kSlots);
    }
    for (auto& u : r.used) u = false;
}

}  // namespace nb
