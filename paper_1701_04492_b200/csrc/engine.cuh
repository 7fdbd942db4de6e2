// Host-side engine interfaces shared by the transform implementations.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace nb {

// Per-device constants: forward twiddle tables tw_L[m] = exp(-2 pi i m/L) for
// L = 2^l, l = 1..12 (consumed by the block FFT), created once per device.
struct DeviceCtx {
    int device = 0;
    int sms = 0;
    const double2* tw[13] = {};
    cudaMemPool_t pool = nullptr;  // the library's own scratch pool (never the device default)
    static DeviceCtx& get(int device);
    const double2* table(int L) const { return tw[ilog2(static_cast<size_t>(L))]; }
};

// RAII stream-ordered device buffer (cudaMallocFromPoolAsync / cudaFreeAsync on
// the library's private memory pool of the current device: its release
// threshold is raised so repeated executions reuse scratch instead of
// re-allocating, and trim_scratch() hands the cached memory back — the
// device's default pool, which PyTorch and other libraries share, is left
// alone).
class DevBuf {
  public:
    DevBuf() = default;
    DevBuf(size_t bytes, cudaStream_t s) { alloc(bytes, s); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), s_(o.s_) { o.p_ = nullptr; }
    void alloc(size_t bytes, cudaStream_t s);
    void release();
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    void* get() const { return p_; }

  private:
    void* p_ = nullptr;
    cudaStream_t s_ = nullptr;
};

// Persistent device allocation (plan-owned buffers).
class DevArray {
  public:
    DevArray() = default;
    explicit DevArray(size_t bytes) { alloc(bytes); }
    ~DevArray();
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; }
    DevArray& operator=(DevArray&& o) noexcept;
    void alloc(size_t bytes);
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    size_t bytes() const { return bytes_; }

  private:
    void* p_ = nullptr;
    size_t bytes_ = 0;
};

// host <-> device copies that stage pageable host memory through the library's
// page-locked ring (host_stage.cu); page-locked memory goes straight to the copy
// engine.  h2d is ordered on s (returns once `src` may be reused); d2h returns
// when `dst` holds the data.
bool host_pageable(const void* p);
void h2d(void* dst_dev, const void* src_host, size_t bytes, cudaStream_t s);
void d2h(void* dst_host, const void* src_dev, size_t bytes, cudaStream_t s);

// release the scratch cached in the device's private pool (plan destruction)
void trim_scratch(int device);

// ---- logical FFT execution counters (fft.hpp:91-95,126-137 test hook) -----
void fft_count(size_t n, uint64_t times = 1);
uint64_t fft_exec_count(size_t n);
void fft_reset_exec_counts();
unsigned long long launch_count();

// ---- generic uniform FFT engine (any n >= 1, batched, contiguous) --------
// out may equal in.  sign -1 forward, +1 backward (unnormalized).  Does NOT
// touch the logical counters (callers count logical transforms).
void fft_exec(const double2* in, double2* out, size_t n, size_t batch, int sign, cudaStream_t s,
              int device);
// batched out-of-place transpose: in is batch x rows x cols, out batch x cols x rows
void transpose(const double2* in, double2* out, size_t rows, size_t cols, size_t batch,
               cudaStream_t s);

}  // namespace nb
