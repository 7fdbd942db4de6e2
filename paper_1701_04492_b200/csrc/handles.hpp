// Opaque C-ABI handle types and the entry-point guard shared by the C-ABI
// translation units (capi.cu, nufft2_multi.cu).
#pragma once

#include <array>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/nufft_b200.h"
#include "plans.hpp"

struct nufft_plan2 {
    nb::CorePlan core;
    // per-pass timing events for the benchmark (exec_timed / timing_read)
    mutable std::mutex timing_mu;
    mutable std::vector<std::array<cudaEvent_t, 3>> timing;
    ~nufft_plan2() {
        for (auto& e : timing)
            for (auto& x : e) cudaEventDestroy(x);
    }
};
struct nufft_plan1 {
    nb::CorePlan core;
};
struct nufft_plan3 {
    nb::Plan3State st;
};
struct nufft_plan2d {
    nb::Plan2DState st;
};
struct nufft_toeplitz {
    nb::ToeplitzState st;
};

namespace nb {

// the calling thread's message for nufft_last_error() (capi.cu)
std::string& last_error();

// Every entry point leaves the caller's current device as it found it (the
// plan's device is made current inside; a PyTorch caller on another device
// must not see its later allocations move).
struct DeviceRestore {
    int dev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&dev) != cudaSuccess) {
            cudaGetLastError();
            dev = -1;
        }
    }
    ~DeviceRestore() {
        if (dev >= 0) cudaSetDevice(dev);
    }
};

template <class F>
int guard(F&& f) {
    DeviceRestore restore;
    try {
        f();
        return NUFFT_OK;
    } catch (const nb::Error& e) {
        last_error() = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        last_error() = std::string("host allocation failed: ") + e.what();
        return NUFFT_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return NUFFT_INTERNAL;
    }
}


}  // namespace nb
