// C-ABI of the B200 low-rank NUFFT (include/nufft_b200.h).
//
// Validation order and messages follow the reference so the C++ layer can
// re-throw the same exception types at the same points:
//   plan_nufft2 transforms.hpp:133-147, plan_nufft1 :246-285,
//   plan_nufft3 :321-380, plan_nufft2d2 transform2d.hpp:65-100,
//   exec length checks :171, :208, :384, transform2d.hpp:109-110.
#include <array>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/nufft_b200.h"
#include "handles.hpp"
#include "lowrank_host.hpp"
#include "plans.hpp"

namespace {

using nb::guard;
using nb::DeviceRestore;

constexpr int kMaxTimingSlots = 1 << 16;  // exec_timed event slots per plan

cudaStream_t as_stream(void* s) { return s ? static_cast<cudaStream_t>(s) : cudaStreamPerThread; }

int pick_device(int device) {
    int count = 0;
    NB_CUDA(cudaGetDeviceCount(&count));
    if (count == 0) throw nb::Error(nb::kCudaError, "no CUDA device");
    if (device < 0) NB_CUDA(cudaGetDevice(&device));
    if (device >= count) nb::throw_invalid("device index out of range");
    NB_CUDA(cudaSetDevice(device));
    nb::DeviceCtx::get(device);
    return device;
}

void check_epsilon(double eps) {  // transforms.hpp:118-121
    if (!(eps > 0.0) || !(eps < 1.0)) nb::throw_domain("epsilon must be in (0, 1)");
}
void check_size(size_t n) {
    if (n >= (size_t(1) << 31)) nb::throw_invalid("transform size exceeds 2^31 - 1 samples");
}

inline unsigned blocks(size_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

__global__ void k_scale(double2* v, long long n, double s) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) v[i] = make_double2(v[i].x * s, v[i].y * s);
}
__global__ void k_any_wrap(const long long* s, const long long* t, long long n, int* flag) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && s[i] != t[i]) atomicOr(flag, 1);
}
__global__ void k_flat_index(const long long* tx, const long long* ty, long long count, long long m,
                             long long* flat) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < count) flat[j] = m * tx[j] + ty[j];
}
__global__ void k_omega_scaled(double* w, long long n) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < n) w[k] = (double)k / (double)n;
}
__global__ void k_fill_ones(double2* u, long long n) {
    const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < n) u[k] = make_double2(1.0, 0.0);
}

template <class T>
void d2h(T* dst, const nb::DevArray& src, size_t count, cudaStream_t s) {
    NB_CUDA(cudaMemcpyAsync(dst, src.as<T>(), sizeof(T) * count, cudaMemcpyDeviceToHost, s));
}

// host -> device -> op -> host with stream-ordered scratch
template <class Op>
void host_roundtrip(const double* in, size_t in_doubles, double* out, size_t out_doubles,
                    cudaStream_t s, Op op) {
    nb::DevBuf din(8 * in_doubles, s), dout(8 * out_doubles, s);
    nb::h2d(din.get(), in, 8 * in_doubles, s);
    op(din.as<double2>(), dout.as<double2>());
    nb::d2h(out, dout.get(), 8 * out_doubles, s);
}

void materialize_u(const nb::CorePlan& p, double2* u_dev, cudaStream_t s) {
    if (p.uniform) {
        k_fill_ones<<<blocks(p.n), 256, 0, s>>>(u_dev, (long long)p.n);
        NB_LAUNCH();
    } else {
        nb::factors_u(p.ax.delta.as<double>(), p.n, p.gamma_factors, p.K, u_dev, s);
    }
}
void materialize_v(const nb::CorePlan& p, double2* v_dev, cudaStream_t s) {
    if (p.uniform) {
        k_fill_ones<<<blocks(p.n), 256, 0, s>>>(v_dev, (long long)p.n);
        NB_LAUNCH();
        return;
    }
    nb::DevBuf w(8 * p.n, s);
    k_omega_scaled<<<blocks(p.n), 256, 0, s>>>(w.as<double>(), (long long)p.n);
    NB_LAUNCH();
    nb::factors_v(w.as<double>(), p.n, p.K, v_dev, s);
}

void core_samples(const nb::CorePlan& p, double* x, long* sv, size_t* t) {
    cudaStream_t s = cudaStreamPerThread;
    NB_CUDA(cudaSetDevice(p.device));
    if (x) d2h(x, p.ax.x, p.n, s);
    static_assert(sizeof(long) == 8 && sizeof(size_t) == 8, "LP64");
    if (sv) d2h(reinterpret_cast<long long*>(sv), p.ax.s, p.n, s);
    if (t) d2h(reinterpret_cast<long long*>(t), p.ax.t, p.n, s);
    NB_CUDA(cudaStreamSynchronize(s));
}

void fill_info(const nb::CorePlan& p, nufft_plan_info* info) {
    std::memset(info, 0, sizeof(*info));
    info->n = p.n;
    info->rank = p.K;
    info->rank2 = p.K;
    info->effective_rank = p.K;
    info->gamma = p.ax.gamma;
    info->epsilon = p.epsilon;
    info->btrivial = 1;
    info->device = p.device;
    info->path = p.fused ? 1 : 0;
}

// fft.hpp:161-178 on the device: rows contiguous; columns via transpose
void rows_fft(double2* d, size_t rows, size_t cols, cudaStream_t s, int dev) {
    nb::fft_exec(d, d, cols, rows, -1, s, dev);
    nb::fft_count(cols, rows);
}
void cols_fft(double2* d, size_t rows, size_t cols, cudaStream_t s, int dev) {
    nb::DevBuf tmp(sizeof(double2) * rows * cols, s);
    nb::transpose(d, tmp.as<double2>(), rows, cols, 1, s);
    nb::fft_exec(tmp.as<double2>(), tmp.as<double2>(), rows, cols, -1, s, dev);
    nb::fft_count(rows, cols);
    nb::transpose(tmp.as<double2>(), d, cols, rows, 1, s);
}

}  // namespace

namespace nb {
std::string& last_error() {
    thread_local std::string msg;
    return msg;
}
}  // namespace nb

extern "C" {

const char* nufft_last_error(void) { return nb::last_error().c_str(); }
int nufft_abi_version(void) { return NUFFT_B200_ABI_VERSION; }
int nufft_device_count(int* count) {
    return guard([&] {
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        *count = c;
    });
}

// ------------------------------------------------------------ special/lowrank
int nufft_lambert_w(double x, double* out) {
    return guard([&] { *out = nb::lambert_w(x); });
}
int nufft_bessel_j_int(int order, double z, double* out) {
    return guard([&] { *out = nb::bessel_j_int(order, z); });
}
int nufft_bessel_j_signed(int order, double z, double* out) {
    return guard([&] { *out = nb::bessel_j_signed(order, z); });
}
int nufft_select_rank(double gamma, double epsilon, size_t* rank) {
    return guard([&] { *rank = nb::select_rank(gamma, epsilon); });
}
int nufft_cheb_coefficients(double gamma, size_t K, double* a) {
    return guard([&] {
        auto v = nb::cheb_coefficients(gamma, K);
        std::memcpy(a, v.data(), 8 * v.size());
    });
}
int nufft_cheb_eval_matrix(const double* points, size_t n, size_t K, double* out) {
    return guard([&] {
        if (K < 1) nb::throw_invalid("cheb_eval_matrix: K must be >= 1");
        const int dev = pick_device(-1);
        (void)dev;
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf din(8 * n, s), dout(8 * n * K, s);
        if (n) NB_CUDA(cudaMemcpyAsync(din.get(), points, 8 * n, cudaMemcpyHostToDevice, s));
        nb::cheb_eval(din.as<double>(), n, K, dout.as<double>(), s);
        if (n) NB_CUDA(cudaMemcpyAsync(out, dout.get(), 8 * n * K, cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaStreamSynchronize(s));
    });
}
int nufft_build_factors(const double* delta, size_t n, double gamma, const double* omega_scaled,
                        size_t m, double epsilon, size_t* rank, double* u, double* v) {
    return guard([&] {
        if (gamma == 0.0) {  // lowrank.hpp:167-172
            *rank = 1;
            for (size_t j = 0; u && j < n; ++j) u[2 * j] = 1.0, u[2 * j + 1] = 0.0;
            for (size_t k = 0; v && k < m; ++k) v[2 * k] = 1.0, v[2 * k + 1] = 0.0;
            return;
        }
        const size_t K = nb::select_rank(gamma, epsilon);
        *rank = K;
        if (!u && !v) return;
        pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        if (u) {
            nb::DevBuf dd(8 * n, s), du(16 * n * K, s);
            if (n) NB_CUDA(cudaMemcpyAsync(dd.get(), delta, 8 * n, cudaMemcpyHostToDevice, s));
            if (n) nb::factors_u(dd.as<double>(), n, gamma, K, du.as<double2>(), s);
            else (void)nb::cheb_coefficients(gamma, K + nb::kCoefficientPadding);
            if (n) NB_CUDA(cudaMemcpyAsync(u, du.get(), 16 * n * K, cudaMemcpyDeviceToHost, s));
            NB_CUDA(cudaStreamSynchronize(s));
        }
        if (v) {
            nb::DevBuf dw(8 * m, s), dv(16 * m * K, s);
            if (m) NB_CUDA(cudaMemcpyAsync(dw.get(), omega_scaled, 8 * m, cudaMemcpyHostToDevice, s));
            if (m) nb::factors_v(dw.as<double>(), m, K, dv.as<double2>(), s);
            if (m) NB_CUDA(cudaMemcpyAsync(v, dv.get(), 16 * m * K, cudaMemcpyDeviceToHost, s));
            NB_CUDA(cudaStreamSynchronize(s));
        }
    });
}

// ------------------------------------------------------------ fft
int nufft_fft_forward_host(const double* in, double* out, size_t n) {
    return guard([&] {
        if (n == 0) nb::throw_invalid("fft_forward: empty input");
        const int dev = pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(in, 2 * n, out, 2 * n, s, [&](double2* a, double2* b) {
            nb::fft_exec(a, b, n, 1, -1, s, dev);
            nb::fft_count(n);
        });
    });
}
int nufft_fft_inverse_host(const double* in, double* out, size_t n) {
    return guard([&] {
        if (n == 0) nb::throw_invalid("fft_inverse: empty input");
        const int dev = pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(in, 2 * n, out, 2 * n, s, [&](double2* a, double2* b) {
            nb::fft_exec(a, b, n, 1, +1, s, dev);
            nb::fft_count(n);
            k_scale<<<blocks(n), 256, 0, s>>>(b, (long long)n, 1.0 / (double)n);
            NB_LAUNCH();
        });
    });
}
int nufft_fft_2d_forward_host(const double* in, double* out, size_t rows, size_t cols) {
    return guard([&] {
        if (rows * cols == 0) nb::throw_invalid("fft_2d_forward: empty input");
        const int dev = pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(in, 2 * rows * cols, out, 2 * rows * cols, s, [&](double2* a, double2* b) {
            NB_CUDA(cudaMemcpyAsync(b, a, 16 * rows * cols, cudaMemcpyDeviceToDevice, s));
            cols_fft(b, rows, cols, s, dev);
            rows_fft(b, rows, cols, s, dev);
        });
    });
}
int nufft_fft_cols_forward_host(double* inout, size_t rows, size_t cols) {
    return guard([&] {
        if (rows * cols == 0) return;
        const int dev = pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(inout, 2 * rows * cols, inout, 2 * rows * cols, s,
                       [&](double2* a, double2* b) {
                           NB_CUDA(cudaMemcpyAsync(b, a, 16 * rows * cols, cudaMemcpyDeviceToDevice, s));
                           cols_fft(b, rows, cols, s, dev);
                       });
    });
}
int nufft_fft_rows_forward_host(double* inout, size_t rows, size_t cols) {
    return guard([&] {
        if (rows * cols == 0) return;
        const int dev = pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(inout, 2 * rows * cols, inout, 2 * rows * cols, s,
                       [&](double2* a, double2* b) {
                           NB_CUDA(cudaMemcpyAsync(b, a, 16 * rows * cols, cudaMemcpyDeviceToDevice, s));
                           rows_fft(b, rows, cols, s, dev);
                       });
    });
}
int nufft_fft_exec(const double* in_dev, double* out_dev, size_t n, size_t batch, int sign,
                   void* stream) {
    return guard([&] {
        if (n == 0) nb::throw_invalid("fft: empty input");
        int dev;
        NB_CUDA(cudaGetDevice(&dev));
        nb::fft_exec(reinterpret_cast<const double2*>(in_dev), reinterpret_cast<double2*>(out_dev),
                     n, batch, sign < 0 ? -1 : +1, as_stream(stream), dev);
        nb::fft_count(n, batch);
    });
}
uint64_t nufft_fft_exec_count(size_t n) { return nb::fft_exec_count(n); }
uint64_t nufft_kernel_launch_count(void) { return nb::launch_count(); }
void nufft_fft_reset_exec_counts(void) { nb::fft_reset_exec_counts(); }

// ------------------------------------------------------------ samples
int nufft_normalize_samples(const double* raw, size_t n, double* out) {
    return guard([&] {
        pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        if (n == 0) return;
        nb::Axis ax;
        nb::assign_samples(ax, raw, false, n, 1, s);
        d2h(out, ax.x, n, s);
        NB_CUDA(cudaStreamSynchronize(s));
    });
}
int nufft_grid_assign(const double* x, size_t n, size_t grid, long* sv, size_t* t, double* gamma) {
    return guard([&] {
        if (grid < 1) nb::throw_invalid("grid_assign: grid size must be >= 1");
        pick_device(-1);
        cudaStream_t s = cudaStreamPerThread;
        if (n == 0) {
            *gamma = 0.0;
            return;
        }
        nb::Axis ax;
        nb::assign_samples(ax, x, false, n, grid, s);
        d2h(reinterpret_cast<long long*>(sv), ax.s, n, s);
        d2h(reinterpret_cast<long long*>(t), ax.t, n, s);
        NB_CUDA(cudaStreamSynchronize(s));
        *gamma = ax.gamma;
    });
}

// ------------------------------------------------------------ type II
static int plan2_create_impl(const double* x, bool on_dev, size_t n, double eps, int device,
                             nufft_plan2** out) {
    return guard([&] {
        if (n == 0) nb::throw_invalid("plan_nufft2: no samples");
        check_epsilon(eps);
        check_size(n);
        const int dev = pick_device(device);
        auto p = std::make_unique<nufft_plan2>();
        nb::CorePlan& c = p->core;
        c.device = dev;
        c.n = n;
        c.epsilon = eps;
        cudaStream_t s = cudaStreamPerThread;
        nb::assign_samples(c.ax, x, on_dev, n, n, s);
        nb::finish_core(c, c.ax.gamma, s);
        if (!c.fused) nb::build_bins(c, s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = p.release();
    });
}
int nufft_plan2_create(const double* x_raw, size_t n, double epsilon, int device, nufft_plan2** out) {
    return plan2_create_impl(x_raw, false, n, epsilon, device, out);
}
int nufft_plan2_create_device(const double* x_raw_dev, size_t n, double epsilon, int device,
                              nufft_plan2** out) {
    return plan2_create_impl(x_raw_dev, true, n, epsilon, device, out);
}
void nufft_plan2_destroy(nufft_plan2* plan) {
    if (!plan) return;
    DeviceRestore restore;
    const int dev = plan->core.device;
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    delete plan;
    nb::trim_scratch(dev);
}
int nufft_plan2_info(const nufft_plan2* plan, nufft_plan_info* info) {
    return guard([&] { fill_info(plan->core, info); });
}
int nufft_plan2_samples(const nufft_plan2* plan, double* x, long* s, size_t* t) {
    return guard([&] { core_samples(plan->core, x, s, t); });
}
int nufft_plan2_factors(const nufft_plan2* plan, double* u, double* v) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf d(16 * p.n * p.K, s);
        if (u) {
            materialize_u(p, d.as<double2>(), s);
            NB_CUDA(cudaMemcpyAsync(u, d.get(), 16 * p.n * p.K, cudaMemcpyDeviceToHost, s));
            NB_CUDA(cudaStreamSynchronize(s));
        }
        if (v) {
            materialize_v(p, d.as<double2>(), s);
            NB_CUDA(cudaMemcpyAsync(v, d.get(), 16 * p.n * p.K, cudaMemcpyDeviceToHost, s));
            NB_CUDA(cudaStreamSynchronize(s));
        }
    });
}
int nufft_plan2_exec_terms(const nufft_plan2* plan, const double* c_dev, double* f_dev,
                           size_t batch, size_t r_begin, size_t r_end, void* stream) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        if (r_end > p.K) r_end = p.K;
        nb::exec_type2(p, reinterpret_cast<const double2*>(c_dev), reinterpret_cast<double2*>(f_dev),
                       batch, r_begin, r_end, as_stream(stream));
        if (r_end > r_begin) nb::fft_count(p.n, (r_end - r_begin) * batch);
    });
}
int nufft_plan2_exec_timed(const nufft_plan2* plan, const double* c_dev, double* f_dev,
                           void* stream, int slot) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        if (!p.fused) nb::throw_invalid("exec_timed: plan does not use the fused two-pass path");
        if (slot < 0 || slot >= kMaxTimingSlots) nb::throw_invalid("exec_timed: slot out of range");
        cudaEvent_t* ev = nullptr;
        {
            std::lock_guard<std::mutex> lock(plan->timing_mu);
            while ((int)plan->timing.size() <= slot) {
                std::array<cudaEvent_t, 3> e{};
                for (auto& x : e) NB_CUDA(cudaEventCreate(&x));
                plan->timing.push_back(e);
            }
            ev = plan->timing[slot].data();
        }
        nb::exec_type2(p, reinterpret_cast<const double2*>(c_dev), reinterpret_cast<double2*>(f_dev),
                       1, 0, p.K, as_stream(stream), ev);
        nb::fft_count(p.n, p.K);
    });
}
int nufft_plan2_timing_read(const nufft_plan2* plan, int nslots, double* ms_pass1,
                            double* ms_pass2) {
    return guard([&] {
        std::lock_guard<std::mutex> lock(plan->timing_mu);
        if (nslots < 0 || nslots > (int)plan->timing.size()) nb::throw_invalid("timing_read: slot out of range");
        double a = 0, b = 0;
        for (int i = 0; i < nslots; ++i) {
            auto& e = plan->timing[i];
            NB_CUDA(cudaEventSynchronize(e[2]));
            float t1 = 0, t2 = 0;
            NB_CUDA(cudaEventElapsedTime(&t1, e[0], e[1]));
            NB_CUDA(cudaEventElapsedTime(&t2, e[1], e[2]));
            a += t1;
            b += t2;
        }
        *ms_pass1 = a;
        *ms_pass2 = b;
    });
}
int nufft_plan2_exec(const nufft_plan2* plan, const double* c_dev, double* f_dev, size_t batch,
                     void* stream) {
    return nufft_plan2_exec_terms(plan, c_dev, f_dev, batch, 0, plan->core.K, stream);
}
// batch > 1: the vectors stream through two device slots on three streams so the
// host->device copy of c_{b+1} and the device->host copy of f_{b-1} overlap the
// transform of vector b (the PCIe copies of one 2^24 vector take longer than its
// transform).  Results are identical to the one-shot path (same kernels per vector).
// Page-locked host buffers only: pageable batches go vector by vector through
// host_roundtrip, whose staged copies (host_stage.cu) pipeline the chunks of
// each vector instead.
namespace {
struct PipeStreams {  // streams + events, drained before anything they touch is freed
    cudaStream_t st[3] = {};
    cudaEvent_t ev[3][2] = {};
    cudaEvent_t ready = nullptr;
    PipeStreams() {
        for (auto& x : st) NB_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        for (auto& e : ev)
            for (auto& x : e) NB_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        NB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    }
    ~PipeStreams() {
        for (auto& x : st)
            if (x) cudaStreamSynchronize(x);
        for (auto& e : ev)
            for (auto& x : e)
                if (x) cudaEventDestroy(x);
        if (ready) cudaEventDestroy(ready);
        for (auto& x : st)
            if (x) cudaStreamDestroy(x);
    }
};
}  // namespace

static void plan2_host_pipelined(const nb::CorePlan& p, const double* c, double* f, size_t batch) {
    const size_t nd = 2 * p.n;  // doubles per vector
    cudaStream_t s0 = cudaStreamPerThread;
    // declared before the streams: on any exit the streams are drained first,
    // then the slots go back to the pool (stream-ordered on s0)
    nb::DevBuf din(8 * nd * 2, s0), dout(8 * nd * 2, s0);
    {
        PipeStreams ps;
        auto& st = ps.st;
        auto& ev = ps.ev;
        NB_CUDA(cudaEventRecord(ps.ready, s0));
        for (auto& x : st) NB_CUDA(cudaStreamWaitEvent(x, ps.ready, 0));
        enum { H2D = 0, COMP = 1, D2H = 2 };
        for (size_t b = 0; b < batch; ++b) {
            const int slot = (int)(b & 1);
            double* a = din.as<double>() + nd * slot;
            double* o = dout.as<double>() + nd * slot;
            if (b >= 2) NB_CUDA(cudaStreamWaitEvent(st[H2D], ev[COMP][slot], 0));  // din[slot] consumed
            NB_CUDA(cudaMemcpyAsync(a, c + nd * b, 8 * nd, cudaMemcpyHostToDevice, st[H2D]));
            NB_CUDA(cudaEventRecord(ev[H2D][slot], st[H2D]));
            NB_CUDA(cudaStreamWaitEvent(st[COMP], ev[H2D][slot], 0));
            if (b >= 2) NB_CUDA(cudaStreamWaitEvent(st[COMP], ev[D2H][slot], 0));  // dout[slot] drained
            nb::exec_type2(p, reinterpret_cast<const double2*>(a), reinterpret_cast<double2*>(o), 1, 0, p.K,
                           st[COMP]);
            NB_CUDA(cudaEventRecord(ev[COMP][slot], st[COMP]));
            NB_CUDA(cudaStreamWaitEvent(st[D2H], ev[COMP][slot], 0));
            NB_CUDA(cudaMemcpyAsync(f + nd * b, o, 8 * nd, cudaMemcpyDeviceToHost, st[D2H]));
            NB_CUDA(cudaEventRecord(ev[D2H][slot], st[D2H]));
        }
        for (auto& x : st) NB_CUDA(cudaStreamSynchronize(x));
    }
    nb::fft_count(p.n, p.K * batch);
}
int nufft_plan2_exec_host(const nufft_plan2* plan, const double* c, size_t len, double* f,
                          size_t batch) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("exec_nufft2: length mismatch");
        NB_CUDA(cudaSetDevice(p.device));
        if (batch > 1 && !nb::host_pageable(c) && !nb::host_pageable(f)) {
            plan2_host_pipelined(p, c, f, batch);
            return;
        }
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(c, 2 * p.n * batch, f, 2 * p.n * batch, s, [&](double2* a, double2* b) {
            nb::exec_type2(p, a, b, batch, 0, p.K, s);
            nb::fft_count(p.n, p.K * batch);
        });
    });
}
static void adjoint_dev(const nb::CorePlan& p, const double2* fin, double2* out, cudaStream_t s) {
    if (p.fused) {  // conj(F2~^T conj(f)) with the conjugations folded into the transpose core
        nb::exec_transpose_fused(p, fin, out, 1, s, nullptr, 0, p.K, /*conj=*/true);
    } else {
        nb::DevBuf g(16 * p.n, s);
        nb::conj_copy(fin, g.as<double2>(), p.n, s);
        nb::exec_transpose(p, g.as<double2>(), out, 1, s);
        nb::conj_copy(out, out, p.n, s);
    }
    nb::fft_count(p.n, p.K);
}
int nufft_plan2_adjoint(const nufft_plan2* plan, const double* f_dev, double* out_dev, void* stream) {
    return guard([&] {
        NB_CUDA(cudaSetDevice(plan->core.device));
        adjoint_dev(plan->core, reinterpret_cast<const double2*>(f_dev),
                    reinterpret_cast<double2*>(out_dev), as_stream(stream));
    });
}
int nufft_plan2_adjoint_host(const nufft_plan2* plan, const double* f, size_t len, double* out) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("nufft transpose: length mismatch");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(f, 2 * p.n, out, 2 * p.n, s,
                       [&](double2* a, double2* b) { adjoint_dev(p, a, b, s); });
    });
}

// ------------------------------------------------------------ type I
int nufft_plan1_create(const double* omega, size_t n, double epsilon, int device, nufft_plan1** out) {
    return guard([&] {
        if (n == 0) nb::throw_invalid("plan_nufft1: no frequencies");
        check_epsilon(epsilon);
        check_size(n);
        const int dev = pick_device(device);
        auto p = std::make_unique<nufft_plan1>();
        nb::CorePlan& c = p->core;
        c.device = dev;
        c.n = n;
        c.epsilon = epsilon;
        cudaStream_t s = cudaStreamPerThread;
        nb::assign_frequencies(c.ax, omega, false, n, false, s);
        c.delta_from_freq = true;
        nb::finish_core(c, c.ax.gamma_raw, s);  // un-snapped gamma, transforms.hpp:282
        if (!c.fused) nb::build_bins(c, s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = p.release();
    });
}
void nufft_plan1_destroy(nufft_plan1* plan) {
    if (!plan) return;
    DeviceRestore restore;
    const int dev = plan->core.device;
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    delete plan;
    nb::trim_scratch(dev);
}
int nufft_plan1_info(const nufft_plan1* plan, nufft_plan_info* info) {
    return guard([&] { fill_info(plan->core, info); });
}
int nufft_plan1_samples(const nufft_plan1* plan, double* x, long* s, size_t* t) {
    return guard([&] { core_samples(plan->core, x, s, t); });
}
int nufft_plan1_exec(const nufft_plan1* plan, const double* c_dev, double* f_dev, size_t batch,
                     void* stream) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        nb::exec_transpose(p, reinterpret_cast<const double2*>(c_dev), reinterpret_cast<double2*>(f_dev),
                           batch, as_stream(stream));
        nb::fft_count(p.n, p.K * batch);
    });
}
int nufft_plan1_exec_host(const nufft_plan1* plan, const double* c, size_t len, double* f,
                          size_t batch) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("nufft transpose: length mismatch");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(c, 2 * p.n * batch, f, 2 * p.n * batch, s, [&](double2* a, double2* b) {
            nb::exec_transpose(p, a, b, batch, s);
            nb::fft_count(p.n, p.K * batch);
        });
    });
}

// ------------------------------------------------------------ type III
static void type1_adjoint_dev(const nb::CorePlan& p, const double2* gin, double2* out, cudaStream_t s) {
    nb::DevBuf g(16 * p.n, s);
    nb::conj_copy(gin, g.as<double2>(), p.n, s);
    nb::exec_type2(p, g.as<double2>(), out, 1, 0, p.K, s);
    nb::conj_copy(out, out, p.n, s);
    nb::fft_count(p.n, p.K);
}
int nufft_plan1_adjoint(const nufft_plan1* plan, const double* g_dev, double* out_dev, void* stream) {
    return guard([&] {
        NB_CUDA(cudaSetDevice(plan->core.device));
        type1_adjoint_dev(plan->core, reinterpret_cast<const double2*>(g_dev), reinterpret_cast<double2*>(out_dev),
                          as_stream(stream));
    });
}
int nufft_plan1_adjoint_host(const nufft_plan1* plan, const double* g, size_t len, double* out) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("nufft transpose: length mismatch");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(g, 2 * p.n, out, 2 * p.n, s, [&](double2* a, double2* b) { type1_adjoint_dev(p, a, b, s); });
    });
}

// ------------------------------------------------------------ inverse
static std::unique_ptr<nufft_toeplitz> toeplitz_make(int device, size_t n) {
    auto op = std::make_unique<nufft_toeplitz>();
    op->st.device = device;
    op->st.n = n;
    return op;
}
int nufft_toeplitz_from_first_column(const double* column, size_t n, int device, nufft_toeplitz** out) {
    return guard([&] {
        if (n == 0) nb::throw_invalid("toeplitz: empty first column");
        const int dev = pick_device(device);
        auto op = toeplitz_make(dev, n);
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf col(16 * n, s);
        NB_CUDA(cudaMemcpyAsync(col.get(), column, 16 * n, cudaMemcpyHostToDevice, s));
        nb::toeplitz_from_column(op->st, col.as<double2>(), s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = op.release();
    });
}
int nufft_toeplitz_from_normal(const nufft_plan2* plan, nufft_toeplitz** out) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        auto op = toeplitz_make(p.device, p.n);
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf e0(16 * p.n, s), f(16 * p.n, s), col(16 * p.n, s);
        NB_CUDA(cudaMemsetAsync(e0.get(), 0, 16 * p.n, s));
        const double one = 1.0;
        NB_CUDA(cudaMemcpyAsync(e0.get(), &one, sizeof(double), cudaMemcpyHostToDevice, s));
        nb::exec_type2(p, e0.as<double2>(), f.as<double2>(), 1, 0, p.K, s);  // F2~ e_0
        nb::fft_count(p.n, p.K);
        adjoint_dev(p, f.as<double2>(), col.as<double2>(), s);               // F2~* F2~ e_0
        nb::toeplitz_from_column(op->st, col.as<double2>(), s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = op.release();
    });
}
int nufft_toeplitz_from_gram(const nufft_plan1* plan, nufft_toeplitz** out) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        auto op = toeplitz_make(p.device, p.n);
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf e0(16 * p.n, s), g(16 * p.n, s), col(16 * p.n, s);
        NB_CUDA(cudaMemsetAsync(e0.get(), 0, 16 * p.n, s));
        const double one = 1.0;
        NB_CUDA(cudaMemcpyAsync(e0.get(), &one, sizeof(double), cudaMemcpyHostToDevice, s));
        type1_adjoint_dev(p, e0.as<double2>(), g.as<double2>(), s);    // F1~* e_0
        nb::exec_transpose(p, g.as<double2>(), col.as<double2>(), 1, s);  // F1~ F1~* e_0
        nb::fft_count(p.n, p.K);
        nb::toeplitz_from_column(op->st, col.as<double2>(), s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = op.release();
    });
}
void nufft_toeplitz_destroy(nufft_toeplitz* op) {
    if (!op) return;
    DeviceRestore restore;
    const int dev = op->st.device;
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    delete op;
    nb::trim_scratch(dev);
}
int nufft_toeplitz_size(const nufft_toeplitz* op, size_t* n) {
    return guard([&] { *n = op->st.n; });
}
int nufft_toeplitz_members(const nufft_toeplitz* op, double* spectrum, double* first_column) {
    return guard([&] {
        const nb::ToeplitzState& t = op->st;
        NB_CUDA(cudaSetDevice(t.device));
        cudaStream_t s = cudaStreamPerThread;
        if (spectrum) {
            std::vector<double> re(2 * t.n);
            d2h(re.data(), t.spectrum, 2 * t.n, s);
            NB_CUDA(cudaStreamSynchronize(s));
            for (size_t j = 0; j < 2 * t.n; ++j) {
                spectrum[2 * j] = re[j];
                spectrum[2 * j + 1] = 0.0;
            }
        }
        if (first_column) {
            NB_CUDA(cudaMemcpyAsync(first_column, t.first_col.as<double2>(), 16 * t.n, cudaMemcpyDeviceToHost, s));
            NB_CUDA(cudaStreamSynchronize(s));
        }
    });
}
int nufft_toeplitz_matvec(const nufft_toeplitz* op, const double* v_dev, double* out_dev, void* stream) {
    return guard([&] {
        NB_CUDA(cudaSetDevice(op->st.device));
        nb::toeplitz_matvec(op->st, reinterpret_cast<const double2*>(v_dev), reinterpret_cast<double2*>(out_dev),
                            as_stream(stream));
    });
}
int nufft_toeplitz_matvec_host(const nufft_toeplitz* op, const double* v, size_t len, double* out) {
    return guard([&] {
        const nb::ToeplitzState& t = op->st;
        if (len != t.n) nb::throw_invalid("toeplitz_matvec: length mismatch");
        NB_CUDA(cudaSetDevice(t.device));
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(v, 2 * t.n, out, 2 * t.n, s, [&](double2* a, double2* b) { nb::toeplitz_matvec(t, a, b, s); });
    });
}
static void fill_report(const nb::CgResult& r, const std::vector<double>& hist, nufft_cg_report* rep,
                        double* history, size_t cap) {
    if (rep) {
        rep->iterations = r.iterations;
        rep->relative_residual = r.relative_residual;
        rep->converged = r.converged ? 1 : 0;
        rep->history_len = std::min(cap, hist.size());
    }
    if (history)
        for (size_t i = 0; i < hist.size() && i < cap; ++i) history[i] = hist[i];
}
int nufft_cg_toeplitz_host(const nufft_toeplitz* op, const double* rhs, size_t len, double tol, size_t max_iter,
                           double* solution, nufft_cg_report* report, double* history, size_t history_cap) {
    return guard([&] {
        if (!(tol > 0.0)) nb::throw_domain("cg_solve: tol must be positive");
        const nb::ToeplitzState& t = op->st;
        if (len != t.n) nb::throw_invalid("toeplitz_matvec: length mismatch");
        NB_CUDA(cudaSetDevice(t.device));
        cudaStream_t s = cudaStreamPerThread;
        std::vector<double> hist;
        nb::CgResult r;
        host_roundtrip(rhs, 2 * t.n, solution, 2 * t.n, s, [&](double2* a, double2* b) {
            r = nb::cg_solve_toeplitz(t, a, b, tol, max_iter, &hist, s);
        });
        fill_report(r, hist, report, history, history_cap);
    });
}
static nb::CgResult inufft2_dev(const nufft_plan2* plan, const nufft_toeplitz* op, const double2* f, double tol,
                                double2* sol, std::vector<double>* hist, cudaStream_t s) {
    const nb::CorePlan& p = plan->core;
    if (!(p.ax.gamma < 0.5)) nb::throw_domain("inufft2: gamma >= 1/2, samples may not be distinct");
    if (!(tol > 0.0)) nb::throw_domain("cg_solve: tol must be positive");
    std::unique_ptr<nufft_toeplitz> own;
    if (!op) {
        nufft_toeplitz* raw = nullptr;
        if (nufft_toeplitz_from_normal(plan, &raw) != NUFFT_OK) throw nb::Error(nb::kInternal, nb::last_error());
        own.reset(raw);
        op = raw;
    }
    nb::DevBuf rhs(16 * p.n, s);
    adjoint_dev(p, f, rhs.as<double2>(), s);
    return nb::cg_solve_toeplitz(op->st, rhs.as<double2>(), sol, tol, nb::default_cg_max_iter(p.n), hist, s);
}
int nufft_inufft2_host(const nufft_plan2* plan, const nufft_toeplitz* op, const double* f, size_t len, double tol,
                       double* solution, nufft_cg_report* report, double* history, size_t history_cap) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("inufft2: length mismatch");
        if (!(p.ax.gamma < 0.5)) nb::throw_domain("inufft2: gamma >= 1/2, samples may not be distinct");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = cudaStreamPerThread;
        std::vector<double> hist;
        nb::CgResult r;
        host_roundtrip(f, 2 * p.n, solution, 2 * p.n, s,
                       [&](double2* a, double2* b) { r = inufft2_dev(plan, op, a, tol, b, &hist, s); });
        fill_report(r, hist, report, history, history_cap);
    });
}
int nufft_inufft2(const nufft_plan2* plan, const nufft_toeplitz* op, const double* f_dev, double tol,
                  double* solution_dev, nufft_cg_report* report, void* stream) {
    return guard([&] {
        NB_CUDA(cudaSetDevice(plan->core.device));
        const nb::CgResult r = inufft2_dev(plan, op, reinterpret_cast<const double2*>(f_dev), tol,
                                           reinterpret_cast<double2*>(solution_dev), nullptr, as_stream(stream));
        fill_report(r, {}, report, nullptr, 0);
    });
}
int nufft_inufft1_host(const nufft_plan1* plan, const nufft_toeplitz* op, const double* f, size_t len, double tol,
                       double* solution, nufft_cg_report* report, double* history, size_t history_cap) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("inufft1: length mismatch");
        if (!(p.ax.gamma < 0.5)) nb::throw_domain("inufft1: gamma >= 1/2, frequencies may not be distinct");
        if (!(tol > 0.0)) nb::throw_domain("cg_solve: tol must be positive");
        NB_CUDA(cudaSetDevice(p.device));
        std::unique_ptr<nufft_toeplitz> own;
        if (!op) {
            nufft_toeplitz* raw = nullptr;
            if (nufft_toeplitz_from_gram(plan, &raw) != NUFFT_OK) throw nb::Error(nb::kInternal, nb::last_error());
            own.reset(raw);
            op = raw;
        }
        cudaStream_t s = cudaStreamPerThread;
        std::vector<double> hist;
        nb::CgResult r;
        host_roundtrip(f, 2 * p.n, solution, 2 * p.n, s, [&](double2* a, double2* b) {
            nb::DevBuf y(16 * p.n, s);
            r = nb::cg_solve_toeplitz(op->st, a, y.as<double2>(), tol, nb::default_cg_max_iter(p.n), &hist, s);
            type1_adjoint_dev(p, y.as<double2>(), b, s);  // c = F1~* y
        });
        fill_report(r, hist, report, history, history_cap);
    });
}
size_t nufft_default_cg_max_iter(size_t n) { return nb::default_cg_max_iter(n); }

// ------------------------------------------------------------ direct sums
int nufft_nudft_direct_host(const double* x, size_t nx, const double* omega, const double* c, size_t n, double* f,
                            int device) {
    return guard([&] {
        pick_device(device);
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf dx(8 * std::max<size_t>(nx, 1), s), dw(8 * std::max<size_t>(n, 1), s),
            dc(16 * std::max<size_t>(n, 1), s), df(16 * std::max<size_t>(nx, 1), s);
        NB_CUDA(cudaMemcpyAsync(dx.get(), x, 8 * nx, cudaMemcpyHostToDevice, s));
        NB_CUDA(cudaMemcpyAsync(dw.get(), omega, 8 * n, cudaMemcpyHostToDevice, s));
        NB_CUDA(cudaMemcpyAsync(dc.get(), c, 16 * n, cudaMemcpyHostToDevice, s));
        nb::nudft_direct(dx.as<double>(), nx, dw.as<double>(), dc.as<double2>(), n, df.as<double2>(), s);
        NB_CUDA(cudaMemcpyAsync(f, df.get(), 16 * nx, cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaStreamSynchronize(s));
    });
}
int nufft_nudft_direct(const double* x_dev, size_t nx, const double* omega_dev, const double* c_dev, size_t n,
                       double* f_dev, void* stream) {
    return guard([&] {
        nb::nudft_direct(x_dev, nx, omega_dev, reinterpret_cast<const double2*>(c_dev), n,
                         reinterpret_cast<double2*>(f_dev), as_stream(stream));
    });
}
int nufft_nudft2d_direct_host(const double* x, const double* y, size_t count, const double* C, size_t m, size_t n,
                              double* f, int device) {
    return guard([&] {
        if (m * n == 0) nb::throw_invalid("nudft2d_direct: inconsistent matrix dimensions");
        pick_device(device);
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf dx(8 * std::max<size_t>(count, 1), s), dy(8 * std::max<size_t>(count, 1), s),
            dC(16 * m * n, s), df(16 * std::max<size_t>(count, 1), s);
        NB_CUDA(cudaMemcpyAsync(dx.get(), x, 8 * count, cudaMemcpyHostToDevice, s));
        NB_CUDA(cudaMemcpyAsync(dy.get(), y, 8 * count, cudaMemcpyHostToDevice, s));
        NB_CUDA(cudaMemcpyAsync(dC.get(), C, 16 * m * n, cudaMemcpyHostToDevice, s));
        nb::nudft2d_direct(dx.as<double>(), dy.as<double>(), count, dC.as<double2>(), m, n, df.as<double2>(), s);
        NB_CUDA(cudaMemcpyAsync(f, df.get(), 16 * count, cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaStreamSynchronize(s));
    });
}

int nufft_plan3_create(const double* x_raw, const double* omega, size_t n_x, size_t n_omega,
                       double epsilon, int device, nufft_plan3** out) {
    return guard([&] {
        if (n_x != n_omega) nb::throw_invalid("plan_nufft3: sample/frequency length mismatch");
        if (n_x == 0) nb::throw_invalid("plan_nufft3: no samples");
        check_epsilon(epsilon);
        check_size(n_x);
        const size_t n = n_x;
        const int dev = pick_device(device);
        auto p = std::make_unique<nufft_plan3>();
        nb::Plan3State& st = p->st;
        cudaStream_t s = cudaStreamPerThread;
        // frequencies first (transforms.hpp:329-331 validates them before the samples)
        st.inner.device = dev;
        st.inner.n = n;
        st.inner.epsilon = epsilon;
        nb::assign_frequencies(st.inner.ax, omega, false, n, true, s);
        st.inner.delta_from_freq = true;
        st.a.device = dev;
        st.a.n = n;
        st.a.epsilon = epsilon;
        nb::assign_samples(st.a.ax, x_raw, false, n, n, s);
        st.omega.alloc(8 * n);
        NB_CUDA(cudaMemcpyAsync(st.omega.as<double>(), omega, 8 * n, cudaMemcpyHostToDevice, s));
        // factors A: gamma = samples.gamma (snapped), v over omega/N (transforms.hpp:337-340)
        st.a.gamma_factors = st.a.ax.gamma;
        st.a.uniform = st.a.gamma_factors == 0.0;
        st.a.K = st.a.uniform ? 1 : nb::select_rank(st.a.gamma_factors, epsilon);
        st.a.series_deg = nb::bessel_series_degrees(st.a.gamma_factors, st.a.K);
        nb::DevBuf flag(4, s);
        NB_CUDA(cudaMemsetAsync(flag.get(), 0, 4, s));
        k_any_wrap<<<blocks(n), 256, 0, s>>>(st.a.ax.s.as<long long>(), st.a.ax.t.as<long long>(),
                                             (long long)n, flag.as<int>());
        NB_LAUNCH();
        int wrap = 0;
        NB_CUDA(cudaMemcpyAsync(&wrap, flag.get(), 4, cudaMemcpyDeviceToHost, s));
        NB_CUDA(cudaStreamSynchronize(s));
        st.btrivial = wrap == 0;
        st.kc = st.btrivial ? st.a.K : 2 * st.a.K;
        nb::build_type3_order(st, s);
        // inner type-I plan on omega (transforms.hpp:378)
        nb::finish_core(st.inner, st.inner.ax.gamma_raw, s);
        if (!st.inner.fused) nb::build_bins(st.inner, s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = p.release();
    });
}
void nufft_plan3_destroy(nufft_plan3* plan) {
    if (!plan) return;
    DeviceRestore restore;
    const int dev = plan->st.a.device;
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    delete plan;
    nb::trim_scratch(dev);
}
int nufft_plan3_info(const nufft_plan3* plan, nufft_plan_info* info) {
    return guard([&] {
        const nb::Plan3State& st = plan->st;
        fill_info(st.a, info);
        info->rank = st.a.K;
        info->rank2 = st.inner.K;
        info->effective_rank = st.kc;
        info->gamma = st.a.ax.gamma;
        info->gamma2 = st.inner.ax.gamma;
        info->btrivial = st.btrivial ? 1 : 0;
        info->path = 0;
    });
}
int nufft_plan3_samples(const nufft_plan3* plan, double* x, long* s, size_t* t) {
    return guard([&] { core_samples(plan->st.a, x, s, t); });
}
int nufft_plan3_exec(const nufft_plan3* plan, const double* c_dev, double* f_dev, size_t batch,
                     void* stream) {
    return guard([&] {
        const nb::Plan3State& st = plan->st;
        NB_CUDA(cudaSetDevice(st.a.device));
        nb::exec_type3(st, reinterpret_cast<const double2*>(c_dev), reinterpret_cast<double2*>(f_dev),
                       batch, as_stream(stream));
        nb::fft_count(st.a.n, st.a.K * st.inner.K * batch);  // the beta family needs no FFTs (exec_type3)
    });
}
int nufft_plan3_exec_host(const nufft_plan3* plan, const double* c, size_t len, double* f,
                          size_t batch) {
    return guard([&] {
        const nb::Plan3State& st = plan->st;
        if (len != st.a.n) nb::throw_invalid("exec_nufft3: length mismatch");
        NB_CUDA(cudaSetDevice(st.a.device));
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(c, 2 * st.a.n * batch, f, 2 * st.a.n * batch, s, [&](double2* a, double2* b) {
            nb::exec_type3(st, a, b, batch, s);
            nb::fft_count(st.a.n, st.a.K * st.inner.K * batch);  // the beta family needs no FFTs (exec_type3)
        });
    });
}

// ------------------------------------------------------------ 2D type II
int nufft_plan2d2_create(const double* x_raw, const double* y_raw, size_t count_x, size_t count_y,
                         size_t m, size_t n, double epsilon, int device, nufft_plan2d** out) {
    return guard([&] {
        if (count_x == 0) nb::throw_invalid("plan_nufft2d2: no samples");
        if (m < 1 || n < 1) nb::throw_invalid("plan_nufft2d2: grid sizes must be >= 1");
        check_epsilon(epsilon);
        check_size(count_x);
        const int dev = pick_device(device);
        auto p = std::make_unique<nufft_plan2d>();
        nb::Plan2DState& st = p->st;
        st.device = dev;
        st.m = m;
        st.n = n;
        st.epsilon = epsilon;
        cudaStream_t s = cudaStreamPerThread;
        nb::assign_samples(st.ax, x_raw, false, count_x, n, s);
        if (count_y) nb::assign_samples(st.ay, y_raw, false, count_y, m, s);
        if (count_x != count_y) nb::throw_invalid("grid_assign_2d: coordinate length mismatch");
        st.count = count_x;
        st.ux_uniform = st.ax.gamma == 0.0;
        st.uy_uniform = st.ay.gamma == 0.0;
        st.kx = st.ux_uniform ? 1 : nb::select_rank(st.ax.gamma, epsilon);
        st.ky = st.uy_uniform ? 1 : nb::select_rank(st.ay.gamma, epsilon);
        st.deg_x = nb::bessel_series_degrees(st.ax.gamma, st.kx);
        st.deg_y = nb::bessel_series_degrees(st.ay.gamma, st.ky);
        st.flat.alloc(8 * st.count);
        k_flat_index<<<blocks(st.count), 256, 0, s>>>(st.ax.t.as<long long>(), st.ay.t.as<long long>(),
                                                      (long long)st.count, (long long)m,
                                                      st.flat.as<long long>());
        NB_LAUNCH();
        if (nb::fused_2d_eligible(m, n, st.count)) nb::build_2d_fused(st, s);
        NB_CUDA(cudaStreamSynchronize(s));
        *out = p.release();
    });
}
void nufft_plan2d2_destroy(nufft_plan2d* plan) {
    if (!plan) return;
    DeviceRestore restore;
    const int dev = plan->st.device;
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    delete plan;
    nb::trim_scratch(dev);
}
int nufft_plan2d2_info(const nufft_plan2d* plan, nufft_plan_info* info) {
    return guard([&] {
        const nb::Plan2DState& st = plan->st;
        std::memset(info, 0, sizeof(*info));
        info->n = st.count;
        info->rank = st.kx;
        info->rank2 = st.ky;
        info->effective_rank = st.kx * st.ky;
        info->gamma = st.ax.gamma;
        info->gamma2 = st.ay.gamma;
        info->epsilon = st.epsilon;
        info->btrivial = 1;
        info->m = st.m;
        info->ncols = st.n;
        info->device = st.device;
        info->path = st.fused ? 1 : 0;
    });
}
int nufft_plan2d2_samples(const nufft_plan2d* plan, double* x, double* y, long* sx, long* sy,
                          size_t* tx, size_t* ty, size_t* flat_index) {
    return guard([&] {
        const nb::Plan2DState& st = plan->st;
        NB_CUDA(cudaSetDevice(st.device));
        cudaStream_t s = cudaStreamPerThread;
        const size_t c = st.count;
        if (x) d2h(x, st.ax.x, c, s);
        if (y) d2h(y, st.ay.x, c, s);
        if (sx) d2h(reinterpret_cast<long long*>(sx), st.ax.s, c, s);
        if (sy) d2h(reinterpret_cast<long long*>(sy), st.ay.s, c, s);
        if (tx) d2h(reinterpret_cast<long long*>(tx), st.ax.t, c, s);
        if (ty) d2h(reinterpret_cast<long long*>(ty), st.ay.t, c, s);
        if (flat_index) d2h(reinterpret_cast<long long*>(flat_index), st.flat, c, s);
        NB_CUDA(cudaStreamSynchronize(s));
    });
}
int nufft_plan2d2_exec(const nufft_plan2d* plan, const double* C_dev, double* f_dev, size_t batch,
                       void* stream) {
    return guard([&] {
        const nb::Plan2DState& st = plan->st;
        NB_CUDA(cudaSetDevice(st.device));
        nb::exec_2d(st, reinterpret_cast<const double2*>(C_dev), reinterpret_cast<double2*>(f_dev),
                    batch, true, as_stream(stream));
    });
}
int nufft_plan2d2_exec_host_impl(const nufft_plan2d* plan, const double* C, size_t rows,
                                 size_t cols, double* f, size_t batch, int reuse_row_stage) {
    return guard([&] {
        const nb::Plan2DState& st = plan->st;
        if (rows != st.m || cols != st.n)
            nb::throw_invalid("exec_nufft2d2: coefficient dimensions mismatch");
        NB_CUDA(cudaSetDevice(st.device));
        cudaStream_t s = cudaStreamPerThread;
        host_roundtrip(C, 2 * st.m * st.n * batch, f, 2 * st.count * batch, s,
                       [&](double2* a, double2* b) { nb::exec_2d(st, a, b, batch, reuse_row_stage != 0, s); });
    });
}
int nufft_plan2d2_exec_host(const nufft_plan2d* plan, const double* C, size_t rows, size_t cols,
                            double* f, size_t batch) {
    return nufft_plan2d2_exec_host_impl(plan, C, rows, cols, f, batch, 1);
}

}  // extern "C"
