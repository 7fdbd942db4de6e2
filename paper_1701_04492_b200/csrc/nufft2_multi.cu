// Multi-GPU type-II execution: the rank-K sum split across GPUs.
//
// Reference: with threads > 1, exec_nufft2 (proj/include/nufft/transforms.hpp:
// 174-197) hands contiguous r-ranges to worker threads, each accumulating a
// partial f over its terms, and merges the partials in a fixed order.  Here a
// "worker" is a GPU (one process per GPU, an NCCL communicator between them):
//
//   rank g of G evaluates terms [K g / G, K (g+1) / G) — pass 1 once, then
//   pass 2 in row chunks that write the partial sum in BUCKET order
//   (fs[i] for sorted sample i, coalesced; no scattered f[perm] stores) —
//   and each chunk's sample range [rowoff[row0], rowoff[row1]) is reduced
//   (fp64 sum, ncclReduce or ncclAllReduce) on a communication stream while
//   the next chunk is computed.  The receiving rank(s) then un-permute once,
//   f[perm[i]] = fs[i].
//
// So the 256 MiB reduce of one vector overlaps all but the last chunk of pass
// 2, and the scattered f write happens once (at the root) instead of on
// every rank.  NCCL is resolved at run time (dlopen of libnccl.so.2, reusing
// the copy PyTorch already loaded when there is one), so single-GPU users of
// the library need no NCCL at all.  Plans without the fused two-pass path
// (N not a power of two, or N < 256) reduce the whole natural-order partial.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "../../include/nufft_b200.h"
#include "handles.hpp"
#include "plans.hpp"

namespace nb {
namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclReduce) reduce = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclCommCount) count = nullptr;
    decltype(&ncclCommUserRank) user_rank = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // PyTorch's copy, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.error = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
        api.init_rank = reinterpret_cast<decltype(api.init_rank)>(sym("ncclCommInitRank"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(sym("ncclCommDestroy"));
        api.reduce = reinterpret_cast<decltype(api.reduce)>(sym("ncclReduce"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
        api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
        api.count = reinterpret_cast<decltype(api.count)>(sym("ncclCommCount"));
        api.user_rank = reinterpret_cast<decltype(api.user_rank)>(sym("ncclCommUserRank"));
    });
    if (!api.error.empty()) throw Error(kNcclError, api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    throw Error(kNcclError, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

// [r_begin, r_end) of rank g of G over K terms: contiguous, balanced, ordered
// by rank (transforms.hpp:181-192 splits the K terms among workers the same way)
void term_range(size_t K, int G, int g, size_t* r0, size_t* r1) {
    *r0 = K * (size_t)g / (size_t)G;
    *r1 = K * (size_t)(g + 1) / (size_t)G;
}

}  // namespace nb

struct nufft_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    bool owned = true;
    cudaStream_t cs = nullptr;  // communication stream (reduces + un-permute)
    ~nufft_comm() {
        if (cs) {
            cudaSetDevice(device);
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
        }
        if (owned && comm) nb::nccl().destroy(comm);
    }
};

namespace {

using nb::guard;

constexpr int kReduceChunks = 4;  // pass-2 row chunks per vector (reduce of chunk q overlaps chunk q + 1)

// One vector: partial over this rank's terms into fs (bucket order), reduced
// chunk by chunk on comm->cs; returns after enqueueing (stream-ordered).
void exec_multi_one(const nb::CorePlan& p, const double2* c, double2* f, double2* fs, double2* Y,
                    nufft_comm* cm, int root, int mode, cudaStream_t s, cudaEvent_t* chunk_ev) {
    const nb::NcclApi& api = nb::nccl();
    size_t r0, r1;
    nb::term_range(p.K, cm->nranks, cm->rank, &r0, &r1);
    const bool all = mode == NUFFT_MULTI_ALLREDUCE;
    const bool receives = all || cm->rank == root;
    if (!p.fused || p.bk.log_n1 == 0) {  // natural-order partial, one reduce
        nb::exec_type2(p, c, fs, 1, r0, r1, s);
        NB_CUDA(cudaEventRecord(chunk_ev[0], s));
        NB_CUDA(cudaStreamWaitEvent(cm->cs, chunk_ev[0], 0));
        if (all)
            nb::nccl_check(api.all_reduce(fs, f, 2 * p.n, ncclDouble, ncclSum, cm->comm, cm->cs), "ncclAllReduce");
        else
            nb::nccl_check(api.reduce(fs, f, 2 * p.n, ncclDouble, ncclSum, root, cm->comm, cm->cs), "ncclReduce");
        return;
    }
    const long long n1 = 1ll << p.bk.log_n1;
    const int nch = (int)std::min<long long>(kReduceChunks, n1);
    if (r1 > r0) nb::exec_type2_pass1(p, c, Y, r0, r1, s);
    for (int q = 0; q < nch; ++q) {
        const long long row0 = n1 * q / nch, row1 = n1 * (q + 1) / nch;
        const size_t i0 = (size_t)p.bk.rowoff_host[row0], i1 = (size_t)p.bk.rowoff_host[row1];
        if (r1 > r0) {
            nb::exec_type2_pass2_rows(p, Y, fs, r0, r1, row0, row1, /*sorted_out=*/true, s);
        } else if (i1 > i0) {  // more ranks than terms: this rank contributes zeros
            NB_CUDA(cudaMemsetAsync(fs + i0, 0, sizeof(double2) * (i1 - i0), s));
        }
        NB_CUDA(cudaEventRecord(chunk_ev[q], s));
        NB_CUDA(cudaStreamWaitEvent(cm->cs, chunk_ev[q], 0));
        if (i1 == i0) continue;
        if (all)
            nb::nccl_check(api.all_reduce(fs + i0, fs + i0, 2 * (i1 - i0), ncclDouble, ncclSum, cm->comm, cm->cs),
                           "ncclAllReduce");
        else
            nb::nccl_check(api.reduce(fs + i0, fs + i0, 2 * (i1 - i0), ncclDouble, ncclSum, root, cm->comm, cm->cs),
                           "ncclReduce");
    }
    if (receives) nb::unpermute(p, fs, f, 1, cm->cs);
}

}  // namespace

extern "C" {

int nufft_comm_unique_id(unsigned char* id) {
    return guard([&] {
        if (!id) nb::throw_invalid("comm_unique_id: null buffer");
        static_assert(sizeof(ncclUniqueId) == NUFFT_UNIQUE_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        nb::nccl_check(nb::nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int nufft_comm_init(const unsigned char* id, int nranks, int rank, int device, nufft_comm** out) {
    return guard([&] {
        if (!id || !out) nb::throw_invalid("comm_init: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) nb::throw_invalid("comm_init: rank out of range");
        NB_CUDA(cudaSetDevice(device));
        nb::DeviceCtx::get(device);
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        auto c = std::make_unique<nufft_comm>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        nb::nccl_check(nb::nccl().init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        NB_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
        *out = c.release();
    });
}

int nufft_comm_wrap(void* nccl_comm, int device, nufft_comm** out) {
    return guard([&] {
        if (!nccl_comm || !out) nb::throw_invalid("comm_wrap: null argument");
        NB_CUDA(cudaSetDevice(device));
        nb::DeviceCtx::get(device);
        auto c = std::make_unique<nufft_comm>();
        c->comm = static_cast<ncclComm_t>(nccl_comm);
        c->owned = false;
        c->device = device;
        nb::nccl_check(nb::nccl().count(c->comm, &c->nranks), "ncclCommCount");
        nb::nccl_check(nb::nccl().user_rank(c->comm, &c->rank), "ncclCommUserRank");
        NB_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
        *out = c.release();
    });
}

void nufft_comm_destroy(nufft_comm* comm) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = -1;
    }
    delete comm;
    if (dev >= 0) cudaSetDevice(dev);
}

int nufft_comm_info(const nufft_comm* comm, int* nranks, int* rank, int* device) {
    return guard([&] {
        if (!comm) nb::throw_invalid("comm_info: null communicator");
        if (nranks) *nranks = comm->nranks;
        if (rank) *rank = comm->rank;
        if (device) *device = comm->device;
    });
}

int nufft_multi_term_range(size_t K, int nranks, int rank, size_t* r_begin, size_t* r_end) {
    return guard([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) nb::throw_invalid("multi_term_range: rank out of range");
        nb::term_range(K, nranks, rank, r_begin, r_end);
    });
}

int nufft_plan2_exec_multi_host(const nufft_plan2* plan, const double* c, size_t len, double* f, size_t batch,
                                nufft_comm* comm, int root, int mode) {
    return guard([&] {
        if (!plan || !comm) nb::throw_invalid("exec_multi: null argument");
        const nb::CorePlan& p = plan->core;
        if (len != p.n) nb::throw_invalid("exec_nufft2: length mismatch");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = cudaStreamPerThread;
        nb::DevBuf din(16 * p.n * batch, s), dout(16 * p.n * batch, s);
        nb::h2d(din.get(), c, 16 * p.n * batch, s);
        const int rc = nufft_plan2_exec_multi(plan, din.as<double>(), dout.as<double>(), batch, comm, root, mode, s);
        if (rc != NUFFT_OK) throw nb::Error(rc, nb::last_error());
        const bool receives = mode == NUFFT_MULTI_ALLREDUCE || comm->rank == root;
        if (receives) nb::d2h(f, dout.get(), 16 * p.n * batch, s);
        else NB_CUDA(cudaStreamSynchronize(s));
    });
}

int nufft_plan1_exec_terms(const nufft_plan1* plan, const double* c_dev, double* f_dev, size_t batch,
                           size_t r_begin, size_t r_end, void* stream) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        NB_CUDA(cudaSetDevice(p.device));
        if (r_end > p.K) r_end = p.K;
        nb::exec_transpose(p, reinterpret_cast<const double2*>(c_dev), reinterpret_cast<double2*>(f_dev), batch,
                           stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread, r_begin, r_end);
        if (r_end > r_begin) nb::fft_count(p.n, (r_end - r_begin) * batch);
    });
}

// Type I over G GPUs: rank g runs the transpose core on its r-range (both passes; pass B
// accumulates v_r X_r of those terms), and the natural-order partial sums are reduced once
// (pass B writes f column by column, so there is no contiguous chunk to reduce early).
int nufft_plan1_exec_multi(const nufft_plan1* plan, const double* c_dev, double* f_dev, size_t batch,
                           nufft_comm* comm, int root, int mode, void* stream) {
    return guard([&] {
        if (!plan || !comm) nb::throw_invalid("exec_multi: null argument");
        if (mode != NUFFT_MULTI_REDUCE && mode != NUFFT_MULTI_ALLREDUCE) nb::throw_invalid("exec_multi: mode");
        if (root < 0 || root >= comm->nranks) nb::throw_invalid("exec_multi: root out of range");
        const nb::CorePlan& p = plan->core;
        if (p.device != comm->device) nb::throw_invalid("exec_multi: plan and communicator on different devices");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        size_t r0, r1;
        nb::term_range(p.K, comm->nranks, comm->rank, &r0, &r1);
        nb::DevBuf part(sizeof(double2) * p.n * batch, s);
        nb::exec_transpose(p, reinterpret_cast<const double2*>(c_dev), part.as<double2>(), batch, s, r0, r1);
        const nb::NcclApi& api = nb::nccl();
        if (mode == NUFFT_MULTI_ALLREDUCE)
            nb::nccl_check(api.all_reduce(part.get(), f_dev, 2 * p.n * batch, ncclDouble, ncclSum, comm->comm, s),
                           "ncclAllReduce");
        else
            nb::nccl_check(api.reduce(part.get(), f_dev, 2 * p.n * batch, ncclDouble, ncclSum, root, comm->comm, s),
                           "ncclReduce");
        if (r1 > r0) nb::fft_count(p.n, (r1 - r0) * batch);
    });
}

int nufft_plan3_exec_terms(const nufft_plan3* plan, const double* c_dev, double* f_dev, size_t batch,
                           size_t r_begin, size_t r_end, void* stream) {
    return guard([&] {
        const nb::Plan3State& st = plan->st;
        NB_CUDA(cudaSetDevice(st.a.device));
        if (r_end > st.a.K) r_end = st.a.K;
        nb::exec_type3(st, reinterpret_cast<const double2*>(c_dev), reinterpret_cast<double2*>(f_dev), batch,
                       stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread, r_begin, r_end);
        if (r_end > r_begin) nb::fft_count(st.a.n, (r_end - r_begin) * st.inner.K * batch);
    });
}

// Type III over G GPUs: rank g takes the outer terms q in [K g/G, K (g+1)/G) (their inner
// type-I transforms, beta dot products and the epilogue's partial Horner sum), and the
// partial f are summed once (shard the (q, r) pairs, reduce f).
int nufft_plan3_exec_multi(const nufft_plan3* plan, const double* c_dev, double* f_dev, size_t batch,
                           nufft_comm* comm, int root, int mode, void* stream) {
    return guard([&] {
        if (!plan || !comm) nb::throw_invalid("exec_multi: null argument");
        if (mode != NUFFT_MULTI_REDUCE && mode != NUFFT_MULTI_ALLREDUCE) nb::throw_invalid("exec_multi: mode");
        if (root < 0 || root >= comm->nranks) nb::throw_invalid("exec_multi: root out of range");
        const nb::Plan3State& st = plan->st;
        if (st.a.device != comm->device) nb::throw_invalid("exec_multi: plan and communicator on different devices");
        NB_CUDA(cudaSetDevice(st.a.device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        size_t r0, r1;
        nb::term_range(st.a.K, comm->nranks, comm->rank, &r0, &r1);
        nb::DevBuf part(sizeof(double2) * st.a.n * batch, s);
        nb::exec_type3(st, reinterpret_cast<const double2*>(c_dev), part.as<double2>(), batch, s, r0, r1);
        const nb::NcclApi& api = nb::nccl();
        if (mode == NUFFT_MULTI_ALLREDUCE)
            nb::nccl_check(api.all_reduce(part.get(), f_dev, 2 * st.a.n * batch, ncclDouble, ncclSum, comm->comm, s),
                           "ncclAllReduce");
        else
            nb::nccl_check(api.reduce(part.get(), f_dev, 2 * st.a.n * batch, ncclDouble, ncclSum, root, comm->comm, s),
                           "ncclReduce");
        if (r1 > r0) nb::fft_count(st.a.n, (r1 - r0) * st.inner.K * batch);
    });
}

int nufft_plan2d2_exec_terms(const nufft_plan2d* plan, const double* C_dev, double* f_dev, size_t batch,
                             size_t r1_begin, size_t r1_end, void* stream) {
    return guard([&] {
        const nb::Plan2DState& st = plan->st;
        if (!st.fused) nb::throw_invalid("exec_terms (2D): fused plans only (power-of-two m, n in [16, 4096])");
        NB_CUDA(cudaSetDevice(st.device));
        nb::exec_2d_fused(st, reinterpret_cast<const double2*>(C_dev), reinterpret_cast<double2*>(f_dev), batch,
                          stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread, r1_begin, r1_end);
    });
}

// 2D over G GPUs: rank g takes the row-stage terms r1 in [Kx g/G, Kx (g+1)/G) (its share of
// the row stage and of the Kx Ky column steps; "shard r1") and the partial f
// are summed once.  Non-fused plans run whole on the root (the others contribute zeros).
int nufft_plan2d2_exec_multi(const nufft_plan2d* plan, const double* C_dev, double* f_dev, size_t batch,
                             nufft_comm* comm, int root, int mode, void* stream) {
    return guard([&] {
        if (!plan || !comm) nb::throw_invalid("exec_multi: null argument");
        if (mode != NUFFT_MULTI_REDUCE && mode != NUFFT_MULTI_ALLREDUCE) nb::throw_invalid("exec_multi: mode");
        if (root < 0 || root >= comm->nranks) nb::throw_invalid("exec_multi: root out of range");
        const nb::Plan2DState& st = plan->st;
        if (st.device != comm->device) nb::throw_invalid("exec_multi: plan and communicator on different devices");
        NB_CUDA(cudaSetDevice(st.device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        nb::DevBuf part(sizeof(double2) * st.count * batch, s);
        const double2* C = reinterpret_cast<const double2*>(C_dev);
        if (st.fused) {
            size_t r0, r1;
            nb::term_range(st.kx, comm->nranks, comm->rank, &r0, &r1);
            nb::exec_2d_fused(st, C, part.as<double2>(), batch, s, r0, r1);
        } else if (comm->rank == root) {
            nb::exec_2d(st, C, part.as<double2>(), batch, true, s);
        } else {
            NB_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(double2) * st.count * batch, s));
        }
        const nb::NcclApi& api = nb::nccl();
        if (mode == NUFFT_MULTI_ALLREDUCE)
            nb::nccl_check(api.all_reduce(part.get(), f_dev, 2 * st.count * batch, ncclDouble, ncclSum, comm->comm, s),
                           "ncclAllReduce");
        else
            nb::nccl_check(api.reduce(part.get(), f_dev, 2 * st.count * batch, ncclDouble, ncclSum, root, comm->comm, s),
                           "ncclReduce");
    });
}

int nufft_plan2_exec_terms_sorted(const nufft_plan2* plan, const double* c_dev, double* fs_dev, size_t r_begin,
                                  size_t r_end, void* stream) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (!p.fused || p.bk.log_n1 == 0) nb::throw_invalid("exec_terms_sorted: plan has no bucket order (fused path only)");
        if (r_end > p.K) r_end = p.K;
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        auto* fs = reinterpret_cast<double2*>(fs_dev);
        if (r_end <= r_begin) {
            NB_CUDA(cudaMemsetAsync(fs, 0, sizeof(double2) * p.n, s));
            return;
        }
        nb::DevBuf Y(sizeof(double2) * p.n * (r_end - r_begin), s);
        nb::exec_type2_pass1(p, reinterpret_cast<const double2*>(c_dev), Y.as<double2>(), r_begin, r_end, s);
        nb::exec_type2_pass2_rows(p, Y.as<double2>(), fs, r_begin, r_end, 0, 1ll << p.bk.log_n1, true, s);
        nb::fft_count(p.n, r_end - r_begin);
    });
}

int nufft_plan2_unpermute(const nufft_plan2* plan, const double* fs_dev, double* f_dev, size_t batch, void* stream) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (!p.fused || p.bk.log_n1 == 0) nb::throw_invalid("unpermute: plan has no bucket order (fused path only)");
        NB_CUDA(cudaSetDevice(p.device));
        nb::unpermute(p, reinterpret_cast<const double2*>(fs_dev), reinterpret_cast<double2*>(f_dev), batch,
                      stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread);
    });
}

int nufft_plan2_reduce_chunks(const nufft_plan2* plan, int nchunks, size_t* offsets) {
    return guard([&] {
        const nb::CorePlan& p = plan->core;
        if (nchunks < 1) nb::throw_invalid("reduce_chunks: nchunks must be >= 1");
        if (!p.fused || p.bk.log_n1 == 0) {
            for (int q = 0; q <= nchunks; ++q) offsets[q] = q == nchunks ? p.n : 0;
            return;
        }
        const long long n1 = 1ll << p.bk.log_n1;
        for (int q = 0; q <= nchunks; ++q) offsets[q] = (size_t)p.bk.rowoff_host[n1 * q / nchunks];
    });
}

int nufft_plan2_exec_multi(const nufft_plan2* plan, const double* c_dev, double* f_dev, size_t batch,
                           nufft_comm* comm, int root, int mode, void* stream) {
    return guard([&] {
        if (!plan || !comm) nb::throw_invalid("exec_multi: null argument");
        if (mode != NUFFT_MULTI_REDUCE && mode != NUFFT_MULTI_ALLREDUCE) nb::throw_invalid("exec_multi: mode");
        if (root < 0 || root >= comm->nranks) nb::throw_invalid("exec_multi: root out of range");
        const nb::CorePlan& p = plan->core;
        if (p.device != comm->device) nb::throw_invalid("exec_multi: plan and communicator on different devices");
        NB_CUDA(cudaSetDevice(p.device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        size_t r0, r1;
        nb::term_range(p.K, comm->nranks, comm->rank, &r0, &r1);
        const bool fused = p.fused && p.bk.log_n1 > 0;
        // scratch: two bucket-order partial slots (vector b reduces from slot b & 1 while
        // b + 1 computes into the other) and the rank's spectra
        nb::DevBuf fs(sizeof(double2) * p.n * std::min<size_t>(2, batch), s);
        nb::DevBuf Y(fused ? sizeof(double2) * p.n * std::max<size_t>(1, r1 - r0) : 16, s);
        cudaEvent_t ev[2][kReduceChunks], done[2];
        for (auto& e : ev)
            for (auto& x : e) NB_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (auto& x : done) NB_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        struct Events {  // destroyed after the streams are ordered (events are reference-counted)
            cudaEvent_t* a;
            cudaEvent_t* b;
            ~Events() {
                for (int i = 0; i < 2 * kReduceChunks; ++i) cudaEventDestroy(a[i]);
                for (int i = 0; i < 2; ++i) cudaEventDestroy(b[i]);
            }
        } guard_ev{&ev[0][0], done};
        // the comm stream must not start on fs before this call's allocations
        NB_CUDA(cudaEventRecord(done[0], s));
        NB_CUDA(cudaStreamWaitEvent(comm->cs, done[0], 0));
        for (size_t b = 0; b < batch; ++b) {
            const int slot = (int)(b & 1);
            double2* fsb = fs.as<double2>() + p.n * slot;
            if (b >= 2) NB_CUDA(cudaStreamWaitEvent(s, done[slot], 0));  // slot reduced + un-permuted
            exec_multi_one(p, reinterpret_cast<const double2*>(c_dev) + b * p.n,
                           reinterpret_cast<double2*>(f_dev) + b * p.n, fsb, Y.as<double2>(), comm, root, mode, s,
                           ev[slot]);
            NB_CUDA(cudaEventRecord(done[slot], comm->cs));
        }
        // the caller's stream (and the scratch frees on it) wait for the last reduce
        NB_CUDA(cudaStreamWaitEvent(s, done[(batch - 1) & 1], 0));
        if (batch >= 2) NB_CUDA(cudaStreamWaitEvent(s, done[batch & 1], 0));
        nb::fft_count(p.n, (r1 - r0) * batch);
    });
}

}  // extern "C"
