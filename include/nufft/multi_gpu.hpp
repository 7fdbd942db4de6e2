#pragma once

// Multi-GPU type II for C++ callers of the drop-in (no counterpart header in the
// reference: its exec_nufft2(plan, c, threads) splits the K terms over host
// threads, transforms.hpp:174-197; here the workers are GPUs, one process each).
//
//     // rank 0 makes the id, every rank receives it (MPI, a file, a socket):
//     nufft::CommId id = nufft::make_comm_id();                     // on rank 0
//     nufft::Communicator comm(id, world, rank, device);            // every rank
//     nufft::Plan2 plan = nufft::plan_nufft2(x, eps);               // same x everywhere
//     nufft::ComplexVector f = nufft::exec_nufft2(plan, c, comm);   // f complete on root
//
// Rank g evaluates the terms [K g/G, K (g+1)/G) and the partial sums are reduced over
// NCCL inside the library, chunk by chunk while pass 2 still runs
// (nufft_plan2_exec_multi, csrc/nufft2_multi.cu).  Results equal the single-GPU exec
// to rounding (the r-ranges are summed in a different order).

#include <array>
#include <memory>
#include <stdexcept>

#include "nufft/transforms.hpp"

namespace nufft {

using CommId = std::array<unsigned char, NUFFT_UNIQUE_ID_BYTES>;

inline CommId make_comm_id() {
    CommId id{};
    detail::check(nufft_comm_unique_id(id.data()));
    return id;
}

/// The library's NCCL communicator on one GPU (owns it, or wraps a caller's ncclComm_t).
class Communicator {
  public:
    Communicator(const CommId& id, int nranks, int rank, int device) {
        nufft_comm* c = nullptr;
        detail::check(nufft_comm_init(id.data(), nranks, rank, device, &c));
        h_.reset(c);
    }
    /// adopt an ncclComm_t the caller owns (it must outlive this object)
    static Communicator wrap(void* nccl_comm, int device) {
        nufft_comm* c = nullptr;
        detail::check(nufft_comm_wrap(nccl_comm, device, &c));
        return Communicator(c);
    }
    int nranks() const { return info()[0]; }
    int rank() const { return info()[1]; }
    int device() const { return info()[2]; }
    nufft_comm* get() const { return h_.get(); }

  private:
    explicit Communicator(nufft_comm* c) : h_(c) {}
    std::array<int, 3> info() const {
        std::array<int, 3> v{};
        detail::check(nufft_comm_info(h_.get(), &v[0], &v[1], &v[2]));
        return v;
    }
    struct Del {
        void operator()(nufft_comm* c) const { nufft_comm_destroy(c); }
    };
    std::unique_ptr<nufft_comm, Del> h_;
};

/// [r_begin, r_end) of one rank (host-only)
inline std::pair<std::size_t, std::size_t> term_range(std::size_t K, int nranks, int rank) {
    std::size_t a = 0, b = 0;
    detail::check(nufft_multi_term_range(K, nranks, rank, &a, &b));
    return {a, b};
}

/// Device pointers (c, f: batch x N complex on the communicator's device), ordered on `stream`.
inline void exec_nufft2_device(const Plan2& plan, const Complex* c_dev, Complex* f_dev, std::size_t batch,
                               const Communicator& comm, int root = 0, bool allreduce = false,
                               void* stream = nullptr) {
    detail::check(nufft_plan2_exec_multi(plan.device.get(), reinterpret_cast<const double*>(c_dev),
                                         reinterpret_cast<double*>(f_dev), batch, comm.get(), root,
                                         allreduce ? NUFFT_MULTI_ALLREDUCE : NUFFT_MULTI_REDUCE, stream));
}

/// Host vectors (the reference's exec_nufft2 signature with a communicator in place of
/// `threads`): every rank passes the same c; the full f is returned on `root` (or on every
/// rank with allreduce), an empty vector elsewhere.
inline ComplexVector exec_nufft2(const Plan2& plan, const ComplexVector& c, const Communicator& comm, int root = 0,
                                 bool allreduce = false) {
    if (c.size() != plan.size()) throw std::invalid_argument("exec_nufft2: length mismatch");
    const bool receives = allreduce || comm.rank() == root;
    ComplexVector f(receives ? c.size() : 0);
    detail::check(nufft_plan2_exec_multi_host(plan.device.get(), detail::dp(c), c.size(),
                                              receives ? detail::dp(f) : nullptr, 1, comm.get(), root,
                                              allreduce ? NUFFT_MULTI_ALLREDUCE : NUFFT_MULTI_REDUCE));
    return f;
}

}  // namespace nufft
