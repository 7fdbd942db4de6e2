#pragma once

// Drop-in for proj/include/nufft/transforms.hpp: one-dimensional NUFFT types
// I, II, III with the reference's plan structs, function names and error
// behaviour.  Plans own a handle to the device plan (sample layout, factors
// metadata, buckets) and keep host mirrors of the members callers read
// (SampleSet x/s/t/gamma, rank, gamma).  The reference's factor matrices
// (K x N complex each) are materialized from the device only when accessed.
// Execution runs the sm_100a kernels; `threads` is accepted and ignored
// (one GPU launch sequence replaces the thread pool, results are
// deterministic regardless).

#include <cmath>
#include <cstddef>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "fft.hpp"
#include "lowrank.hpp"

namespace nufft {

/// Normalized samples with their nearest-grid-node assignment (transforms.hpp:25-32).
struct SampleSet {
    std::vector<double> x;
    std::vector<long> s;
    std::vector<std::size_t> t;
    double gamma = 0.0;

    std::size_t size() const { return x.size(); }
};

inline std::vector<double> normalize_samples(const std::vector<double>& raw) {
    std::vector<double> out(raw.size());
    if (!raw.empty()) detail::check(nufft_normalize_samples(raw.data(), raw.size(), out.data()));
    return out;
}

struct GridAssignment {
    std::vector<long> s;
    std::vector<std::size_t> t;
    double gamma = 0.0;
};

namespace detail {

// N*x - s without the rounding of the N*x product (transforms.hpp:60-64)
inline double exact_perturbation(double grid_size, double x, double s) {
    const double p = grid_size * x;
    const double err = std::fma(grid_size, x, -p);
    return (p - s) + err;
}

inline double snap_gamma(double gamma, double grid_size) {  // transforms.hpp:70-73
    constexpr double quarter_eps = 0x1p-54;
    return gamma <= grid_size * quarter_eps ? 0.0 : gamma;
}

inline void check_epsilon(double epsilon) {
    if (!(epsilon > 0.0) || !(epsilon < 1.0)) throw std::domain_error("epsilon must be in (0, 1)");
}

template <class H, void (*Destroy)(H*)>
std::shared_ptr<H> own(H* h) {
    return std::shared_ptr<H>(h, [](H* p) { Destroy(p); });
}

/// Factor columns materialized from the device plan on first access.
class LazyColumns {
  public:
    using Fill = void (*)(const void* plan, std::vector<ComplexVector>& u, std::vector<ComplexVector>& v);
    struct Cache {
        std::once_flag once;
        std::vector<ComplexVector> u, v;
        std::shared_ptr<const void> plan;
        Fill fill = nullptr;
    };
    LazyColumns() = default;
    LazyColumns(std::shared_ptr<Cache> c, bool is_u, std::size_t rank)
        : cache_(std::move(c)), is_u_(is_u), rank_(rank) {}
    std::size_t size() const { return rank_; }
    bool empty() const { return rank_ == 0; }
    const ComplexVector& operator[](std::size_t r) const { return cols()[r]; }
    const ComplexVector& at(std::size_t r) const { return cols().at(r); }
    auto begin() const { return cols().begin(); }
    auto end() const { return cols().end(); }

  private:
    const std::vector<ComplexVector>& cols() const {
        if (!cache_) throw std::logic_error("factors not available for this plan");
        std::call_once(cache_->once, [&] { cache_->fill(cache_->plan.get(), cache_->u, cache_->v); });
        return is_u_ ? cache_->u : cache_->v;
    }
    std::shared_ptr<Cache> cache_;
    bool is_u_ = true;
    std::size_t rank_ = 0;
};

}  // namespace detail

/// factors of a plan: rank plus lazily materialized u / v (lowrank.hpp:147-151 layout)
struct PlanFactors {
    std::size_t rank = 0;
    detail::LazyColumns u, v;
};

inline GridAssignment grid_assign(const std::vector<double>& x, std::size_t grid_size) {
    if (grid_size < 1) throw std::invalid_argument("grid_assign: grid size must be >= 1");
    GridAssignment out;
    out.s.resize(x.size());
    out.t.resize(x.size());
    detail::check(nufft_grid_assign(x.data(), x.size(), grid_size, out.s.data(), out.t.data(),
                                    &out.gamma));
    return out;
}

/// Type-II plan: nonuniform samples, integer frequencies 0..N-1 (transforms.hpp:105-114).
struct Plan2 {
    SampleSet samples;
    double epsilon = 0.0;
    PlanFactors factors;
    std::shared_ptr<detail::FftPlan> fft;
    std::shared_ptr<nufft_plan2> device;  // the B200 plan

    std::size_t size() const { return samples.size(); }
    std::size_t rank() const { return factors.rank; }
    double gamma() const { return samples.gamma; }
};

namespace detail {

inline void fill_plan2_factors(const void* h, std::vector<ComplexVector>& u,
                               std::vector<ComplexVector>& v) {
    auto* p = static_cast<const nufft_plan2*>(h);
    nufft_plan_info info{};
    check(nufft_plan2_info(p, &info));
    std::vector<Complex> U(info.rank * info.n), V(info.rank * info.n);
    check(nufft_plan2_factors(p, reinterpret_cast<double*>(U.data()), reinterpret_cast<double*>(V.data())));
    u.resize(info.rank);
    v.resize(info.rank);
    for (std::size_t r = 0; r < info.rank; ++r) {
        u[r].assign(U.begin() + r * info.n, U.begin() + (r + 1) * info.n);
        v[r].assign(V.begin() + r * info.n, V.begin() + (r + 1) * info.n);
    }
}

inline Plan2 wrap_plan2(nufft_plan2* raw, double epsilon) {
    Plan2 plan;
    plan.device = own<nufft_plan2, nufft_plan2_destroy>(raw);
    nufft_plan_info info{};
    check(nufft_plan2_info(raw, &info));
    plan.epsilon = epsilon;
    plan.samples.x.resize(info.n);
    plan.samples.s.resize(info.n);
    plan.samples.t.resize(info.n);
    check(nufft_plan2_samples(raw, plan.samples.x.data(), plan.samples.s.data(), plan.samples.t.data()));
    plan.samples.gamma = info.gamma;
    auto cache = std::make_shared<LazyColumns::Cache>();
    cache->plan = plan.device;
    cache->fill = &fill_plan2_factors;
    plan.factors.rank = info.rank;
    plan.factors.u = LazyColumns(cache, true, info.rank);
    plan.factors.v = LazyColumns(cache, false, info.rank);
    plan.fft = fft_plan_for(info.n);
    return plan;
}

}  // namespace detail

inline SampleSet make_sample_set(const std::vector<double>& raw, std::size_t grid_size) {
    SampleSet set;
    set.x = normalize_samples(raw);
    GridAssignment a = grid_assign(set.x, grid_size);
    set.s = std::move(a.s);
    set.t = std::move(a.t);
    set.gamma = a.gamma;
    return set;
}

inline Plan2 plan_nufft2(const std::vector<double>& x_raw, double epsilon) {
    nufft_plan2* raw = nullptr;
    detail::check(nufft_plan2_create(x_raw.data(), x_raw.size(), epsilon, -1, &raw));
    return detail::wrap_plan2(raw, epsilon);
}

/// f ~ F2~ c (transforms.hpp:168-199); `threads` kept for signature compatibility.
inline ComplexVector exec_nufft2(const Plan2& plan, const ComplexVector& c, unsigned threads = 1) {
    (void)threads;
    if (c.size() != plan.size()) throw std::invalid_argument("exec_nufft2: length mismatch");
    ComplexVector f(c.size());
    detail::check(nufft_plan2_exec_host(plan.device.get(), detail::dp(c), c.size(), detail::dp(f), 1));
    return f;
}

/// F2~* f (transforms.hpp:226-232)
inline ComplexVector exec_nufft2_adjoint(const Plan2& plan, const ComplexVector& f) {
    if (f.size() != plan.size()) throw std::invalid_argument("nufft transpose: length mismatch");
    ComplexVector out(f.size());
    detail::check(nufft_plan2_adjoint_host(plan.device.get(), detail::dp(f), f.size(), detail::dp(out)));
    return out;
}

/// Type-I plan: equispaced samples j/N, frequencies in [0, N] (transforms.hpp:237-244).
struct Plan1Inner {
    SampleSet samples;
    double epsilon = 0.0;
    PlanFactors factors;  // rank only (u/v not mirrored for type I)
    std::shared_ptr<detail::FftPlan> fft;

    std::size_t size() const { return samples.size(); }
    std::size_t rank() const { return factors.rank; }
    double gamma() const { return samples.gamma; }
};

struct Plan1 {
    std::vector<double> freqs;
    Plan1Inner inner;
    std::shared_ptr<nufft_plan1> device;

    std::size_t size() const { return freqs.size(); }
    std::size_t rank() const { return inner.rank(); }
    double gamma() const { return inner.gamma(); }
};

inline Plan1 plan_nufft1(const std::vector<double>& omega, double epsilon) {
    nufft_plan1* raw = nullptr;
    detail::check(nufft_plan1_create(omega.data(), omega.size(), epsilon, -1, &raw));
    Plan1 plan;
    plan.device = detail::own<nufft_plan1, nufft_plan1_destroy>(raw);
    nufft_plan_info info{};
    detail::check(nufft_plan1_info(raw, &info));
    plan.freqs = omega;
    auto& in = plan.inner;
    in.epsilon = epsilon;
    in.samples.x.resize(info.n);
    in.samples.s.resize(info.n);
    in.samples.t.resize(info.n);
    detail::check(nufft_plan1_samples(raw, in.samples.x.data(), in.samples.s.data(), in.samples.t.data()));
    in.samples.gamma = info.gamma;
    in.factors.rank = info.rank;
    in.fft = fft_plan_for(info.n);
    return plan;
}

inline ComplexVector exec_nufft1(const Plan1& plan, const ComplexVector& c) {
    if (c.size() != plan.size()) throw std::invalid_argument("nufft transpose: length mismatch");
    ComplexVector f(c.size());
    detail::check(nufft_plan1_exec_host(plan.device.get(), detail::dp(c), c.size(), detail::dp(f), 1));
    return f;
}

namespace detail {
/// F1~* g = conj(F2~ conj(g)) on the inner plan (transforms.hpp:294-300)
inline ComplexVector exec_nufft1_adjoint(const Plan1& plan, const ComplexVector& g) {
    if (g.size() != plan.size()) throw std::invalid_argument("nufft transpose: length mismatch");
    ComplexVector out(g.size());
    check(nufft_plan1_adjoint_host(plan.device.get(), dp(g), g.size(), dp(out)));
    return out;
}
}  // namespace detail

/// Type-III plan (transforms.hpp:308-319).
struct Plan3 {
    SampleSet samples;
    std::vector<double> freqs;
    PlanFactors factorsA;  // rank only
    bool bTrivial = true;
    std::size_t kc = 0;
    std::shared_ptr<nufft_plan3> device;

    std::size_t size() const { return samples.size(); }
    std::size_t effective_rank() const { return kc; }
};

inline Plan3 plan_nufft3(const std::vector<double>& x_raw, const std::vector<double>& omega,
                         double epsilon) {
    nufft_plan3* raw = nullptr;
    detail::check(nufft_plan3_create(x_raw.data(), omega.data(), x_raw.size(), omega.size(), epsilon,
                                     -1, &raw));
    Plan3 plan;
    plan.device = detail::own<nufft_plan3, nufft_plan3_destroy>(raw);
    nufft_plan_info info{};
    detail::check(nufft_plan3_info(raw, &info));
    plan.freqs = omega;
    plan.samples.x.resize(info.n);
    plan.samples.s.resize(info.n);
    plan.samples.t.resize(info.n);
    detail::check(nufft_plan3_samples(raw, plan.samples.x.data(), plan.samples.s.data(), plan.samples.t.data()));
    plan.samples.gamma = info.gamma;
    plan.factorsA.rank = info.rank;
    plan.bTrivial = info.btrivial != 0;
    plan.kc = info.effective_rank;
    return plan;
}

inline ComplexVector exec_nufft3(const Plan3& plan, const ComplexVector& c) {
    if (c.size() != plan.size()) throw std::invalid_argument("exec_nufft3: length mismatch");
    ComplexVector f(c.size());
    detail::check(nufft_plan3_exec_host(plan.device.get(), detail::dp(c), c.size(), detail::dp(f), 1));
    return f;
}

}  // namespace nufft
