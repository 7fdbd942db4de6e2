// C-ABI of the seeded Gaussian sampler (include/nufft/random.hpp, the drop-in
// for the reference's GaussianSampler, random.hpp:14-60).  Host-only: bench.py
// and non-C++ callers draw the reference's seeded inputs through it, so the
// B200 arm and the reference arm of a benchmark see identical x and c.
#include <complex>
#include <cstring>
#include <new>

#include "../../include/nufft/random.hpp"
#include "../../include/nufft_b200.h"

struct nufft_sampler {
    nufft::GaussianSampler g;
    explicit nufft_sampler(uint64_t seed) : g(seed) {}
};

extern "C" {

int nufft_sampler_create(uint64_t seed, nufft_sampler** out) {
    if (!out) return NUFFT_INVALID_ARGUMENT;
    *out = new (std::nothrow) nufft_sampler(seed);
    return *out ? NUFFT_OK : NUFFT_OUT_OF_MEMORY;
}
void nufft_sampler_destroy(nufft_sampler* s) { delete s; }
double nufft_sampler_normal(nufft_sampler* s) { return s->g(); }
double nufft_sampler_uniform(nufft_sampler* s) { return s->g.uniform(); }
int nufft_sampler_uniform_vector(nufft_sampler* s, size_t n, double lo, double hi, double* out) {
    const double w = hi - lo;
    for (size_t i = 0; i < n; ++i) out[i] = lo + w * s->g.uniform();
    return NUFFT_OK;
}
int nufft_sampler_complex_vector(nufft_sampler* s, size_t n, double* out) {
    for (size_t i = 0; i < 2 * n; ++i) out[i] = s->g();
    return NUFFT_OK;
}

}  // extern "C"
