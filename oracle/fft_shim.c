/* TEST INFRASTRUCTURE ONLY (oracle).
 *
 * FFTW-API shim: the three FFTW3 functions the reference library calls
 * (proj/include/nufft/fft.hpp:51-54 plan, :59-60 destroy, :98-107 execute),
 * implemented from the published definition of the unnormalized DFT
 *     out_j = sum_k in_k exp(sign * 2*pi*i*j*k/n),  sign = FFTW_FORWARD(-1)/BACKWARD(+1).
 * FFTW3 is a third-party dependency that is absent here and unpinned by the
 * reference (proj/CMakeLists.txt:12-13 only does find_library); see DESIGN.md.
 *
 *   n = 2^k : iterative radix-2 decimation-in-time over a bit-reversed copy,
 *             twiddles exp(sign*2*pi*i*j/n) evaluated in long double and rounded once.
 *   other n : direct O(n^2) sum with the exact index (j*k mod n) into the same
 *             kind of twiddle table, accumulated in long double.
 * in == out is allowed (the reference executes in place at fft.hpp:165).
 * Plans are immutable after creation, so concurrent executes are safe.
 * Used to build the reference headers unmodified (oracle/_ref) and by the
 * C restatement in oracle/nufft_oracle.c.  Never linked into the product. */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct fftw_plan_s {
    int n;
    int sign;
    int log2n; /* -1 when n is not a power of two */
    double* tw; /* tw[2*k], tw[2*k+1] = cos/sin(sign*2*pi*k/n), k < n */
    int* rev;   /* bit reversal permutation (power-of-two n only) */
};

static int ilog2_exact(int n) {
    int l = 0;
    while ((1 << l) < n) ++l;
    return (1 << l) == n ? l : -1;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
    (void)in;
    (void)out;
    (void)flags;
    if (n < 1) return NULL;
    struct fftw_plan_s* p = (struct fftw_plan_s*)calloc(1, sizeof(*p));
    if (!p) return NULL;
    p->n = n;
    p->sign = sign;
    p->log2n = ilog2_exact(n);
    p->tw = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    if (!p->tw) {
        free(p);
        return NULL;
    }
    const long double two_pi = 6.28318530717958647692528676655900577L;
    for (int k = 0; k < n; ++k) {
        const long double ang = (long double)sign * two_pi * (long double)k / (long double)n;
        p->tw[2 * k] = (double)cosl(ang);
        p->tw[2 * k + 1] = (double)sinl(ang);
    }
    if (p->log2n >= 0) {
        p->rev = (int*)malloc(sizeof(int) * (size_t)n);
        if (!p->rev) {
            free(p->tw);
            free(p);
            return NULL;
        }
        for (int i = 0; i < n; ++i) {
            int r = 0;
            for (int b = 0; b < p->log2n; ++b)
                if (i & (1 << b)) r |= 1 << (p->log2n - 1 - b);
            p->rev[i] = r;
        }
    }
    return p;
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    free(p->tw);
    free(p->rev);
    free(p);
}

static void exec_pow2(const struct fftw_plan_s* p, const double* in, double* out) {
    const int n = p->n;
    if (in == out) {
        for (int i = 0; i < n; ++i) {
            const int r = p->rev[i];
            if (r > i) {
                double a = out[2 * i], b = out[2 * i + 1];
                out[2 * i] = out[2 * r];
                out[2 * i + 1] = out[2 * r + 1];
                out[2 * r] = a;
                out[2 * r + 1] = b;
            }
        }
    } else {
        for (int i = 0; i < n; ++i) {
            out[2 * p->rev[i]] = in[2 * i];
            out[2 * p->rev[i] + 1] = in[2 * i + 1];
        }
    }
    for (int half = 1; half < n; half <<= 1) {
        const int stride = n / (2 * half); /* twiddle index step */
        for (int base = 0; base < n; base += 2 * half) {
            for (int j = 0; j < half; ++j) {
                const double wr = p->tw[2 * (j * stride)];
                const double wi = p->tw[2 * (j * stride) + 1];
                double* a = out + 2 * (base + j);
                double* b = out + 2 * (base + j + half);
                const double br = b[0] * wr - b[1] * wi;
                const double bi = b[0] * wi + b[1] * wr;
                b[0] = a[0] - br;
                b[1] = a[1] - bi;
                a[0] = a[0] + br;
                a[1] = a[1] + bi;
            }
        }
    }
}

static void exec_direct(const struct fftw_plan_s* p, const double* in, double* out) {
    const int n = p->n;
    double* tmp = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    if (!tmp) abort();
    for (int j = 0; j < n; ++j) {
        long double sr = 0.0L, si = 0.0L;
        int idx = 0; /* (j*k) mod n, advanced by j each step */
        for (int k = 0; k < n; ++k) {
            const long double wr = p->tw[2 * idx], wi = p->tw[2 * idx + 1];
            const long double xr = in[2 * k], xi = in[2 * k + 1];
            sr += xr * wr - xi * wi;
            si += xr * wi + xi * wr;
            idx += j;
            if (idx >= n) idx -= n;
        }
        tmp[2 * j] = (double)sr;
        tmp[2 * j + 1] = (double)si;
    }
    memcpy(out, tmp, sizeof(double) * 2 * (size_t)n);
    free(tmp);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    if (p->log2n >= 0)
        exec_pow2(p, (const double*)in, (double*)out);
    else
        exec_direct(p, (const double*)in, (double*)out);
}
