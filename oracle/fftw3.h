/* TEST INFRASTRUCTURE ONLY (oracle). Declarations of the three FFTW3 entry
 * points the reference calls (proj/include/nufft/fft.hpp:51-54, 59-60, 98-107),
 * written from FFTW's public API so the reference headers compile here.
 * FFTW3 itself is absent from this container; the matching
 * implementation is oracle/fft_shim.c.  Not shipped, not on the product path. */
#ifndef ORACLE_FFTW3_SHIM_H
#define ORACLE_FFTW3_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;
#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
#ifdef __cplusplus
}
#endif
#endif
