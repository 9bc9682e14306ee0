/* TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * Plain-C mixed-radix complex DFT used (1) by the FFTW-API shim that lets the
 * unmodified reference sources build in this image (FFTW3 is absent), and (2)
 * by the oracle restatement. Convention follows the reference's FftProvider
 * contract (proj/src/core/fft.hpp:7-10): forward is the unnormalised DFT with
 * kernel exp(-2*pi*i*l*k/N); "backward" is the unnormalised exp(+...) sum (the
 * 1/N factor is applied by the caller, as FftwProvider::inverse does at
 * proj/src/core/fft.cpp:69-75). Pinned against a direct O(n^2) DFT by
 * tests/test_oracle_cpu.py (mirrors proj/tests/unit/test_fft.cpp:66-80).
 */
#ifndef ORACLE_FFT_C_H
#define ORACLE_FFT_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fftc_plan fftc_plan;

/* sign = -1 forward, +1 backward (unnormalised). n >= 1. */
fftc_plan* fftc_plan_create(int64_t n, int sign);
void fftc_plan_destroy(fftc_plan* p);
int64_t fftc_plan_n(const fftc_plan* p);
/* In-place transform of one contiguous fiber of n interleaved (re,im)
 * doubles. work must hold 2*n doubles. */
void fftc_exec(const fftc_plan* p, double* x, double* work);

/* Strided batch: every fiber x[o*n*inner + k*inner + i], o<outer, i<inner. */
void fftc_axis(double* data, int64_t outer, int64_t n, int64_t inner, int sign);

#ifdef __cplusplus
}
#endif

#endif
