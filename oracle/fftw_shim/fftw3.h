/* TEST INFRASTRUCTURE ONLY. Minimal FFTW3-API shim: exactly the names the
 * reference's FftwProvider uses (proj/src/core/fft.cpp:21,46,85), backed by
 * oracle/fft_c.c. FFTW3 itself is not installed in this image; every number
 * obtained through this shim is "reference engine + substitute FFT". */
#ifndef ORACLE_FFTW3_SHIM_H
#define ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;
typedef struct fftw_iodim64_do_not_use_me {
    ptrdiff_t n;
    ptrdiff_t is;
    ptrdiff_t os;
} fftw_iodim64;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_guru64_dft(int rank, const fftw_iodim64* dims, int howmany_rank,
                               const fftw_iodim64* howmany_dims, fftw_complex* in,
                               fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
