/* TEST INFRASTRUCTURE ONLY — see fftw3.h. Supports rank-1 transforms with an
 * arbitrary howmany loop nest (the reference uses howmany_rank 2:
 * {outer, n*inner} x {inner, 1}, proj/src/core/fft.cpp:32-42), in place or
 * out of place, unnormalised like FFTW. */
#include "fftw3.h"

#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../fft_c.h"

struct fftw_plan_s {
    fftc_plan* p;
    int64_t n, is, os;
    int hr;
    int64_t hn[8], his[8], hos[8];
};

fftw_plan fftw_plan_guru64_dft(int rank, const fftw_iodim64* dims, int howmany_rank,
                               const fftw_iodim64* howmany_dims, fftw_complex* in,
                               fftw_complex* out, int sign, unsigned flags)
{
    (void)in;
    (void)out;
    (void)flags;
    if (rank != 1 || howmany_rank < 0 || howmany_rank > 8)
        return NULL;
    struct fftw_plan_s* pl = (struct fftw_plan_s*)calloc(1, sizeof(*pl));
    pl->n = dims[0].n;
    pl->is = dims[0].is;
    pl->os = dims[0].os;
    pl->hr = howmany_rank;
    for (int i = 0; i < howmany_rank; ++i) {
        pl->hn[i] = howmany_dims[i].n;
        pl->his[i] = howmany_dims[i].is;
        pl->hos[i] = howmany_dims[i].os;
    }
    pl->p = fftc_plan_create(pl->n, sign);
    return pl;
}

void fftw_execute_dft(const fftw_plan pl, fftw_complex* in, fftw_complex* out)
{
    const int64_t n = pl->n;
    int64_t total = 1;
    for (int i = 0; i < pl->hr; ++i)
        total *= pl->hn[i];
    if (n == 0 || total == 0)
        return;
    /* Fast path: innermost howmany dim is unit stride in and out: gather
     * blocks of B consecutive fibers (cache-line friendly on strided axes). */
    enum { B = 16 };
    const int unit_inner = pl->hr >= 1 && pl->his[pl->hr - 1] == 1 && pl->hos[pl->hr - 1] == 1;
    const int64_t inner_n = unit_inner ? pl->hn[pl->hr - 1] : 1;
    const int outer_rank = unit_inner ? pl->hr - 1 : pl->hr;
    const int64_t blk = unit_inner ? B : 1;
    double* buf = (double*)malloc(sizeof(double) * 2 * (size_t)(n * blk));
    double* work = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    int64_t outer_total = 1;
    for (int i = 0; i < outer_rank; ++i)
        outer_total *= pl->hn[i];
    for (int64_t o = 0; o < outer_total; ++o) {
        int64_t rem = o, ioff = 0, ooff = 0;
        for (int i = outer_rank - 1; i >= 0; --i) {
            const int64_t idx = rem % pl->hn[i];
            rem /= pl->hn[i];
            ioff += idx * pl->his[i];
            ooff += idx * pl->hos[i];
        }
        for (int64_t i0 = 0; i0 < inner_n; i0 += blk) {
            const int64_t cnt = inner_n - i0 < blk ? inner_n - i0 : blk;
            const double* src = (const double*)(in + ioff + i0);
            double* dst = (double*)(out + ooff + i0);
            for (int64_t k = 0; k < n; ++k)
                for (int64_t b = 0; b < cnt; ++b) {
                    buf[2 * (b * n + k)] = src[2 * (k * pl->is + b)];
                    buf[2 * (b * n + k) + 1] = src[2 * (k * pl->is + b) + 1];
                }
            for (int64_t b = 0; b < cnt; ++b)
                fftc_exec(pl->p, buf + 2 * b * n, work);
            for (int64_t k = 0; k < n; ++k)
                for (int64_t b = 0; b < cnt; ++b) {
                    dst[2 * (k * pl->os + b)] = buf[2 * (b * n + k)];
                    dst[2 * (k * pl->os + b) + 1] = buf[2 * (b * n + k) + 1];
                }
        }
    }
    free(work);
    free(buf);
}

void fftw_destroy_plan(fftw_plan pl)
{
    if (!pl)
        return;
    fftc_plan_destroy(pl->p);
    free(pl);
}
