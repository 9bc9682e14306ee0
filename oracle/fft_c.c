/* TEST INFRASTRUCTURE ONLY — see fft_c.h. Stockham autosort mixed-radix DFT
 * (radix 4, 2 and a direct prime-radix butterfly), roots of unity from an
 * octant-reduced sin/cos so the tables are accurate to ~1 ulp. */
#include "fft_c.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct fftc_plan {
    int64_t n;
    int sign;
    int nf;
    int64_t fac[64];
    double* tw; /* n roots exp(sign*2*pi*i*k/n), interleaved */
};

/* exp(sign * 2*pi*i * k / n) with octant reduction (k in [0, n)). */
static void unit_root(int64_t k, int64_t n, int sign, double* re, double* im)
{
    k %= n;
    if (k < 0)
        k += n;
    const int64_t a = 8 * k; /* angle = (pi/4) * a / n */
    const int64_t o = a / n;
    const int64_t r = a - o * n;
    double c, s;
    if ((o & 1) == 0) {
        const double th = (M_PI / 4.0) * ((double)r / (double)n);
        c = cos(th);
        s = sin(th);
    } else {
        /* angle = (o+1)*pi/4 - th', th' = (pi/4)(n-r)/n; write as quadrant
         * q*pi/2 + (pi/2 - th') where q = (o-1)/2 */
        const double th = (M_PI / 4.0) * ((double)(n - r) / (double)n);
        c = sin(th);
        s = cos(th);
    }
    /* rotate by quadrant q * pi/2 */
    const int64_t q = o / 2;
    double cr, sr;
    switch (q & 3) {
    case 0: cr = c; sr = s; break;
    case 1: cr = -s; sr = c; break;
    case 2: cr = -c; sr = -s; break;
    default: cr = s; sr = -c; break;
    }
    *re = cr;
    *im = sign < 0 ? -sr : sr;
}

fftc_plan* fftc_plan_create(int64_t n, int sign)
{
    fftc_plan* p = (fftc_plan*)calloc(1, sizeof(fftc_plan));
    p->n = n;
    p->sign = sign;
    int64_t m = n;
    while (m % 4 == 0) {
        p->fac[p->nf++] = 4;
        m /= 4;
    }
    while (m % 2 == 0) {
        p->fac[p->nf++] = 2;
        m /= 2;
    }
    for (int64_t f = 3; m > 1; f += 2) {
        while (m % f == 0) {
            p->fac[p->nf++] = f;
            m /= f;
        }
        if (f * f > m && m > 1) {
            p->fac[p->nf++] = m;
            m = 1;
        }
    }
    p->tw = (double*)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    for (int64_t k = 0; k < n; ++k)
        unit_root(k, n, sign, &p->tw[2 * k], &p->tw[2 * k + 1]);
    return p;
}

void fftc_plan_destroy(fftc_plan* p)
{
    if (!p)
        return;
    free(p->tw);
    free(p);
}

int64_t fftc_plan_n(const fftc_plan* p)
{
    return p->n;
}

void fftc_exec(const fftc_plan* p, double* x, double* work)
{
    const int64_t n = p->n;
    if (n <= 1)
        return;
    double* src = x;
    double* dst = work;
    const double* tw = p->tw;
    int64_t ns = 1;
    double vr[64], vi[64];
    double* big_r = NULL;
    double* big_i = NULL;
    for (int s = 0; s < p->nf; ++s) {
        const int64_t R = p->fac[s];
        const int64_t m = n / R;
        double* ar = vr;
        double* ai = vi;
        if (R > 64) {
            big_r = (double*)realloc(big_r, sizeof(double) * 2 * (size_t)R);
            big_i = big_r + R;
            ar = big_r;
            ai = big_i;
        }
        const int64_t tstep = n / (ns * R);
        for (int64_t j = 0; j < m; ++j) {
            const int64_t jm = j % ns;
            for (int64_t r = 0; r < R; ++r) {
                const double a = src[2 * (j + r * m)];
                const double b = src[2 * (j + r * m) + 1];
                const int64_t t = r * jm * tstep; /* < n */
                const double wr = tw[2 * t], wi = tw[2 * t + 1];
                ar[r] = a * wr - b * wi;
                ai[r] = a * wi + b * wr;
            }
            const int64_t base = (j / ns) * ns * R + jm;
            if (R == 2) {
                const double r0 = ar[0] + ar[1], i0 = ai[0] + ai[1];
                const double r1 = ar[0] - ar[1], i1 = ai[0] - ai[1];
                dst[2 * base] = r0;
                dst[2 * base + 1] = i0;
                dst[2 * (base + ns)] = r1;
                dst[2 * (base + ns) + 1] = i1;
            } else if (R == 4) {
                /* X_q = sum_r a_r w4^{rq}, w4 = exp(sign*i*pi/2) */
                const double s0r = ar[0] + ar[2], s0i = ai[0] + ai[2];
                const double d0r = ar[0] - ar[2], d0i = ai[0] - ai[2];
                const double s1r = ar[1] + ar[3], s1i = ai[1] + ai[3];
                const double d1r = ar[1] - ar[3], d1i = ai[1] - ai[3];
                /* j*d1 where j = w4 = sign*i */
                const double jr = p->sign < 0 ? d1i : -d1i;
                const double ji = p->sign < 0 ? -d1r : d1r;
                dst[2 * base] = s0r + s1r;
                dst[2 * base + 1] = s0i + s1i;
                dst[2 * (base + ns)] = d0r + jr;
                dst[2 * (base + ns) + 1] = d0i + ji;
                dst[2 * (base + 2 * ns)] = s0r - s1r;
                dst[2 * (base + 2 * ns) + 1] = s0i - s1i;
                dst[2 * (base + 3 * ns)] = d0r - jr;
                dst[2 * (base + 3 * ns) + 1] = d0i - ji;
            } else {
                const int64_t rstep = n / R;
                for (int64_t q = 0; q < R; ++q) {
                    double sr = 0.0, si = 0.0;
                    for (int64_t r = 0; r < R; ++r) {
                        const int64_t t = ((r * q) % R) * rstep;
                        const double wr = tw[2 * t], wi = tw[2 * t + 1];
                        sr += ar[r] * wr - ai[r] * wi;
                        si += ar[r] * wi + ai[r] * wr;
                    }
                    dst[2 * (base + q * ns)] = sr;
                    dst[2 * (base + q * ns) + 1] = si;
                }
            }
        }
        ns *= R;
        double* t = src;
        src = dst;
        dst = t;
    }
    free(big_r);
    if (src != x)
        memcpy(x, src, sizeof(double) * 2 * (size_t)n);
}

void fftc_axis(double* data, int64_t outer, int64_t n, int64_t inner, int sign)
{
    if (n <= 1)
        return;
    fftc_plan* p = fftc_plan_create(n, sign);
    /* gather blocks of up to B consecutive fibers to stay cache friendly on
     * strided axes */
    enum { B = 16 };
    double* buf = (double*)malloc(sizeof(double) * 2 * (size_t)n * B);
    double* work = (double*)malloc(sizeof(double) * 2 * (size_t)n);
    for (int64_t o = 0; o < outer; ++o) {
        double* base = data + 2 * o * n * inner;
        for (int64_t i0 = 0; i0 < inner; i0 += B) {
            const int64_t cnt = inner - i0 < B ? inner - i0 : B;
            for (int64_t k = 0; k < n; ++k)
                for (int64_t b = 0; b < cnt; ++b) {
                    buf[2 * (b * n + k)] = base[2 * (k * inner + i0 + b)];
                    buf[2 * (b * n + k) + 1] = base[2 * (k * inner + i0 + b) + 1];
                }
            for (int64_t b = 0; b < cnt; ++b)
                fftc_exec(p, buf + 2 * b * n, work);
            for (int64_t k = 0; k < n; ++k)
                for (int64_t b = 0; b < cnt; ++b) {
                    base[2 * (k * inner + i0 + b)] = buf[2 * (b * n + k)];
                    base[2 * (k * inner + i0 + b) + 1] = buf[2 * (b * n + k) + 1];
                }
        }
    }
    free(work);
    free(buf);
    fftc_plan_destroy(p);
}
