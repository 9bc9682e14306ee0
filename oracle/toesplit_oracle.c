/* TEST INFRASTRUCTURE ONLY — see toesplit_oracle.h for the contract and pin.
 * Plain-C restatement of the reference split-FFT engine; references are
 * relative to /root/reference/proj. */
#include "toesplit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fft_c.h"

/* ------------------------------------------------------------------ util */

static int64_t volume(int d, const int64_t* shape)
{
    int64_t v = 1;
    for (int a = 0; a < d; ++a)
        v *= shape[a];
    return v;
}

/* tensor.cpp:170-186: inner = prod of lengths after axis, outer = before */
static int64_t inner_count(int d, const int64_t* shape, int axis)
{
    int64_t v = 1;
    for (int a = axis + 1; a < d; ++a)
        v *= shape[a];
    return v;
}

static int64_t outer_count(const int64_t* shape, int axis)
{
    int64_t v = 1;
    for (int a = 0; a < axis; ++a)
        v *= shape[a];
    return v;
}

static int check_levels(int d, const int64_t* levels)
{
    if (d < 1 || d > 31 || !levels)
        return ORC_EINVAL;
    for (int a = 0; a < d; ++a)
        if (levels[a] < 1)
            return ORC_ESHAPE;
    return ORC_OK;
}

/* complex helpers on interleaved doubles; operand order follows
 * std::complex<double> (a+bi)(c+di) = (ac-bd) + (ad+bc)i */
static inline void cmul(double a, double b, double c, double d, double* re, double* im)
{
    *re = a * c - b * d;
    *im = a * d + b * c;
}

/* ------------------------------------------------------------ instances */

/* instance.hpp:11-26 */
uint64_t orc_splitmix_next(uint64_t* state)
{
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double next_unit(uint64_t* s)
{
    return (double)(orc_splitmix_next(s) >> 11) * 0x1.0p-53;
}

typedef struct {
    uint64_t state;
    double sigma;
    double spare;
    int has_spare;
} gauss_t;

/* instance.cpp:8-11 (stream split) and :13-34 (Box-Muller, cached spare) */
static void gauss_init(gauss_t* g, uint64_t seed, uint64_t role, double variance)
{
    g->state = seed ^ ((role + 1) * 0x9E3779B97F4A7C15ull);
    g->sigma = sqrt(variance);
    g->spare = 0.0;
    g->has_spare = 0;
}

static double gauss_next(gauss_t* g)
{
    if (g->has_spare) {
        g->has_spare = 0;
        return g->spare;
    }
    const double u1 = 1.0 - next_unit(&g->state);
    const double u2 = next_unit(&g->state);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * M_PI * u2;
    g->spare = g->sigma * r * sin(a);
    g->has_spare = 1;
    return g->sigma * r * cos(a);
}

/* instance.cpp:43-103: group average over single-level lag negations */
static void symmetrize_lags(double* lags, int d, const int64_t* levels, int skew)
{
    const uint32_t patterns = 1u << d;
    const double weight = 1.0 / (double)patterns;
    int64_t lag_shape[32];
    for (int a = 0; a < d; ++a)
        lag_shape[a] = 2 * levels[a] - 1;
    const int64_t total = volume(d, lag_shape);
    int64_t idx[32] = {0};
    for (int64_t off = 0; off < total; ++off) {
        int canonical = 1;
        for (int a = 0; a < d && canonical; ++a)
            canonical = idx[a] >= levels[a] - 1;
        if (canonical) {
            int zero_lag = 0;
            for (int a = 0; a < d && !zero_lag; ++a)
                zero_lag = idx[a] == levels[a] - 1;
            double ar = 0.0, ai = 0.0;
            if (!(skew && zero_lag))
                for (uint32_t sig = 0; sig < patterns; ++sig) {
                    int64_t src = 0;
                    double chi = 1.0;
                    for (int a = 0; a < d; ++a) {
                        int64_t k = idx[a];
                        if ((sig >> a) & 1u) {
                            k = lag_shape[a] - 1 - k;
                            if (skew)
                                chi = -chi;
                        }
                        src = src * lag_shape[a] + k;
                    }
                    const double w = chi * weight;
                    ar += w * lags[2 * src];
                    ai += w * lags[2 * src + 1];
                }
            for (uint32_t sig = 0; sig < patterns; ++sig) {
                int64_t dst = 0;
                double chi = 1.0;
                for (int a = 0; a < d; ++a) {
                    int64_t k = idx[a];
                    if ((sig >> a) & 1u) {
                        k = lag_shape[a] - 1 - k;
                        if (skew)
                            chi = -chi;
                    }
                    dst = dst * lag_shape[a] + k;
                }
                lags[2 * dst] = chi * ar;
                lags[2 * dst + 1] = chi * ai;
            }
        }
        for (int a = d - 1; a >= 0; --a) {
            if (++idx[a] < lag_shape[a])
                break;
            idx[a] = 0;
        }
    }
}

/* instance.cpp:107-122 */
int orc_random_lags(int d, const int64_t* levels, uint64_t seed, double variance, int symmetry,
                    double* out)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    if (!(variance >= 0.0) || symmetry < 0 || symmetry > 2 || !out)
        return ORC_EINVAL;
    int64_t lag_shape[32];
    for (int a = 0; a < d; ++a)
        lag_shape[a] = 2 * levels[a] - 1;
    const int64_t total = volume(d, lag_shape);
    gauss_t g;
    gauss_init(&g, seed, 0, variance);
    for (int64_t i = 0; i < total; ++i) {
        out[2 * i] = gauss_next(&g);
        out[2 * i + 1] = gauss_next(&g);
    }
    if (symmetry != 0)
        symmetrize_lags(out, d, levels, symmetry == 2);
    return ORC_OK;
}

/* instance.cpp:124-131 */
int orc_random_vector(int d, const int64_t* levels, uint64_t seed, double variance, double* out)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    if (!(variance >= 0.0) || !out)
        return ORC_EINVAL;
    const int64_t s = volume(d, levels);
    gauss_t g;
    gauss_init(&g, seed, 1, variance);
    for (int64_t i = 0; i < s; ++i) {
        out[2 * i] = gauss_next(&g);
        out[2 * i + 1] = gauss_next(&g);
    }
    return ORC_OK;
}

/* BASELINE.json configs[1]: G_ij(m) = (d_ij - rh_i rh_j) e^{ikr}/r
 *   + (d_ij - 3 rh_i rh_j) e^{ikr}/(k^2 r^3), G(0) = self * I. rh_i rh_j is
 * formed as m_i m_j / r^2 so mirrored lags are bit-exact (+/-). */
int orc_dyadic_lags(int d, const int64_t* levels, int i, int j, double k, double self_re,
                    double self_im, double* out)
{
    return orc_dyadic_lags_slab(d, levels, i, j, k, self_re, self_im, 0, 2 * levels[0] - 1, out);
}

/* The same values for the axis-0 lag rows [row0, row1) only (written at their
 * place in the full tensor), so a caller can fill one tensor from several
 * threads. */
int orc_dyadic_lags_slab(int d, const int64_t* levels, int i, int j, double k, double self_re,
                         double self_im, int64_t row0, int64_t row1, double* out)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    if (i < 0 || j < 0 || i >= d || j >= d || !out)
        return ORC_EINVAL;
    int64_t lag_shape[32];
    for (int a = 0; a < d; ++a)
        lag_shape[a] = 2 * levels[a] - 1;
    if (row0 < 0 || row1 > lag_shape[0] || row0 > row1)
        return ORC_EINVAL;
    const int64_t row = volume(d, lag_shape) / lag_shape[0];
    const int64_t total = row1 * row;
    int64_t idx[32] = {0};
    idx[0] = row0;
    const double delta = i == j ? 1.0 : 0.0;
    for (int64_t off = row0 * row; off < total; ++off) {
        double r2 = 0.0;
        for (int a = 0; a < d; ++a) {
            const double m = (double)(idx[a] - (levels[a] - 1));
            r2 += m * m;
        }
        if (r2 == 0.0) {
            out[2 * off] = delta * self_re;
            out[2 * off + 1] = delta * self_im;
        } else {
            const double mi = (double)(idx[i] - (levels[i] - 1));
            const double mj = (double)(idx[j] - (levels[j] - 1));
            const double rr = mi * mj / r2;
            const double r = sqrt(r2);
            const double c = cos(k * r), s = sin(k * r);
            const double a1 = (delta - rr) / r;
            const double a2 = (delta - 3.0 * rr) / (k * k * r2 * r);
            const double amp = a1 + a2;
            out[2 * off] = amp * c;
            out[2 * off + 1] = amp * s;
        }
        for (int a = d - 1; a >= 0; --a) {
            if (++idx[a] < lag_shape[a])
                break;
            idx[a] = 0;
        }
    }
    return ORC_OK;
}

/* generator.cpp:38-62, per-axis generalisation */
int orc_validate_symmetry(int d, const int64_t* levels, const double* lags, const int* axis_sign)
{
    int64_t lag_shape[32];
    for (int a = 0; a < d; ++a)
        lag_shape[a] = 2 * levels[a] - 1;
    for (int a = 0; a < d; ++a) {
        if (axis_sign[a] == 0)
            continue;
        const int64_t len = lag_shape[a];
        const int64_t inner = inner_count(d, lag_shape, a);
        const int64_t outer = outer_count(lag_shape, a);
        for (int64_t o = 0; o < outer; ++o)
            for (int64_t k = 0; k < len; ++k)
                for (int64_t i = 0; i < inner; ++i) {
                    const int64_t l = (o * len + k) * inner + i;
                    const int64_t r = (o * len + (len - 1 - k)) * inner + i;
                    if (axis_sign[a] > 0) {
                        if (lags[2 * l] != lags[2 * r] || lags[2 * l + 1] != lags[2 * r + 1])
                            return ORC_ESYM;
                    } else {
                        if (lags[2 * l] != -lags[2 * r] || lags[2 * l + 1] != -lags[2 * r + 1])
                            return ORC_ESYM;
                    }
                }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------- spectra */

/* kernel.cpp:17-21 */
static int64_t stored_axis_length(int64_t n, int odd)
{
    return odd ? (n + 1) / 2 : n / 2 + 1;
}

/* kernel.cpp:25-37: full index -> stored index, *mirrored flag */
static int64_t mirror_source(int64_t n, int odd, int64_t k, int* mirrored)
{
    if (odd) {
        const int64_t stored = stored_axis_length(n, 1);
        if (k < stored) {
            *mirrored = 0;
            return k;
        }
        *mirrored = 1;
        return n - 1 - k;
    }
    if (k <= n / 2) {
        *mirrored = 0;
        return k;
    }
    *mirrored = 1;
    return n - k;
}

static void block_shape(int d, const int64_t* levels, uint32_t bits, int compressed, int64_t* out)
{
    for (int a = 0; a < d; ++a)
        out[a] = compressed ? stored_axis_length(levels[a], (bits >> a) & 1u) : levels[a];
}

int64_t orc_spectra_elems(int d, const int64_t* levels, int compressed)
{
    if (check_levels(d, levels))
        return -1;
    int64_t total = 0;
    int64_t shp[32];
    for (uint32_t b = 0; b < (1u << d); ++b) {
        block_shape(d, levels, b, compressed, shp);
        total += volume(d, shp);
    }
    return total;
}

/* kernel.cpp:50-82 */
int orc_embed_generator(int d, const int64_t* levels, const double* lags, double s0_re,
                        double s0_im, double* out)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    int64_t shp[32];
    for (int a = 0; a < d; ++a)
        shp[a] = 2 * levels[a];
    const int64_t total = volume(d, shp);
    int64_t idx[32] = {0};
    for (int64_t off = 0; off < total; ++off) {
        int padding = 0;
        int64_t lag_off = 0;
        for (int a = 0; a < d; ++a) {
            const int64_t n = levels[a];
            const int64_t j = idx[a];
            if (j == n) {
                padding = 1;
                break;
            }
            const int64_t m = j < n ? j : j - 2 * n;
            lag_off = lag_off * (2 * n - 1) + (m + n - 1);
        }
        out[2 * off] = padding ? s0_re : lags[2 * lag_off];
        out[2 * off + 1] = padding ? s0_im : lags[2 * lag_off + 1];
        for (int a = d - 1; a >= 0; --a) {
            if (++idx[a] < shp[a])
                break;
            idx[a] = 0;
        }
    }
    return ORC_OK;
}

/* fft.cpp:65-87 (forward unnormalised; inverse then 1/n sweep) */
static void fft_axis(int d, const int64_t* shape, double* t, int axis, int inverse)
{
    const int64_t n = shape[axis];
    fftc_axis(t, outer_count(shape, axis), n, inner_count(d, shape, axis), inverse ? +1 : -1);
    if (inverse) {
        const double scale = 1.0 / (double)n;
        const int64_t s = volume(d, shape);
        for (int64_t i = 0; i < 2 * s; ++i)
            t[i] *= scale;
    }
}

int orc_fft_axis(int d, const int64_t* shape, double* t, int axis, int inverse)
{
    if (check_levels(d, shape) || axis < 0 || axis >= d)
        return ORC_EINVAL;
    fft_axis(d, shape, t, axis, inverse);
    return ORC_OK;
}

/* kernel.cpp:223-258 */
static void fold_axis(int d, const int64_t* shape, const double* t, int axis, int odd, double* out)
{
    const int64_t n = shape[axis] / 2;
    int64_t oshape[32];
    memcpy(oshape, shape, sizeof(int64_t) * (size_t)d);
    oshape[axis] = n;
    const int64_t inner = inner_count(d, shape, axis);
    const int64_t outer = outer_count(shape, axis);
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t k = 0; k < n; ++k) {
            const double ang = -M_PI * (double)k / (double)n;
            const double fr = cos(ang), fi = sin(ang);
            const double* lo = t + 2 * ((o * 2 * n + k) * inner);
            const double* hi = lo + 2 * n * inner;
            double* row = out + 2 * ((o * n + k) * inner);
            for (int64_t i = 0; i < inner; ++i) {
                if (odd) {
                    const double dr = lo[2 * i] - hi[2 * i], di = lo[2 * i + 1] - hi[2 * i + 1];
                    cmul(fr, fi, dr, di, &row[2 * i], &row[2 * i + 1]);
                } else {
                    row[2 * i] = lo[2 * i] + hi[2 * i];
                    row[2 * i + 1] = lo[2 * i + 1] + hi[2 * i + 1];
                }
            }
        }
}

/* kernel.cpp:260-275 */
static void branchwise_blocks(int d, const int64_t* shape, const double* t, int axis, uint32_t bits,
                              double** blocks)
{
    if (axis == d) {
        const int64_t s = volume(d, shape);
        memcpy(blocks[bits], t, sizeof(double) * 2 * (size_t)s);
        for (int a = 0; a < d; ++a)
            fft_axis(d, shape, blocks[bits], a, 0);
        return;
    }
    int64_t oshape[32];
    memcpy(oshape, shape, sizeof(int64_t) * (size_t)d);
    oshape[axis] /= 2;
    double* half = (double*)malloc(sizeof(double) * 2 * (size_t)volume(d, oshape));
    fold_axis(d, shape, t, axis, 0, half);
    branchwise_blocks(d, oshape, half, axis + 1, bits, blocks);
    fold_axis(d, shape, t, axis, 1, half);
    branchwise_blocks(d, oshape, half, axis + 1, bits | (1u << axis), blocks);
    free(half);
}

static double max_abs(const double* t, int64_t s)
{
    double m = 0.0;
    for (int64_t i = 0; i < s; ++i) {
        const double v = hypot(t[2 * i], t[2 * i + 1]);
        if (v > m)
            m = v;
    }
    return m;
}

/* kernel.cpp:308-323 (branchwise precompute) + kernel.cpp:325-390
 * (compression with numerical mirror validation, per-axis sign) */
int orc_precompute(int d, const int64_t* levels, const double* lags, double s0_re, double s0_im,
                   int compressed, const int* axis_sign, double* out_blocks)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    if (compressed)
        for (int a = 0; a < d; ++a)
            if (!axis_sign || axis_sign[a] == 0)
                return ORC_ESYM;
    const int64_t s = volume(d, levels);
    int64_t eshape[32];
    for (int a = 0; a < d; ++a)
        eshape[a] = 2 * levels[a];
    double* emb = (double*)malloc(sizeof(double) * 2 * (size_t)volume(d, eshape));
    orc_embed_generator(d, levels, lags, s0_re, s0_im, emb);
    const uint32_t nb = 1u << d;
    double** full = (double**)malloc(sizeof(double*) * nb);
    for (uint32_t b = 0; b < nb; ++b)
        full[b] = (double*)malloc(sizeof(double) * 2 * (size_t)s);
    branchwise_blocks(d, eshape, emb, 0, 0, full);
    free(emb);

    st = ORC_OK;
    double* dst = out_blocks;
    for (uint32_t b = 0; b < nb && st == ORC_OK; ++b) {
        if (!compressed) {
            memcpy(dst, full[b], sizeof(double) * 2 * (size_t)s);
            dst += 2 * s;
            continue;
        }
        const double scale = max_abs(full[b], s);
        const double tol = 1e-9 * (scale > 1.0 ? scale : 1.0);
        for (int a = 0; a < d && st == ORC_OK; ++a) {
            const int64_t n = levels[a];
            const int64_t inner = inner_count(d, levels, a);
            const int64_t outer = outer_count(levels, a);
            const int odd = (b >> a) & 1u;
            const double sg = axis_sign[a] > 0 ? 1.0 : -1.0;
            for (int64_t o = 0; o < outer && st == ORC_OK; ++o)
                for (int64_t kk = 0; kk < n && st == ORC_OK; ++kk) {
                    const int64_t mk = odd ? n - 1 - kk : (n - kk) % n;
                    const double* lhs = full[b] + 2 * ((o * n + kk) * inner);
                    const double* rhs = full[b] + 2 * ((o * n + mk) * inner);
                    for (int64_t i = 0; i < inner; ++i)
                        if (hypot(lhs[2 * i] - sg * rhs[2 * i], lhs[2 * i + 1] - sg * rhs[2 * i + 1]) > tol) {
                            st = ORC_ESYM;
                            break;
                        }
                }
        }
        if (st)
            break;
        int64_t sshape[32];
        block_shape(d, levels, b, 1, sshape);
        const int64_t cnt = volume(d, sshape);
        int64_t sidx[32] = {0};
        for (int64_t off = 0; off < cnt; ++off) {
            int64_t src = 0;
            for (int a = 0; a < d; ++a)
                src = src * levels[a] + sidx[a];
            dst[2 * off] = full[b][2 * src];
            dst[2 * off + 1] = full[b][2 * src + 1];
            for (int a = d - 1; a >= 0; --a) {
                if (++sidx[a] < sshape[a])
                    break;
                sidx[a] = 0;
            }
        }
        dst += 2 * cnt;
    }
    for (uint32_t b = 0; b < nb; ++b)
        free(full[b]);
    free(full);
    return st;
}

/* -------------------------------------------------------------- engine */

typedef struct {
    int d;
    const int64_t* levels;
    int64_t s;
    const double* const* blocks; /* per branch id */
    int compressed;
    const int* axis_sign;
    int64_t fwd, inv, diag, phase, live, peak;
    int part, q; /* partition: follow only bit (part>>depth)&1 for depth < q */
} ctx_t;

/* tensor.cpp:227-247 */
static void phase_inplace(int d, const int64_t* shape, double* t, int axis, int conjugate)
{
    const int64_t n = shape[axis];
    const int64_t inner = inner_count(d, shape, axis);
    const int64_t outer = outer_count(shape, axis);
    const double sign = conjugate ? 1.0 : -1.0;
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t k = 0; k < n; ++k) {
            const double ang = sign * M_PI * (double)k / (double)n;
            const double fr = cos(ang), fi = sin(ang);
            double* row = t + 2 * ((o * n + k) * inner);
            for (int64_t i = 0; i < inner; ++i) {
                const double a = row[2 * i], b = row[2 * i + 1];
                cmul(a, b, fr, fi, &row[2 * i], &row[2 * i + 1]);
            }
        }
}

int orc_phase_axis(int d, const int64_t* shape, double* t, int axis, int conjugate)
{
    if (check_levels(d, shape) || axis < 0 || axis >= d)
        return ORC_EINVAL;
    phase_inplace(d, shape, t, axis, conjugate);
    return ORC_OK;
}

/* engine_split.cpp:13-37: even = 0.5 * (even + e^{+i pi k/n} odd) */
static void merge_loop(ctx_t* c, double* even, const double* odd, int axis)
{
    const int64_t n = c->levels[axis];
    const int64_t inner = inner_count(c->d, c->levels, axis);
    const int64_t outer = outer_count(c->levels, axis);
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t k = 0; k < n; ++k) {
            const double ang = M_PI * (double)k / (double)n;
            const double fr = cos(ang), fi = sin(ang);
            double* re = even + 2 * ((o * n + k) * inner);
            const double* ro = odd ? odd + 2 * ((o * n + k) * inner) : NULL;
            for (int64_t i = 0; i < inner; ++i) {
                double pr = 0.0, pi = 0.0;
                if (ro)
                    cmul(fr, fi, ro[2 * i], ro[2 * i + 1], &pr, &pi);
                re[2 * i] = 0.5 * (re[2 * i] + pr);
                re[2 * i + 1] = 0.5 * (re[2 * i + 1] + pi);
            }
        }
}

/* kernel.cpp:126-219 (full multiply and remapped mirror multiply) */
static void multiply_into(ctx_t* c, double* t, uint32_t b)
{
    const int d = c->d;
    const double* q = c->blocks[b];
    if (!c->compressed) {
        for (int64_t i = 0; i < c->s; ++i) {
            const double a = t[2 * i], bb = t[2 * i + 1];
            cmul(a, bb, q[2 * i], q[2 * i + 1], &t[2 * i], &t[2 * i + 1]);
        }
        return;
    }
    int64_t sshape[32], stride[32];
    block_shape(d, c->levels, b, 1, sshape);
    int64_t acc = 1;
    for (int a = d - 1; a >= 0; --a) {
        stride[a] = acc;
        acc *= sshape[a];
    }
    int64_t idx[32] = {0};
    for (int64_t i = 0; i < c->s; ++i) {
        int64_t off = 0;
        double sign = 1.0;
        for (int a = 0; a < d; ++a) {
            int mirrored = 0;
            const int64_t src = mirror_source(c->levels[a], (b >> a) & 1u, idx[a], &mirrored);
            off += src * stride[a];
            if (mirrored)
                sign *= c->axis_sign[a] > 0 ? 1.0 : -1.0;
        }
        const double qr = sign * q[2 * off], qi = sign * q[2 * off + 1];
        const double a = t[2 * i], bb = t[2 * i + 1];
        cmul(a, bb, qr, qi, &t[2 * i], &t[2 * i + 1]);
        for (int a2 = d - 1; a2 >= 0; --a2) {
            if (++idx[a2] < c->levels[a2])
                break;
            idx[a2] = 0;
        }
    }
}

static double* alloc_live(ctx_t* c)
{
    c->live += c->s;
    if (c->live > c->peak)
        c->peak = c->live;
    return (double*)malloc(sizeof(double) * 2 * (size_t)c->s);
}

static void free_live(ctx_t* c, double* p)
{
    c->live -= c->s;
    free(p);
}

/* engine_split.cpp:61-100, with the partition restriction for depth < q */
static void branch(ctx_t* c, double* t, int depth, uint32_t b)
{
    const int d = c->d;
    if (depth > 0) {
        fft_axis(d, c->levels, t, depth - 1, 0);
        c->fwd++;
    }
    if (depth < d) {
        const uint32_t odd_id = b | (1u << depth);
        if (depth < c->q) {
            const int take_odd = (c->part >> depth) & 1;
            if (!take_odd) {
                branch(c, t, depth + 1, b);
                merge_loop(c, t, NULL, depth);
            } else {
                phase_inplace(d, c->levels, t, depth, 0);
                branch(c, t, depth + 1, odd_id);
                double* tmp = alloc_live(c);
                memcpy(tmp, t, sizeof(double) * 2 * (size_t)c->s);
                memset(t, 0, sizeof(double) * 2 * (size_t)c->s);
                merge_loop(c, t, tmp, depth);
                free_live(c, tmp);
            }
        } else {
            double* child = alloc_live(c);
            memcpy(child, t, sizeof(double) * 2 * (size_t)c->s);
            phase_inplace(d, c->levels, child, depth, 0);
            c->phase += c->s;
            branch(c, t, depth + 1, b);
            branch(c, child, depth + 1, odd_id);
            merge_loop(c, t, child, depth);
            c->phase += c->s;
            free_live(c, child);
        }
    } else {
        multiply_into(c, t, b);
        c->diag += c->s;
    }
    if (depth > 0) {
        fft_axis(d, c->levels, t, depth - 1, 1);
        c->inv++;
    }
}

static int run_split(int d, const int64_t* levels, const double* blocks, int compressed,
                     const int* axis_sign, const double* v, double* y, int part, int nparts,
                     int64_t* counters)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    if (!blocks || !v || !y)
        return ORC_EINVAL;
    if (compressed)
        for (int a = 0; a < d; ++a)
            if (!axis_sign || axis_sign[a] == 0)
                return ORC_ESYM;
    int q = 0;
    while ((1 << q) < nparts)
        ++q;
    if ((1 << q) != nparts || q > d || part < 0 || part >= nparts)
        return ORC_EINVAL;
    ctx_t c;
    memset(&c, 0, sizeof(c));
    c.d = d;
    c.levels = levels;
    c.s = volume(d, levels);
    c.compressed = compressed;
    c.axis_sign = axis_sign;
    c.part = part;
    c.q = q;
    const uint32_t nb = 1u << d;
    const double** ptrs = (const double**)malloc(sizeof(double*) * nb);
    const double* p = blocks;
    int64_t shp[32];
    for (uint32_t b = 0; b < nb; ++b) {
        ptrs[b] = p;
        block_shape(d, levels, b, compressed, shp);
        p += 2 * volume(d, shp);
    }
    c.blocks = ptrs;
    c.live = c.s; /* y = v.clone() (engine_split.cpp:120) */
    c.peak = c.s;
    memcpy(y, v, sizeof(double) * 2 * (size_t)c.s);
    branch(&c, y, 0, 0);
    free(ptrs);
    if (counters) {
        counters[0] = c.fwd;
        counters[1] = c.inv;
        counters[2] = c.diag;
        counters[3] = c.phase;
        counters[4] = c.peak;
    }
    return ORC_OK;
}

int orc_split_apply(int d, const int64_t* levels, const double* blocks, int compressed,
                    const int* axis_sign, const double* v, double* y, int64_t* counters)
{
    return run_split(d, levels, blocks, compressed, axis_sign, v, y, 0, 1, counters);
}

int orc_split_apply_partial(int d, const int64_t* levels, const double* blocks, int compressed,
                            const int* axis_sign, const double* v, double* y, int part, int nparts)
{
    return run_split(d, levels, blocks, compressed, axis_sign, v, y, part, nparts, NULL);
}

/* engine_embed.cpp:113-168 with the full (2n)^d symbol */
int orc_embed_apply(int d, const int64_t* levels, const double* lags, double s0_re, double s0_im,
                    const double* v, double* y)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    int64_t eshape[32];
    for (int a = 0; a < d; ++a)
        eshape[a] = 2 * levels[a];
    const int64_t es = volume(d, eshape);
    double* sym = (double*)malloc(sizeof(double) * 2 * (size_t)es);
    double* work = (double*)calloc(2 * (size_t)es, sizeof(double));
    orc_embed_generator(d, levels, lags, s0_re, s0_im, sym);
    for (int a = 0; a < d; ++a)
        fft_axis(d, eshape, sym, a, 0);
    /* embed_corner (tensor.cpp) */
    const int64_t s = volume(d, levels);
    int64_t idx[32] = {0};
    for (int64_t i = 0; i < s; ++i) {
        int64_t off = 0;
        for (int a = 0; a < d; ++a)
            off = off * eshape[a] + idx[a];
        work[2 * off] = v[2 * i];
        work[2 * off + 1] = v[2 * i + 1];
        for (int a = d - 1; a >= 0; --a) {
            if (++idx[a] < levels[a])
                break;
            idx[a] = 0;
        }
    }
    for (int a = 0; a < d; ++a)
        fft_axis(d, eshape, work, a, 0);
    for (int64_t i = 0; i < es; ++i) {
        const double a = work[2 * i], b = work[2 * i + 1];
        cmul(a, b, sym[2 * i], sym[2 * i + 1], &work[2 * i], &work[2 * i + 1]);
    }
    for (int a = 0; a < d; ++a)
        fft_axis(d, eshape, work, a, 1);
    memset(idx, 0, sizeof(idx));
    for (int64_t i = 0; i < s; ++i) {
        int64_t off = 0;
        for (int a = 0; a < d; ++a)
            off = off * eshape[a] + idx[a];
        y[2 * i] = work[2 * off];
        y[2 * i + 1] = work[2 * off + 1];
        for (int a = d - 1; a >= 0; --a) {
            if (++idx[a] < levels[a])
                break;
            idx[a] = 0;
        }
    }
    free(work);
    free(sym);
    return ORC_OK;
}

/* engine_embed.cpp:190-227 */
int orc_naive_matvec(int d, const int64_t* levels, const double* lags, const double* v, double* y,
                     int64_t cap)
{
    int st = check_levels(d, levels);
    if (st)
        return st;
    const int64_t s = volume(d, levels);
    if (s > cap)
        return ORC_ECAP;
    int64_t jdx[32] = {0};
    for (int64_t j = 0; j < s; ++j) {
        double ar = 0.0, ai = 0.0;
        int64_t kdx[32] = {0};
        for (int64_t k = 0; k < s; ++k) {
            int64_t lag_off = 0;
            for (int a = 0; a < d; ++a) {
                const int64_t n = levels[a];
                lag_off = lag_off * (2 * n - 1) + (jdx[a] - kdx[a] + n - 1);
            }
            double pr, pi;
            cmul(lags[2 * lag_off], lags[2 * lag_off + 1], v[2 * k], v[2 * k + 1], &pr, &pi);
            ar += pr;
            ai += pi;
            for (int a = d - 1; a >= 0; --a) {
                if (++kdx[a] < levels[a])
                    break;
                kdx[a] = 0;
            }
        }
        y[2 * j] = ar;
        y[2 * j + 1] = ai;
        for (int a = d - 1; a >= 0; --a) {
            if (++jdx[a] < levels[a])
                break;
            jdx[a] = 0;
        }
    }
    return ORC_OK;
}

/* analysis.cpp:21-56: {d, n, s, c_embed, c_split, r_c, r_c_asym, r_m, r_m_sym} */
int orc_predict(int d, double n, double out[9])
{
    if (d < 1 || n < 2.0)
        return ORC_EINVAL;
    const double s = pow(n, d), p = pow(2.0, d);
    out[0] = d;
    out[1] = n;
    out[2] = s;
    out[3] = 2.0 * p * s * log2(p * s) + p * s;
    out[4] = 2.0 * (p - 1.0) * s * (2.0 * log2(n) + 1.0) + p * s;
    out[5] = (d * log2(2.0 * n) + 1.0) / ((1.0 - 1.0 / p) * (2.0 * log2(n) + 1.0) + 1.0);
    out[6] = d / (2.0 - pow(2.0, -d + 1));
    out[7] = 2.0 / ((d + 1.0) / p + 1.0);
    out[8] = (p + 1.0) / (d + 2.0);
    return ORC_OK;
}
