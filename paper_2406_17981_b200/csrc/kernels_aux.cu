// Setup-side and auxiliary sm_100a kernels: device spectra precompute
// (embedding, branchwise fold, mirror validation and compression, precision
// conversion) and the full-embedding engine pieces. All HBM-bound
// element-wise sweeps; one thread per output element, grid-stride.
//
// Reference behaviour (paths relative to /root/reference/proj):
//   embed_generator  src/core/kernel.cpp:50-82
//   fold_axis        src/core/kernel.cpp:223-258
//   compress_spectra src/core/kernel.cpp:325-390
//   EmbedOperator    src/core/engine_embed.cpp:113-168
#include <cuda_runtime.h>

#include "tsk_common.cuh"

namespace tsk {

struct Shape32 {
    int32_t d;
    int64_t n[TSK_MAX_D];
};

static Shape32 make_shape(int32_t d, const int64_t* levels, int64_t mul = 1)
{
    Shape32 s;
    s.d = d;
    for (int a = 0; a < d; ++a)
        s.n[a] = levels[a] * mul;
    return s;
}

static int64_t vol(const Shape32& s)
{
    int64_t v = 1;
    for (int a = 0; a < s.d; ++a)
        v *= s.n[a];
    return v;
}

static unsigned grid1d(int64_t total)
{
    const int64_t b = (total + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

#define GRID_STRIDE(i, total) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (total); \
         i += (int64_t)gridDim.x * blockDim.x)

// Value of the embedded first column at embedded index off of the (2n)^d
// layout: per axis j < n -> lag j, j == n -> s0 (padding), j > n -> lag j-2n
// (ref kernel.cpp:50-82). Two sources: an explicit lag tensor and the
// analytic dyadic G of BASELINE.json configs[1].
struct LagSource {
    const double2* __restrict__ lags;
    double2 s0;
    __device__ __forceinline__ double2 at(const Shape32& lv, int64_t off) const
    {
        int64_t rem = off;
        int64_t lag_off = 0, lag_stride = 1;
        bool pad = false;
        for (int a = lv.d - 1; a >= 0; --a) {
            const int64_t n = lv.n[a];
            const int64_t j = rem % (2 * n);
            rem /= 2 * n;
            if (j == n)
                pad = true;
            const int64_t m = j < n ? j : j - 2 * n;
            lag_off += (m + n - 1) * lag_stride;
            lag_stride *= 2 * n - 1;
        }
        return pad ? s0 : lags[lag_off];
    }
};

// same formula as oracle/toesplit_oracle.c:orc_dyadic_lags (rh_i rh_j formed
// as m_i m_j / r^2, so mirrored lags are bit-exact)
struct DyadicSource {
    int ci, cj;
    double k;
    double2 self, s0;
    __device__ __forceinline__ double2 at(const Shape32& lv, int64_t off) const
    {
        int64_t rem = off;
        bool pad = false;
        double r2 = 0.0, mi = 0.0, mj = 0.0;
        for (int a = lv.d - 1; a >= 0; --a) {
            const int64_t n = lv.n[a];
            const int64_t j = rem % (2 * n);
            rem /= 2 * n;
            if (j == n)
                pad = true;
            const double m = (double)(j < n ? j : j - 2 * n);
            r2 += m * m;
            if (a == ci)
                mi = m;
            if (a == cj)
                mj = m;
        }
        double2 v;
        const double delta = ci == cj ? 1.0 : 0.0;
        if (pad) {
            v = s0;
        } else if (r2 == 0.0) {
            v.x = delta * self.x;
            v.y = delta * self.y;
        } else {
            const double rr = mi * mj / r2;
            const double r = sqrt(r2);
            double s, c;
            sincos(k * r, &s, &c);
            const double amp = (delta - rr) / r + (delta - 3.0 * rr) / (k * k * r2 * r);
            v.x = amp * c;
            v.y = amp * s;
        }
        return v;
    }
};

template <class Src>
__global__ void k_embed(Shape32 lv, Src src, double2* __restrict__ out, int64_t total)
{
    GRID_STRIDE(off, total)
    out[off] = src.at(lv, off);
}

// Embedding and the first branchwise fold (axis 0, ref kernel.cpp:223-258)
// in one sweep: out[k0, ...] = lo + hi (even) or e^{-i pi k0/n0} (lo - hi)
// (odd) with lo / hi the embedded values at k0 and k0 + n0, evaluated on the
// fly — the (2n)^d embedding is never materialised (half the setup memory).
// Same operations in the same order as k_embed + k_fold_axis: bit-identical.
template <class Src>
__global__ void k_embed_fold0(Shape32 lv, Src src, int odd, double2* __restrict__ out, int64_t total_out)
{
    const int64_t n = lv.n[0];
    int64_t inner = 1;
    for (int a = 1; a < lv.d; ++a)
        inner *= 2 * lv.n[a];
    GRID_STRIDE(off, total_out)
    {
        const int64_t i = off % inner;
        const int64_t k = off / inner;
        const double2 lo = src.at(lv, k * inner + i);
        const double2 hi = src.at(lv, (n + k) * inner + i);
        double2 r;
        if (odd) {
            double s, c;
            sincospi(-(double)k / (double)n, &s, &c);
            double2 dd;
            dd.x = lo.x - hi.x;
            dd.y = lo.y - hi.y;
            double2 f;
            f.x = c;
            f.y = s;
            r = cmul(f, dd);
        } else {
            r.x = lo.x + hi.x;
            r.y = lo.y + hi.y;
        }
        out[off] = r;
    }
}

// small integers are exact, so the sum is order independent.

__global__ void k_fold_axis(Shape32 in_shape, int axis, int odd, const double2* __restrict__ in,
                            double2* __restrict__ out, int64_t total_out)
{
    const int64_t n = in_shape.n[axis] / 2;
    int64_t inner = 1;
    for (int a = axis + 1; a < in_shape.d; ++a)
        inner *= in_shape.n[a];
    GRID_STRIDE(off, total_out)
    {
        const int64_t i = off % inner;
        const int64_t t = off / inner;
        const int64_t k = t % n;
        const int64_t o = t / n;
        const double2 lo = in[(o * 2 * n + k) * inner + i];
        const double2 hi = in[(o * 2 * n + n + k) * inner + i];
        double2 r;
        if (odd) {
            double s, c;
            sincospi(-(double)k / (double)n, &s, &c);
            double2 dd;
            dd.x = lo.x - hi.x;
            dd.y = lo.y - hi.y;
            double2 f;
            f.x = c;
            f.y = s;
            r = cmul(f, dd);
        } else {
            r.x = lo.x + hi.x;
            r.y = lo.y + hi.y;
        }
        out[off] = r;
    }
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v)
{
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

__global__ void k_mirror_check(Shape32 lv, uint32_t bits, uint32_t skew_mask,
                               const double2* __restrict__ blk, double* out2, int64_t total)
{
    double mabs = 0.0, mdiff = 0.0;
    GRID_STRIDE(off, total)
    {
        const double2 v = blk[off];
        mabs = fmax(mabs, hypot(v.x, v.y));
        int64_t stride = 1;
        int64_t rem = off;
        for (int a = lv.d - 1; a >= 0; --a) {
            const int64_t n = lv.n[a];
            const int64_t k = rem % n;
            rem /= n;
            const int64_t mk = ((bits >> a) & 1u) ? n - 1 - k : (n - k) % n;
            const double2 w = blk[off + (mk - k) * stride];
            const double sg = ((skew_mask >> a) & 1u) ? -1.0 : 1.0;
            mdiff = fmax(mdiff, hypot(v.x - sg * w.x, v.y - sg * w.y));
            stride *= n;
        }
    }
    // warp reduce, then one atomic per warp (max is order independent)
    for (int o = 16; o > 0; o >>= 1) {
        mabs = fmax(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
        mdiff = fmax(mdiff, __shfl_xor_sync(0xffffffffu, mdiff, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_nonneg(out2, mabs);
        atomic_max_nonneg(out2 + 1, mdiff);
    }
}

template <typename TO>
__device__ __forceinline__ void put(TO* dst, int64_t i, double2 v);
template <>
__device__ __forceinline__ void put<double2>(double2* dst, int64_t i, double2 v)
{
    dst[i] = v;
}
template <>
__device__ __forceinline__ void put<float2>(float2* dst, int64_t i, double2 v)
{
    dst[i] = make_float2((float)v.x, (float)v.y);
}

template <typename TO>
__global__ void k_store_block(Shape32 lv, uint32_t bits, int compressed,
                              const double2* __restrict__ blk, TO* __restrict__ dst, int64_t total)
{
    GRID_STRIDE(off, total)
    {
        int64_t rem = off, src = 0, stride = 1;
        for (int a = lv.d - 1; a >= 0; --a) {
            const int64_t st = compressed ? stored_len(lv.n[a], (bits >> a) & 1u) : lv.n[a];
            const int64_t k = rem % st;
            rem /= st;
            src += k * stride;
            stride *= lv.n[a];
        }
        put<TO>(dst, off, blk[src]);
    }
}

__global__ void k_c128_to_c64(const double2* __restrict__ s, float2* __restrict__ d, int64_t n)
{
    GRID_STRIDE(i, n) d[i] = make_float2((float)s[i].x, (float)s[i].y);
}

__global__ void k_c64_to_c128(const float2* __restrict__ s, double2* __restrict__ d, int64_t n)
{
    GRID_STRIDE(i, n) d[i] = make_double2((double)s[i].x, (double)s[i].y);
}

// pad (extract == 0): dst[(2n)^d] = corner(src[n^d]) with zeros elsewhere;
// extract: dst[n^d] = corner of src[(2n)^d]. One thread per big-tensor element.
template <typename T2, typename I = int64_t>
__global__ void k_embed_corner(Shape32 lv, const T2* __restrict__ src, T2* __restrict__ dst,
                               int extract, int64_t total_big)
{
    GRID_STRIDE(off, total_big)
    {
        I rem = (I)off, small = 0, sstride = 1;  // I = 32-bit when the grid fits
        bool inside = true;
        for (int a = lv.d - 1; a >= 0; --a) {
            const I n = (I)lv.n[a];
            const I j = rem % (2 * n);
            rem /= 2 * n;
            if (j >= n)
                inside = false;
            small += j * sstride;
            sstride *= n;
        }
        if (extract) {
            if (inside)
                dst[small] = src[off];
        } else {
            T2 z;
            z.x = 0;
            z.y = 0;
            dst[off] = inside ? src[small] : z;
        }
    }
}

// work[(2n)^d] *= symbol, full or (n+1)^d mirror corner (ref
// engine_embed.cpp:14-35,136-147: f_l = +-f_{2n-l} for l > n)
template <typename T2>
__global__ void k_symbol_multiply(Shape32 lv, T2* __restrict__ work, const T2* __restrict__ sym,
                                  int corner, int skew, int64_t total)
{
    GRID_STRIDE(off, total)
    {
        int64_t idx = off;
        bool neg = false;
        if (corner) {
            int64_t rem = off, cs = 1;
            idx = 0;
            for (int a = lv.d - 1; a >= 0; --a) {
                const int64_t n = lv.n[a];
                const int64_t l = rem % (2 * n);
                rem /= 2 * n;
                int64_t src = l;
                if (l > n) {
                    src = 2 * n - l;
                    if (skew)
                        neg = !neg;
                }
                idx += src * cs;
                cs *= n + 1;
            }
        }
        T2 s = sym[idx];
        if (neg) {
            s.x = -s.x;
            s.y = -s.y;
        }
        work[off] = cmul(work[off], s);
    }
}

template <typename T2, typename I>
__global__ void k_block_symbol(Shape32 lv, T2* __restrict__ work, int64_t cstride, tsk_block_symbol bs,
                               int64_t total)
{
    const T2* sym = static_cast<const T2*>(bs.data);
    GRID_STRIDE(off, total)
    {
        int64_t idx = off;
        uint32_t mir = 0;  // axes read through the mirror
        if (bs.corner) {
            I rem = (I)off, cs = 1, acc = 0;  // I = 32-bit when the grid fits
            for (int a = lv.d - 1; a >= 0; --a) {
                const I n = (I)lv.n[a];
                const I l = rem % (2 * n);
                rem /= 2 * n;
                I src = l;
                if (l > n) {
                    src = 2 * n - l;
                    mir |= 1u << a;
                }
                acc += src * cs;
                cs *= n + 1;
            }
            idx = (int64_t)acc;
        }
        T2 xv[TSK_MAX_M];
        for (int c = 0; c < bs.m; ++c)
            xv[c] = work[c * cstride + off];
        for (int c = 0; c < bs.m; ++c) {
            T2 acc;
            acc.x = 0;
            acc.y = 0;
            for (int c2 = 0; c2 < bs.m; ++c2) {
                const int u = bs.comp_map[c * bs.m + c2];
                T2 sv = sym[u * bs.block_elems + idx];
                if (__popc(mir & bs.skew_mask[u]) & 1) {
                    sv.x = -sv.x;
                    sv.y = -sv.y;
                }
                const T2 p = cmul(sv, xv[c2]);
                acc.x += p.x;
                acc.y += p.y;
            }
            work[c * cstride + off] = acc;
        }
    }
}


// As k_block_symbol, one row of the last axis per block iteration.
__global__ void k_block_symbol_rows(Shape32 lv, float2* __restrict__ work, int64_t cstride, tsk_block_symbol bs,
                                    int64_t rows)
{
    const float2* sym = static_cast<const float2*>(bs.data);
    const int d = lv.d;
    const int64_t nl = lv.n[d - 1], L = 2 * nl;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        // outer axes: row-uniform corner offset and mirror mask
        int64_t rem = row, srow = 0, cs = 1;
        uint32_t mir_row = 0;
        for (int a = d - 2; a >= 0; --a) {
            const int64_t n = lv.n[a];
            const int64_t l = rem % (2 * n);
            rem /= 2 * n;
            int64_t src = l;
            if (l > n) {
                src = 2 * n - l;
                mir_row |= 1u << a;
            }
            srow += src * cs;
            cs *= n + 1;
        }
        for (int64_t j = threadIdx.x; j < L; j += blockDim.x) {
            const int64_t off = row * L + j;
            int64_t idx = off;
            uint32_t mir = 0;
            if (bs.corner) {
                const int64_t jj = j > nl ? L - j : j;
                idx = srow * (nl + 1) + jj;
                mir = mir_row | (j > nl ? 1u << (d - 1) : 0u);
            }
            float2 xv[TSK_MAX_M];
            for (int c = 0; c < bs.m; ++c)
                xv[c] = work[c * cstride + off];
            for (int c = 0; c < bs.m; ++c) {
                float2 acc = make_float2(0.f, 0.f);
                for (int c2 = 0; c2 < bs.m; ++c2) {
                    const int u = bs.comp_map[c * bs.m + c2];
                    float2 sv = sym[u * bs.block_elems + idx];
                    if (__popc(mir & bs.skew_mask[u]) & 1) {
                        sv.x = -sv.x;
                        sv.y = -sv.y;
                    }
                    const float2 p = cmul(sv, xv[c2]);
                    acc.x += p.x;
                    acc.y += p.y;
                }
                work[c * cstride + off] = acc;
            }
        }
    }
}
}  // namespace tsk

using namespace tsk;

extern "C" {

int tsk_embed_generator(int32_t d, const int64_t* levels, const void* lags, double s0_re,
                        double s0_im, void* out, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    const int64_t total = vol(lv) << d;
    k_embed<<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(
        lv, LagSource{(const double2*)lags, make_double2(s0_re, s0_im)}, (double2*)out, total);
    return (int)cudaGetLastError();
}

int tsk_embed_dyadic(int32_t d, const int64_t* levels, int32_t i, int32_t j, double k,
                     double self_re, double self_im, double s0_re, double s0_im, void* out,
                     void* stream)
{
    Shape32 lv = make_shape(d, levels);
    const int64_t total = vol(lv) << d;
    k_embed<<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(
        lv, DyadicSource{i, j, k, make_double2(self_re, self_im), make_double2(s0_re, s0_im)},
        (double2*)out, total);
    return (int)cudaGetLastError();
}

int tsk_embed_fold0(int32_t d, const int64_t* levels, const void* lags, int32_t dyadic_i, int32_t dyadic_j,
                    double k, double self_re, double self_im, double s0_re, double s0_im, int32_t odd,
                    void* out, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    const int64_t total_out = vol(lv) << (d - 1);
    const double2 s0 = make_double2(s0_re, s0_im);
    if (lags)
        k_embed_fold0<<<grid1d(total_out), 256, 0, (cudaStream_t)stream>>>(
            lv, LagSource{(const double2*)lags, s0}, odd, (double2*)out, total_out);
    else
        k_embed_fold0<<<grid1d(total_out), 256, 0, (cudaStream_t)stream>>>(
            lv, DyadicSource{dyadic_i, dyadic_j, k, make_double2(self_re, self_im), s0}, odd,
            (double2*)out, total_out);
    return (int)cudaGetLastError();
}

int tsk_fold_axis(int32_t d, const int64_t* shape, int32_t axis, int32_t odd, const void* in,
                  void* out, void* stream)
{
    Shape32 s = make_shape(d, shape);
    const int64_t total_out = vol(s) / 2;
    k_fold_axis<<<grid1d(total_out), 256, 0, (cudaStream_t)stream>>>(
        s, axis, odd, (const double2*)in, (double2*)out, total_out);
    return (int)cudaGetLastError();
}

int tsk_mirror_check(int32_t d, const int64_t* levels, uint32_t branch_bits, uint32_t skew_mask,
                     const void* block, double* out2, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    const int64_t total = vol(lv);
    cudaMemsetAsync(out2, 0, 2 * sizeof(double), (cudaStream_t)stream);
    k_mirror_check<<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(
        lv, branch_bits, skew_mask, (const double2*)block, out2, total);
    return (int)cudaGetLastError();
}

int tsk_store_block(int32_t d, const int64_t* levels, uint32_t branch_bits, int32_t compressed,
                    const void* block, void* dst, int32_t prec, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    int64_t total = 1;
    for (int a = 0; a < d; ++a)
        total *= compressed ? stored_len(levels[a], (branch_bits >> a) & 1u) : levels[a];
    if (prec)
        k_store_block<float2><<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(
            lv, branch_bits, compressed, (const double2*)block, (float2*)dst, total);
    else
        k_store_block<double2><<<grid1d(total), 256, 0, (cudaStream_t)stream>>>(
            lv, branch_bits, compressed, (const double2*)block, (double2*)dst, total);
    return (int)cudaGetLastError();
}

int tsk_block_symbol_multiply(int32_t d, const int64_t* levels, int32_t prec, void* work, int64_t cstride,
                              const tsk_block_symbol* sym, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    if (prec && d >= 2 && 2 * levels[d - 1] <= 4096) {
        // row-wise: the outer-axis mirror bookkeeping once per row (block),
        // the last axis across the threads (coalesced reads of x and symbol)
        int64_t rows = 1;
        for (int a = 0; a < d - 1; ++a)
            rows *= 2 * levels[a];
        const unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 64);
        tsk::k_block_symbol_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(lv, (float2*)work, cstride, *sym, rows);
        return (int)cudaGetLastError();
    }
    const int64_t total = vol(lv) << d;
    auto st = (cudaStream_t)stream;
    const bool i32 = total < (int64_t(1) << 31);
    if (prec && i32)
        tsk::k_block_symbol<float2, int32_t><<<grid1d(total), 256, 0, st>>>(lv, (float2*)work, cstride, *sym, total);
    else if (prec)
        tsk::k_block_symbol<float2, int64_t><<<grid1d(total), 256, 0, st>>>(lv, (float2*)work, cstride, *sym, total);
    else if (i32)
        tsk::k_block_symbol<double2, int32_t><<<grid1d(total), 256, 0, st>>>(lv, (double2*)work, cstride, *sym,
                                                                            total);
    else
        tsk::k_block_symbol<double2, int64_t><<<grid1d(total), 256, 0, st>>>(lv, (double2*)work, cstride, *sym,
                                                                            total);
    return (int)cudaGetLastError();
}

int tsk_convert(const void* src, int32_t src_prec, void* dst, int32_t dst_prec, int64_t count,
                void* stream)
{
    auto st = (cudaStream_t)stream;
    if (src_prec == dst_prec)
        return (int)cudaMemcpyAsync(dst, src, (size_t)count * (src_prec ? 8 : 16),
                                    cudaMemcpyDeviceToDevice, st);
    if (src_prec == 0)
        k_c128_to_c64<<<grid1d(count), 256, 0, st>>>((const double2*)src, (float2*)dst, count);
    else
        k_c64_to_c128<<<grid1d(count), 256, 0, st>>>((const float2*)src, (double2*)dst, count);
    return (int)cudaGetLastError();
}

int tsk_embed_corner(int32_t d, const int64_t* levels, int32_t prec, const void* src, void* dst,
                     int32_t extract, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    int64_t total = 1;
    for (int a = 0; a < d; ++a)
        total *= 2 * levels[a];
    auto st = (cudaStream_t)stream;
    const bool i32 = total < (int64_t(1) << 31);
    if (prec && i32)
        k_embed_corner<float2, int32_t><<<grid1d(total), 256, 0, st>>>(lv, (const float2*)src, (float2*)dst,
                                                                       extract, total);
    else if (prec)
        k_embed_corner<float2><<<grid1d(total), 256, 0, st>>>(lv, (const float2*)src,
                                                              (float2*)dst, extract, total);
    else if (i32)
        k_embed_corner<double2, int32_t><<<grid1d(total), 256, 0, st>>>(lv, (const double2*)src, (double2*)dst,
                                                                        extract, total);
    else
        k_embed_corner<double2><<<grid1d(total), 256, 0, st>>>(lv, (const double2*)src,
                                                               (double2*)dst, extract, total);
    return (int)cudaGetLastError();
}

int tsk_symbol_multiply(int32_t d, const int64_t* levels, int32_t prec, void* work,
                        const void* symbol, int32_t corner, int32_t skew, void* stream)
{
    Shape32 lv = make_shape(d, levels);
    int64_t total = 1;
    for (int a = 0; a < d; ++a)
        total *= 2 * levels[a];
    auto st = (cudaStream_t)stream;
    if (prec)
        k_symbol_multiply<float2><<<grid1d(total), 256, 0, st>>>(
            lv, (float2*)work, (const float2*)symbol, corner, skew, total);
    else
        k_symbol_multiply<double2><<<grid1d(total), 256, 0, st>>>(
            lv, (double2*)work, (const double2*)symbol, corner, skew, total);
    return (int)cudaGetLastError();
}

}  // extern "C"
