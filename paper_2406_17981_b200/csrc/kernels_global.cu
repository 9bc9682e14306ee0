// Long-axis passes: the same three operations as the tiled kernels (forward
// split, inverse merge, leaf pair) for axes too long to stage a fiber tile in
// shared memory (kernels_generic.cu covers n up to ~1.4k-4k depending on
// precision and block size; the reference accepts any n). Every Stockham stage
// is one launch over global memory (one butterfly per thread, ping-pong
// buffers from the stream-ordered pool), phases / merges / the leaf multiply
// are elementwise launches. Correctness path: no shape the reference accepts is
// refused for being long.
//
// Reference behaviour mirrored (paths relative to /root/reference/proj):
//   forward DFT kernel exp(-2 pi i lk/N), inverse with 1/N  src/core/fft.hpp:7-10
//   split phase P_k = exp(-i pi k/n)                        src/core/tensor.cpp:227-254
//   merge  even = (even + exp(+i pi k/n) odd)/2             src/core/engine_split.cpp:13-37
//   leaf multiply, full / mirror remap                      src/core/kernel.cpp:126-219
#include <cuda_runtime.h>

#include <cstdint>

#include "tsk_common.cuh"

namespace tsk {
namespace glob {

__device__ __forceinline__ int64_t gidx(const tsk_axis& p, int64_t c, int64_t o, int64_t k, int64_t i)
{
    return c * p.cstride + (o * p.n + k) * p.inner + i;
}

// One Stockham stage (radix R, stride ns) for every fiber: thread per butterfly.
template <typename T, int R, bool INV>
__global__ void __launch_bounds__(256) k_pass(tsk_axis p, const typename cx<T>::t* __restrict__ in,
                                              typename cx<T>::t* __restrict__ out, int64_t ns)
{
    using T2 = typename cx<T>::t;
    const int64_t n = p.n, m = n / R, tstep = n / (ns * R);
    const int64_t total = p.ncomp * p.outer * p.inner * m;
    const T2* __restrict__ roots = static_cast<const T2*>(p.roots);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        // i fastest (coalesced for strided axes), then j, o, c
        const int64_t i = t % p.inner;
        int64_t r_ = t / p.inner;
        const int64_t j = r_ % m;
        r_ /= m;
        const int64_t o = r_ % p.outer;
        const int64_t c = r_ / p.outer;
        const int64_t jm = j % ns;
        T2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
            v[r] = in[gidx(p, c, o, j + r * m, i)];
        if (jm > 0) {
#pragma unroll
            for (int r = 1; r < R; ++r)
                v[r] = cmul(v[r], twiddle<T, INV>(roots, (int)((r * jm * tstep) % n)));
        }
        dft_small<T, R, INV>(v, roots, (int)m);
        const int64_t base = (j - jm) * R + jm;
#pragma unroll
        for (int q = 0; q < R; ++q)
            out[gidx(p, c, o, base + q * ns, i)] = v[q];
    }
}

// Direct stage for a prime radix > 8: thread per output.
template <typename T, bool INV>
__global__ void __launch_bounds__(256) k_pass_direct(tsk_axis p, const typename cx<T>::t* __restrict__ in,
                                                     typename cx<T>::t* __restrict__ out, int64_t ns, int R)
{
    using T2 = typename cx<T>::t;
    const int64_t n = p.n, m = n / R, tstep = n / (ns * R);
    const int64_t total = p.ncomp * p.outer * p.inner * n;
    const T2* __restrict__ roots = static_cast<const T2*>(p.roots);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % p.inner;
        int64_t r_ = t / p.inner;
        const int64_t rem = r_ % n;
        r_ /= n;
        const int64_t o = r_ % p.outer;
        const int64_t c = r_ / p.outer;
        const int64_t q = rem / m, j = rem - q * m, jm = j % ns;
        T2 acc = make_c<T>(0, 0);
        for (int r = 0; r < R; ++r) {
            T2 xv = in[gidx(p, c, o, j + r * m, i)];
            if (jm > 0 && r > 0)
                xv = cmul(xv, twiddle<T, INV>(roots, (int)((r * jm * tstep) % n)));
            acc = cadd(acc, cmul(xv, twiddle<T, INV>(roots, (int)(((r * q) % R) * m))));
        }
        out[gidx(p, c, o, (j - jm) * R + jm + q * ns, i)] = acc;
    }
}

// dst = src * P_k (split phase along the axis)
template <typename T>
__global__ void __launch_bounds__(256) k_phase(tsk_axis p, const typename cx<T>::t* __restrict__ src,
                                               typename cx<T>::t* __restrict__ dst)
{
    using T2 = typename cx<T>::t;
    const T2* __restrict__ phase = static_cast<const T2*>(p.phase);
    const int64_t total = p.ncomp * p.outer * p.n * p.inner;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % p.inner;
        int64_t r_ = t / p.inner;
        const int64_t k = r_ % p.n;
        r_ /= p.n;
        const int64_t o = r_ % p.outer, c = r_ / p.outer;
        const int64_t a = gidx(p, c, o, k, i);
        dst[a] = cmul(src[a], phase[k]);
    }
}

// dst = scale (e + conj(P_k) o); either input may be absent
template <typename T>
__global__ void __launch_bounds__(256) k_merge(tsk_axis p, const typename cx<T>::t* e, const typename cx<T>::t* o_,
                                               typename cx<T>::t* dst)
{
    using T2 = typename cx<T>::t;
    const T2* __restrict__ phase = static_cast<const T2*>(p.phase);
    const T scale = (T)p.scale;
    const int64_t total = p.ncomp * p.outer * p.n * p.inner;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % p.inner;
        int64_t r_ = t / p.inner;
        const int64_t k = r_ % p.n;
        r_ /= p.n;
        const int64_t o = r_ % p.outer, c = r_ / p.outer;
        const int64_t a = gidx(p, c, o, k, i);
        T2 acc = make_c<T>(0, 0);
        if (e)
            acc = e[a];
        if (o_)
            acc = cadd(acc, cmulc(o_[a], phase[k]));
        dst[a] = make_c<T>(scale * acc.x, scale * acc.y);
    }
}

// y_i = sum_j T[b](map(i,j)) x_j at every (fiber, k) of the leaf axis, in place
// (ref kernel.cpp:126-219; the mirror remap as in kernels_generic.cu)
template <typename T>
__global__ void __launch_bounds__(256) k_leaf_mul(tsk_axis p, tsk_spectra sp, int beta, typename cx<T>::t* buf)
{
    using T2 = typename cx<T>::t;
    const T2* __restrict__ spec = static_cast<const T2*>(sp.data) + sp.branch_base[beta];
    const int64_t bstride = sp.block_elems[beta];
    const int m = sp.m, d = sp.d;
    const uint32_t bits = sp.branch_bits[beta];
    const int odd_last = (bits >> (d - 1)) & 1u;
    const int64_t n = p.n;
    const int64_t total = p.outer * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t % n, g = t / n;
        int64_t idx = 0;
        uint32_t neg = 0;
        if (!sp.compressed) {
            idx = g * n + k;
        } else {
            int64_t gg = g;
            int64_t stride = stored_len(n, odd_last);
            for (int a = d - 2; a >= 0; --a) {
                const int64_t na = sp.levels[a];
                const int64_t ka = gg % na;
                gg /= na;
                const int odd = (bits >> a) & 1u;
                bool mirrored;
                idx += mirror_src(na, odd, ka, mirrored) * stride;
                stride *= stored_len(na, odd);
                if (mirrored)
                    for (int u = 0; u < sp.n_unique; ++u)
                        neg ^= ((sp.skew_mask[u] >> a) & 1u) << u;
            }
            bool mirrored;
            idx += mirror_src(n, odd_last, k, mirrored);
            if (mirrored)
                for (int u = 0; u < sp.n_unique; ++u)
                    neg ^= ((sp.skew_mask[u] >> (d - 1)) & 1u) << u;
        }
        T2 x[TSK_MAX_M];
        for (int j = 0; j < m; ++j)
            x[j] = buf[gidx(p, j, g, k, 0)];
        for (int i = 0; i < m; ++i) {
            T2 acc = make_c<T>(0, 0);
            for (int j = 0; j < m; ++j) {
                const int u = sp.comp_map[i * m + j];
                T2 tv = ldg_c(spec + (int64_t)u * bstride + idx);
                if ((neg >> u) & 1u)
                    tv = make_c<T>(-tv.x, -tv.y);
                acc = cadd(acc, cmul(x[j], tv));
            }
            buf[gidx(p, i, g, k, 0)] = acc;
        }
    }
}

static int grid_for(int64_t work)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t blocks = (work + 255) / 256;
    return (int)(blocks < (int64_t)sms * 16 ? (blocks > 0 ? blocks : 1) : (int64_t)sms * 16);
}

// Stream-ordered scratch of one operand (ncomp component tensors).
struct Scratch {
    void* p = nullptr;
    cudaStream_t st;
    Scratch(size_t bytes, cudaStream_t s) : st(s) { cudaMallocAsync(&p, bytes, s); }
    ~Scratch()
    {
        if (p)
            cudaFreeAsync(p, st);
    }
};

template <typename T>
static size_t operand_bytes(const tsk_axis& a)
{
    // components at cstride apart (cstride may be 0 with a single component)
    const size_t one = (size_t)a.outer * (size_t)a.n * (size_t)a.inner;
    return ((size_t)(a.ncomp - 1) * (size_t)a.cstride + one) * sizeof(typename cx<T>::t);
}

// Mixed-radix FFT along the axis, in -> out (out may equal in), through the
// two scratch buffers.
template <typename T, bool INV>
static int fft(const tsk_axis& a, const void* in, void* out, void* s0, void* s1, cudaStream_t st)
{
    using T2 = typename cx<T>::t;
    const int64_t work_b = a.ncomp * a.outer * a.inner * a.n;
    const void* cur = in;
    int64_t ns = 1;
    for (int s = 0; s < a.nrad; ++s) {
        const int R = a.rad[s];
        void* next = (s == a.nrad - 1 && out != cur) ? out : (cur == s0 ? s1 : s0);
        const T2* ci = static_cast<const T2*>(cur);
        T2* no = static_cast<T2*>(next);
        const int g = grid_for(work_b / (R <= 8 ? R : 1));
        switch (R) {
        case 2: k_pass<T, 2, INV><<<g, 256, 0, st>>>(a, ci, no, ns); break;
        case 3: k_pass<T, 3, INV><<<g, 256, 0, st>>>(a, ci, no, ns); break;
        case 4: k_pass<T, 4, INV><<<g, 256, 0, st>>>(a, ci, no, ns); break;
        case 5: k_pass<T, 5, INV><<<g, 256, 0, st>>>(a, ci, no, ns); break;
        case 7: k_pass<T, 7, INV><<<g, 256, 0, st>>>(a, ci, no, ns); break;
        case 8: k_pass<T, 8, INV><<<g, 256, 0, st>>>(a, ci, no, ns); break;
        default: k_pass_direct<T, INV><<<g, 256, 0, st>>>(a, ci, no, ns, R); break;
        }
        if (int e = (int)cudaGetLastError())
            return e;
        cur = next;
        ns *= R;
    }
    if (cur != out)  // n = 1 (no stages) or the last stage could not land in place
        return (int)cudaMemcpyAsync(out, cur, operand_bytes<T>(a), cudaMemcpyDeviceToDevice, st);
    return 0;
}

template <typename T>
static int fwd_split(const tsk_axis& a, cudaStream_t st)
{
    const size_t b = operand_bytes<T>(a);
    Scratch s0(b, st), s1(b, st), t1(b, st);
    if (!s0.p || !s1.p || !t1.p)
        return (int)cudaErrorMemoryAllocation;
    using T2 = typename cx<T>::t;
    const int g = grid_for(a.ncomp * a.outer * a.n * a.inner);
    // odd first: the even child may be written over the input
    if (a.use_odd) {
        k_phase<T><<<g, 256, 0, st>>>(a, static_cast<const T2*>(a.src0), static_cast<T2*>(t1.p));
        if (int e = fft<T, false>(a, t1.p, a.dst1, s0.p, s1.p, st))
            return e;
    }
    if (a.use_even)
        if (int e = fft<T, false>(a, a.src0, a.dst0, s0.p, s1.p, st))
            return e;
    return (int)cudaGetLastError();
}

template <typename T>
static int inv_merge(const tsk_axis& a, cudaStream_t st)
{
    const size_t b = operand_bytes<T>(a);
    Scratch s0(b, st), s1(b, st), te(b, st), to(b, st);
    if (!s0.p || !s1.p || !te.p || !to.p)
        return (int)cudaErrorMemoryAllocation;
    using T2 = typename cx<T>::t;
    if (a.use_even)
        if (int e = fft<T, true>(a, a.src0, te.p, s0.p, s1.p, st))
            return e;
    if (a.use_odd)
        if (int e = fft<T, true>(a, a.src1, to.p, s0.p, s1.p, st))
            return e;
    k_merge<T><<<grid_for(a.ncomp * a.outer * a.n * a.inner), 256, 0, st>>>(
        a, a.use_even ? static_cast<const T2*>(te.p) : nullptr,
        a.use_odd ? static_cast<const T2*>(to.p) : nullptr, static_cast<T2*>(a.dst0));
    return (int)cudaGetLastError();
}

template <typename T>
static int leaf_pair(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    const size_t b = operand_bytes<T>(a);
    Scratch s0(b, st), s1(b, st), te(b, st), to(b, st);
    if (!s0.p || !s1.p || !te.p || !to.p)
        return (int)cudaErrorMemoryAllocation;
    using T2 = typename cx<T>::t;
    const int g = grid_for(a.ncomp * a.outer * a.n);
    const int gm = grid_for(a.outer * a.n);
    if (a.use_odd) {
        k_phase<T><<<g, 256, 0, st>>>(a, static_cast<const T2*>(a.src0), static_cast<T2*>(to.p));
        if (int e = fft<T, false>(a, to.p, to.p, s0.p, s1.p, st))
            return e;
        k_leaf_mul<T><<<gm, 256, 0, st>>>(a, sp, 1, static_cast<T2*>(to.p));
        if (int e = fft<T, true>(a, to.p, to.p, s0.p, s1.p, st))
            return e;
    }
    if (a.use_even) {
        if (int e = fft<T, false>(a, a.src0, te.p, s0.p, s1.p, st))
            return e;
        k_leaf_mul<T><<<gm, 256, 0, st>>>(a, sp, 0, static_cast<T2*>(te.p));
        if (int e = fft<T, true>(a, te.p, te.p, s0.p, s1.p, st))
            return e;
    }
    k_merge<T><<<g, 256, 0, st>>>(a, a.use_even ? static_cast<const T2*>(te.p) : nullptr,
                                  a.use_odd ? static_cast<const T2*>(to.p) : nullptr,
                                  static_cast<T2*>(a.dst0));
    return (int)cudaGetLastError();
}

}  // namespace glob
}  // namespace tsk

extern "C" int tsk_global_fwd_split(const tsk_axis* a, void* stream)
{
    auto st = static_cast<cudaStream_t>(stream);
    return a->prec ? tsk::glob::fwd_split<float>(*a, st) : tsk::glob::fwd_split<double>(*a, st);
}

extern "C" int tsk_global_inv_merge(const tsk_axis* a, void* stream)
{
    auto st = static_cast<cudaStream_t>(stream);
    return a->prec ? tsk::glob::inv_merge<float>(*a, st) : tsk::glob::inv_merge<double>(*a, st);
}

extern "C" int tsk_global_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    if (a->inner != 1)
        return (int)cudaErrorInvalidValue;
    auto st = static_cast<cudaStream_t>(stream);
    return a->prec ? tsk::glob::leaf_pair<float>(*a, *sp, st) : tsk::glob::leaf_pair<double>(*a, *sp, st);
}
