// Shared device helpers for the toesplit sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>

#include "tsk_launch.h"

namespace tsk {

template <typename T>
struct cx;
template <>
struct cx<float> {
    using t = float2;
};
template <>
struct cx<double> {
    using t = double2;
};

template <typename T>
__device__ __forceinline__ typename cx<T>::t make_c(T x, T y)
{
    typename cx<T>::t r;
    r.x = x;
    r.y = y;
    return r;
}

// ---- packed f32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2) ------------------
// A complex64 value is one 64-bit register pair; ptxas folds broadcasts
// make_float2(a.x, a.x) and lane swaps make_float2(a.y, a.x) into operand
// swizzles, so complex add/sub is one instruction and a complex multiply by a
// pre-rotated twiddle two.
__device__ __forceinline__ unsigned long long f2_u(float2 a)
{
    union {
        float2 f;
        unsigned long long u;
    } c;
    c.f = a;
    return c.u;
}
__device__ __forceinline__ float2 u_f2(unsigned long long a)
{
    union {
        float2 f;
        unsigned long long u;
    } c;
    c.u = a;
    return c.f;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b)
{
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)));
    return u_f2(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b)
{
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)));
    return u_f2(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b)
{
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)));
    return u_f2(d);
}

// v * s for a real s: one packed multiply for complex64
template <typename T>
__device__ __forceinline__ typename cx<T>::t scale_c(typename cx<T>::t v, T s)
{
    if constexpr (sizeof(T) == 4)
        return mul2(v, make_float2(s, s));
    else
        return make_c<T>(v.x * s, v.y * s);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c)
{
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_u(a)), "l"(f2_u(b)), "l"(f2_u(c)));
    return u_f2(d);
}
__device__ __forceinline__ float2 bc_x(float2 a) { return make_float2(a.x, a.x); }
__device__ __forceinline__ float2 bc_y(float2 a) { return make_float2(a.y, a.y); }
__device__ __forceinline__ float2 swz(float2 a) { return make_float2(a.y, a.x); }

template <typename T2>
__device__ __forceinline__ T2 cadd(T2 a, T2 b)
{
    T2 r;
    r.x = a.x + b.x;
    r.y = a.y + b.y;
    return r;
}
template <>
__device__ __forceinline__ float2 cadd<float2>(float2 a, float2 b)
{
    return add2(a, b);
}

template <typename T2>
__device__ __forceinline__ T2 csub(T2 a, T2 b)
{
    T2 r;
    r.x = a.x - b.x;
    r.y = a.y - b.y;
    return r;
}
template <>
__device__ __forceinline__ float2 csub<float2>(float2 a, float2 b)
{
    return sub2(a, b);
}

// (a.x + i a.y)(b.x + i b.y)
template <typename T2>
__device__ __forceinline__ T2 cmul(T2 a, T2 b)
{
    T2 r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}

// a * conj(b)
template <typename T2>
__device__ __forceinline__ T2 cmulc(T2 a, T2 b)
{
    T2 r;
    r.x = a.x * b.x + a.y * b.y;
    r.y = a.y * b.x - a.x * b.y;
    return r;
}

__device__ __forceinline__ float2 ldg_c(const float2* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldg_c(const double2* p) { return __ldg(p); }

// Root table entry k (exp(-2 pi i k/n)); conjugated for inverse transforms.
template <typename T, bool INV>
__device__ __forceinline__ typename cx<T>::t twiddle(const typename cx<T>::t* __restrict__ roots,
                                                     int k)
{
    typename cx<T>::t w = ldg_c(roots + k);
    if (INV)
        w.y = -w.y;
    return w;
}

// multiply by -i (forward) or +i (inverse)
template <typename T2, bool INV>
__device__ __forceinline__ T2 mul_mi(T2 a)
{
    T2 r;
    if (INV) {
        r.x = -a.y;
        r.y = a.x;
    } else {
        r.x = a.y;
        r.y = -a.x;
    }
    return r;
}

template <typename T, bool INV>
__device__ __forceinline__ void dft4(typename cx<T>::t& x0, typename cx<T>::t& x1,
                                     typename cx<T>::t& x2, typename cx<T>::t& x3)
{
    using T2 = typename cx<T>::t;
    const T2 s0 = cadd(x0, x2), d0 = csub(x0, x2);
    const T2 s1 = cadd(x1, x3), d1 = mul_mi<T2, INV>(csub(x1, x3));
    x0 = cadd(s0, s1);
    x2 = csub(s0, s1);
    x1 = cadd(d0, d1);
    x3 = csub(d0, d1);
}

// +-i a as a lane swap with one lane negated: ptxas folds it into the
// consuming FADD2/FFMA2 operand (.LO_HI.NP), so it costs no instruction.
__device__ __forceinline__ float2 mul_i(float2 a) { return make_float2(-a.y, a.x); }
__device__ __forceinline__ float2 mul_negi(float2 a) { return make_float2(a.y, -a.x); }

// Packed complex64 radix-4: 8 FADD2, the -+i folded into operands.
template <>
__device__ __forceinline__ void dft4<float, false>(float2& x0, float2& x1, float2& x2, float2& x3)
{
    const float2 s0 = add2(x0, x2), d0 = sub2(x0, x2);
    const float2 s1 = add2(x1, x3), d1 = sub2(x1, x3);
    x0 = add2(s0, s1);
    x2 = sub2(s0, s1);
    x1 = add2(d0, mul_negi(d1));  // d0 - i d1
    x3 = add2(d0, mul_i(d1));     // d0 + i d1
}
template <>
__device__ __forceinline__ void dft4<float, true>(float2& x0, float2& x1, float2& x2, float2& x3)
{
    const float2 s0 = add2(x0, x2), d0 = sub2(x0, x2);
    const float2 s1 = add2(x1, x3), d1 = sub2(x1, x3);
    x0 = add2(s0, s1);
    x2 = sub2(s0, s1);
    x1 = add2(d0, mul_i(d1));     // d0 + i d1
    x3 = add2(d0, mul_negi(d1));  // d0 - i d1
}

// Packed complex64 radix-4 whose x2 arrives as t2 with a pending real factor
// hs (a 45-degree twiddle h (1 -+ i) x = h t, t = x -+ i x): the factor rides
// on the first butterfly (x0 +- hs t2 as two FFMA2), one instruction fewer
// than scaling t2 first.
template <bool INV>
__device__ __forceinline__ void dft4_h(float2& x0, float2& x1, float2& t2, float2& x3, float hs)
{
    const float2 s0 = fma2(t2, make_float2(hs, hs), x0), d0 = fma2(t2, make_float2(-hs, -hs), x0);
    const float2 s1 = add2(x1, x3), d1 = sub2(x1, x3);
    x0 = add2(s0, s1);
    t2 = sub2(s0, s1);
    x1 = add2(d0, INV ? mul_i(d1) : mul_negi(d1));
    x3 = add2(d0, INV ? mul_negi(d1) : mul_i(d1));
}

// Packed complex64 radix-8 (DIT from two radix-4): 26 FP instructions.
// H: v[4] carries a pending real factor hs (see dft4_h).
template <bool INV, bool H = false>
__device__ __forceinline__ void dft8_packed(float2* v, float hs = 0.f)
{
    float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
    float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    if constexpr (H)
        dft4_h<INV>(e0, e1, e2, e3, hs);
    else
        dft4<float, INV>(e0, e1, e2, e3);
    dft4<float, INV>(o0, o1, o2, o3);
    // twiddles with broadcast immediates: w8 = h (1 - i), w8^3 = -h (1 + i)
    const float h = 0.70710678118654752440f;
    // the h scaling of the two 45-degree twiddles rides on the final
    // butterflies (e +- h t as two FFMA2): 26 FP instructions
    if (!INV) {
        o1 = add2(o1, mul_negi(o1));
        o3 = add2(o3, mul_i(o3));
        v[2] = add2(e2, mul_negi(o2));
        v[6] = add2(e2, mul_i(o2));
    } else {
        o1 = add2(o1, mul_i(o1));
        o3 = add2(o3, mul_negi(o3));
        v[2] = add2(e2, mul_i(o2));
        v[6] = add2(e2, mul_negi(o2));
    }
    const float2 hp = make_float2(h, h), hm = make_float2(-h, -h);
    v[0] = add2(e0, o0);
    v[4] = sub2(e0, o0);
    v[1] = fma2(o1, hp, e1);
    v[5] = fma2(o1, hm, e1);
    v[3] = fma2(o3, hm, e3);
    v[7] = fma2(o3, hp, e3);
}

// In-register DFT of size R: v[q] <- sum_r v[r] w_R^{rq}, w_R = exp(-+2 pi i/R).
// roots/m give w_R^e = roots[e*m] for the generic odd radices.
template <typename T, int R, bool INV>
__device__ __forceinline__ void dft_small(typename cx<T>::t* v,
                                          const typename cx<T>::t* __restrict__ roots, int m)
{
    using T2 = typename cx<T>::t;
    if constexpr (R == 2) {
        const T2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (R == 4) {
        dft4<T, INV>(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 8 && sizeof(T) == 4) {
        dft8_packed<INV>(reinterpret_cast<float2*>(v));
    } else if constexpr (R == 8) {
        T2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
        T2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
        dft4<T, INV>(e0, e1, e2, e3);
        dft4<T, INV>(o0, o1, o2, o3);
        const T h = (T)0.70710678118654752440084436210484903928;
        // o_q *= w8^q
        {
            T2 t;
            t.x = h * (o1.x + (INV ? -o1.y : o1.y));
            t.y = h * (o1.y + (INV ? o1.x : -o1.x));
            o1 = t;
        }
        o2 = mul_mi<T2, INV>(o2);
        {
            T2 t;
            t.x = h * (-o3.x + (INV ? -o3.y : o3.y));
            t.y = h * (-o3.y + (INV ? o3.x : -o3.x));
            o3 = t;
        }
        v[0] = cadd(e0, o0);
        v[4] = csub(e0, o0);
        v[1] = cadd(e1, o1);
        v[5] = csub(e1, o1);
        v[2] = cadd(e2, o2);
        v[6] = csub(e2, o2);
        v[3] = cadd(e3, o3);
        v[7] = csub(e3, o3);
    } else {
        T2 out[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            T2 acc = v[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
                acc = cadd(acc, cmul(v[r], twiddle<T, INV>(roots, ((r * q) % R) * m)));
            out[q] = acc;
        }
#pragma unroll
        for (int q = 0; q < R; ++q)
            v[q] = out[q];
    }
}

// ref kernel.cpp:17-21
__host__ __device__ __forceinline__ int64_t stored_len(int64_t n, int odd)
{
    return odd ? (n + 1) / 2 : n / 2 + 1;
}

// ref kernel.cpp:25-37
__host__ __device__ __forceinline__ int64_t mirror_src(int64_t n, int odd, int64_t k,
                                                       bool& mirrored)
{
    if (odd) {
        const int64_t st = (n + 1) / 2;
        mirrored = k >= st;
        return mirrored ? n - 1 - k : k;
    }
    mirrored = k > n / 2;
    return mirrored ? n - k : k;
}

#ifdef __CUDACC__
// n / d for n < 2^31 by a multiply-high (divisor fixed for the launch)
struct FastDiv {
    uint32_t d, mul, shift;
    __device__ __forceinline__ explicit FastDiv(uint32_t dv) : d(dv), mul(0), shift(0)
    {
        if (dv > 1) {
            uint32_t l = 32 - __clz(dv - 1);  // ceil(log2 d)
            const uint32_t pw = 31 + l;
            mul = (uint32_t)(((1ull << pw) + dv - 1) / dv);
            shift = pw - 32;
        }
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const
    {
        return d > 1 ? __umulhi(n, mul) >> shift : n;
    }
};

// ---- programmatic dependent launch: the hot passes (k_wide, k_wtma,
// k_leaf1) are launched with programmatic stream serialisation; each CTA of a
// pass signals on its last tile, so the next pass's CTAs are scheduled as the
// previous pass's CTAs retire and run their prologue (tables, tensor-memory
// allocation, barriers) under its tail; each waits (griddepcontrol.wait: the
// previous grid complete, its writes visible) before touching the vectors. A
// no-op for plain launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // TSK_NO_PDL=1 turns it off (A/B); dispatch.cu

// PDL pays where launch latency and pass prologues are a visible share
// (configs[1] +11%, [4] +4%, [2] +1%); on 3.2 GB vectors it gained nothing
// for compressed spectra and cost 16% with full 512^3 spectra (25.8 -> 30.0 ms
// per MVM, profiles/r02_ab_ix.txt), so passes over vectors above 1 GB launch
// plainly.
__host__ inline bool pdl_for(const tsk_axis& a)
{
    const double bytes = (double)a.outer * (double)a.n * (double)a.inner * (double)(a.ncomp > 0 ? a.ncomp : 1) *
                         (a.prec ? 8.0 : 16.0) * (double)(a.nrhs > 1 ? a.nrhs : 1);
    return pdl_enabled() && bytes <= 1073741824.0;
}

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(bool use, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                                     cudaStream_t st, Args&&... args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = use ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#endif

}  // namespace tsk
