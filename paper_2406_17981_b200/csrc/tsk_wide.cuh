// Register-FFT building blocks with R elements per thread (radix up to 32):
// compile-time twiddle constants (64th roots of unity), the in-register DFT
// split P = P1 x P2, the per-stage plan and 64-bit twiddle-table access.
// Shared by the wide strided kernels and the leaf kernel.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "tsk_common.cuh"

namespace tsk {
namespace wide {

constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// cos(2 pi k / 64), k = 0..16 (quarter wave; the rest by symmetry)
__host__ __device__ constexpr double cos64q(int k)
{
    constexpr double t[17] = {1.0,
                              0.99518472667219688624,
                              0.98078528040323044913,
                              0.95694033573220886494,
                              0.92387953251128675613,
                              0.88192126434835502971,
                              0.83146961230254523708,
                              0.77301045336273696081,
                              0.70710678118654752440,
                              0.63439328416364549822,
                              0.55557023301960222474,
                              0.47139673682599764856,
                              0.38268343236508977173,
                              0.29028467725446236764,
                              0.19509032201612826785,
                              0.09801714032956060199,
                              0.0};
    return t[k];
}
__host__ __device__ constexpr double cos64(int k)
{
    k = ((k % 64) + 64) % 64;
    if (k <= 16)
        return cos64q(k);
    if (k <= 32)
        return -cos64q(32 - k);
    if (k <= 48)
        return -cos64q(k - 32);
    return cos64q(64 - k);
}
__host__ __device__ constexpr double sin64(int k) { return cos64(k - 16); }

// v * exp(sgn 2 pi i k / P) for a compile-time angle (P | 64).
template <typename T, int P, int K, bool INV>
__device__ __forceinline__ typename cx<T>::t cmul_const(typename cx<T>::t v)
{
    constexpr int k64 = ((K % P) + P) % P * (64 / P);
    constexpr double c = cos64(k64);
    constexpr double s = (INV ? 1.0 : -1.0) * sin64(k64);
    if constexpr (k64 == 0) {
        return v;
    } else if constexpr (k64 == 32) {
        return make_c<T>(-v.x, -v.y);
    } else if constexpr (k64 == 16 || k64 == 48) {
        // multiply by +-i: a lane swap + negate, folded into the consumer
        return s > 0 ? make_c<T>(-v.y, v.x) : make_c<T>(v.y, -v.x);
    } else {
        // c v + s (i v): broadcast immediates, (i v) an operand modifier
        if constexpr (sizeof(T) == 4)
            return fma2(make_float2(-v.y, v.x), make_float2((float)s, (float)s),
                        mul2(v, make_float2((float)c, (float)c)));
        else
            return make_c<T>(v.x * c - v.y * s, v.x * s + v.y * c);
    }
}

// In-register DFT of size P on a[0..P), natural order in and out.
template <typename T, int P, bool INV>
struct Dft {
    using T2 = typename cx<T>::t;
    // split P = P1 * P2: input r = P2 a + b, output q = c + P1 e
    static constexpr int P1 = P >= 16 ? 4 : 2;
    static constexpr int P2 = P / P1;
    // 45-degree twiddles h (+-1 +- i) on the element that enters the next
    // stage's first butterfly as x2 (B = P2 / 2) against an untwiddled x0:
    // only the rotation t = x -+ i x is applied here, the real factor +-h
    // rides on that butterfly (dft4_h), saving one instruction each
    template <int B, int C>
    static constexpr int k64_of()
    {
        return ((B * C) % P) * (64 / P);
    }
    template <int B, int C>
    static constexpr bool h_fused()
    {
        return sizeof(T) == 4 && P >= 16 && B == P2 / 2 && k64_of<B, C>() % 16 == 8;
    }
    template <int B, int C>
    __device__ __forceinline__ static void tw(T2* a)
    {
        if constexpr (h_fused<B, C>()) {
            constexpr int k = k64_of<B, C>();
            // forward: k = 8, 40 -> (1 - i), k = 24, 56 -> (1 + i); inverse swapped
            constexpr bool minus_i = ((k == 8 || k == 40) != INV);
            const float2 x = a[P2 * C + B];
            a[P2 * C + B] = add2(x, minus_i ? mul_negi(x) : mul_i(x));
        } else {
            a[P2 * C + B] = cmul_const<T, P, B * C, INV>(a[P2 * C + B]);
        }
    }
    // step 2 of group C: one transform of length P2 on a[P2 C ..), outputs to o[C + P1 e]
    template <int C>
    __device__ __forceinline__ static void group(T2* a, T2* o)
    {
        T2 s[P2];
#pragma unroll
        for (int i = 0; i < P2; ++i)
            s[i] = a[P2 * C + i];
        if constexpr (h_fused<P2 / 2, C>()) {
            constexpr int k = k64_of<P2 / 2, C>();
            constexpr float hs = (k == 8 || k == 56) ? 0.70710678118654752440f : -0.70710678118654752440f;
            if constexpr (P2 == 4)
                dft4_h<INV>(s[0], s[1], s[2], s[3], hs);
            else
                dft8_packed<INV, true>(s, hs);
        } else {
            Dft<T, P2, INV>::run(s);
        }
#pragma unroll
        for (int e = 0; e < P2; ++e)
            o[C + P1 * e] = s[e];
    }
    template <int... Cs>
    __device__ __forceinline__ static void groups(T2* a, T2* o, std::integer_sequence<int, Cs...>)
    {
        (group<Cs>(a, o), ...);
    }
    __device__ __forceinline__ static void run(T2* a)
    {
        if constexpr (P == 1) {
        } else if constexpr (P == 2) {
            const T2 x = a[0], y = a[1];
            a[0] = cadd(x, y);
            a[1] = csub(x, y);
        } else if constexpr (P == 4) {
            dft4<T, INV>(a[0], a[1], a[2], a[3]);
        } else if constexpr (P == 8) {
            dft_small<T, 8, INV>(a, nullptr, 0);
        } else {
            static_assert(P2 == 4 || P2 == 8, "step 2 runs radix-4 or radix-8 groups");
            // step 1: P2 transforms of length P1 on stride-P2 subsequences
#pragma unroll
            for (int b = 0; b < P2; ++b) {
                T2 s[P1];
#pragma unroll
                for (int i = 0; i < P1; ++i)
                    s[i] = a[P2 * i + b];
                Dft<T, P1, INV>::run(s);
#pragma unroll
                for (int i = 0; i < P1; ++i)
                    a[P2 * i + b] = s[i];
            }
            // twiddles w_P^{b c}
            twiddles(a, std::make_integer_sequence<int, P1 * P2>{});
            // step 2: P1 transforms of length P2 on contiguous groups
            T2 o[P];
            groups(a, o, std::make_integer_sequence<int, P1>{});
#pragma unroll
            for (int q = 0; q < P; ++q)
                a[q] = o[q];
        }
    }
    template <int... Is>
    __device__ __forceinline__ static void twiddles(T2* a, std::integer_sequence<int, Is...>)
    {
        (tw<Is % P2, Is / P2>(a), ...);
    }
};

template <int N, int R>
struct Plan {
    static constexpr int TF = N / R;
    static constexpr int L = ilog2(N), LR = ilog2(R);
    static constexpr int NST = (L + LR - 1) / LR;
    static constexpr int radix(int s)
    {
        return s < NST - 1 ? R : (1 << (L - LR * (NST - 1)));
    }
    static constexpr int ns(int s)
    {
        int v = 1;
        for (int i = 0; i < s; ++i)
            v *= radix(i);
        return v;
    }
    static constexpr int tw_off(int s)
    {
        int o = 0;
        for (int i = 1; i < s; ++i)
            o += ns(i) * (radix(i) - 1);
        return o;
    }
    static constexpr int TW = tw_off(NST) > 0 ? tw_off(NST) : 1;
};

template <typename T>
struct tw4;
template <>
struct tw4<float> {
    using t = float4;
};
template <>
struct tw4<double> {
    using t = double4;
};

template <typename T>
struct Tw {
    typename cx<T>::t lo, hi;
};

// Tables keep only w (64-bit reads: 2 wavefronts per warp even when
// broadcast, a 128-bit read costs 4); cmul_tw needs no rotated copy.
template <typename T>
__device__ __forceinline__ Tw<T> load_tw(const typename cx<T>::t* p)
{
    Tw<T> w;
    w.lo = *p;
    w.hi = w.lo;
    return w;
}

template <typename T>
__device__ __forceinline__ typename tw4<T>::t make_tw(typename cx<T>::t w)
{
    typename tw4<T>::t r;
    r.x = w.x;
    r.y = w.y;
    r.z = -w.y;
    r.w = w.x;
    return r;
}

// v w = w.x v + w.y (i v); v conj(w) = w.x v - w.y (i v)
template <typename T, bool CONJ>
__device__ __forceinline__ typename cx<T>::t cmul_tw(typename cx<T>::t v, const Tw<T>& w)
{
    if constexpr (sizeof(T) == 4) {
        const float2 iv = CONJ ? make_float2(v.y, -v.x) : make_float2(-v.y, v.x);
        return fma2(iv, bc_y(w.lo), mul2(v, bc_x(w.lo)));
    } else {
        return CONJ ? cmulc(v, w.lo) : cmul(v, w.lo);
    }
}

}  // namespace wide
}  // namespace tsk
