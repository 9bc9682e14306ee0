// Register-resident sm_100a kernels for power-of-two axis lengths (8..1024),
// the hot path of the headline configs (512^3, 256^3, 64^3, 64^4).
//
// Layout of one length-N transform: TF = N/8 threads each hold 8 elements in
// registers at positions k = t + m*TF (m < 8, "row pattern"). A Stockham
// stage of radix p (8, then a final 4 or 2) reads the row pattern and writes
// positions (j - j%Ns)*p + j%Ns + q*Ns; all but the last stage exchange
// through shared memory (ping-pong buffers, one __syncthreads each); the
// last stage lands back in the row pattern in registers, in natural order.
// So a transform costs (#stages - 1) shared-memory exchanges and no global
// re-reads; loads and stores of the row pattern are coalesced (lanes over
// adjacent columns for strided axes, over adjacent t for the contiguous axis).
//
// K1 fwd_split (strided axes):  even = F(t), odd = F(P t)      read 1, write 2
// K3 inv_merge (strided axes):  out = (B(e) + conj(P) B(o)) * scale
// K2 leaf_pair (last axis):     per branch F -> m x m spectra multiply in
//                               registers -> B; out = (e' + conj(P) o') * scale
// Reference semantics as in kernels_generic.cu (fft.cpp:65-87,
// tensor.cpp:227-254, engine_split.cpp:13-37, kernel.cpp:126-219).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "tsk_common.cuh"

namespace tsk {
namespace fast {

constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int N>
struct Plan {
    static constexpr int TF = N / 8;
    static constexpr int L = ilog2(N);
    static constexpr int NST = (L + 2) / 3;  // radix-8 stages, last one 8, 4 or 2
    static constexpr int radix(int s)
    {
        return s < NST - 1 ? 8 : (L - 3 * (NST - 1) == 3 ? 8 : (L - 3 * (NST - 1) == 2 ? 4 : 2));
    }
    static constexpr int ns(int s)  // product of earlier radices
    {
        int v = 1;
        for (int i = 0; i < s; ++i)
            v *= radix(i);
        return v;
    }
    // twiddle table: stage s >= 1 holds ns(s) x (radix(s)-1) entries
    static constexpr int tw_off(int s)
    {
        int o = 0;
        for (int i = 1; i < s; ++i)
            o += ns(i) * (radix(i) - 1);
        return o;
    }
    static constexpr int TW = tw_off(NST) > 0 ? tw_off(NST) : 1;
    // register twiddle bases: one per (stage >= 1, butterfly i < 8/radix)
    static constexpr int slot(int s, int i)
    {
        int o = 0;
        for (int k = 1; k < s; ++k)
            o += 8 / radix(k);
        return o + i;
    }
    static constexpr int NSLOT = slot(NST, 0) > 0 ? slot(NST, 0) : 1;
};

// Twiddle / phase entries as {w, rot(w)} with rot(w) = (-w.y, w.x): a
// complex64 multiply by w is then FMUL2 + FFMA2 and by conj(w) the same two
// instructions on lane-swapped operands (swz(rot w) = conj w, swz(w) =
// rot(conj w)). complex128 uses the plain pair.
template <typename T>
struct Tw {
    typename cx<T>::t lo, hi;
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

// Table entries keep only w: a 64-bit shared read costs 2 wavefronts per warp
// (a 128-bit one 4, even when broadcast); rot(w) = (-w.y, w.x) is one FMUL2.
template <typename T>
__device__ __forceinline__ Tw<T> load_tw(const typename tw4<T>::t* p)
{
    Tw<T> w;
    w.lo = *reinterpret_cast<const typename cx<T>::t*>(p);
    if constexpr (sizeof(T) == 4)
        w.hi = mul2(swz(w.lo), make_float2(-1.f, 1.f));
    else
        w.hi = make_c<T>(-w.lo.y, w.lo.x);
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

// v * w (CONJ: v * conj(w))
template <typename T, bool CONJ>
__device__ __forceinline__ typename cx<T>::t cmul_tw(typename cx<T>::t v, const Tw<T>& w)
{
    if constexpr (sizeof(T) == 4) {
        if (CONJ)
            return fma2(bc_y(v), swz(w.lo), mul2(bc_x(v), swz(w.hi)));
        return fma2(bc_y(v), w.hi, mul2(bc_x(v), w.lo));
    } else {
        return CONJ ? cmulc(v, w.lo) : cmul(v, w.lo);
    }
}

__device__ __forceinline__ void opaque(float2& v) { asm volatile("" : "+f"(v.x), "+f"(v.y)); }
__device__ __forceinline__ void opaque(double2& v) { asm volatile("" : "+d"(v.x), "+d"(v.y)); }

template <typename T>
__device__ __forceinline__ Tw<T> make_twv(typename cx<T>::t w)
{
    Tw<T> r;
    r.lo = w;
    if constexpr (sizeof(T) == 4)
        r.hi = mul2(swz(w), make_float2(-1.f, 1.f));
    else
        r.hi = make_c<T>(-w.y, w.x);
    return r;
}

// w^r for r = 1..P-1 from w (depth <= 3 products, ~3 ulp in complex64).
template <typename T, int P>
__device__ __forceinline__ void tw_powers(const Tw<T>& b, Tw<T> (&pw)[8])
{
    pw[1] = b;
    if (P > 2)
        pw[2] = make_twv<T>(cmul_tw<T, false>(b.lo, b));
    if (P > 3)
        pw[3] = make_twv<T>(cmul_tw<T, false>(pw[2].lo, b));
    if (P > 4) {
        pw[4] = make_twv<T>(cmul_tw<T, false>(pw[2].lo, pw[2]));
        pw[5] = make_twv<T>(cmul_tw<T, false>(pw[4].lo, b));
        pw[6] = make_twv<T>(cmul_tw<T, false>(pw[4].lo, pw[2]));
        pw[7] = make_twv<T>(cmul_tw<T, false>(pw[4].lo, pw[3]));
    }
}

// Split phase P_k = exp(-i pi k/N) at the row pattern k = t + m N/8:
// P_k = P_t * exp(-i pi m/8), P_t held in registers, the eighth-turn factors
// compile-time constants.
template <typename T>
struct PhaseReg {
    Tw<T> pt;
    template <bool CONJ>
    __device__ __forceinline__ typename cx<T>::t apply(typename cx<T>::t v, int m) const
    {
        constexpr double C1 = 0.92387953251128675613, S1 = 0.38268343236508977173,
                         H = 0.70710678118654752440;
        const double cr[8] = {1.0, C1, H, S1, 0.0, -S1, -H, -C1};
        const double ci[8] = {0.0, -S1, -H, -C1, -1.0, -C1, -H, -S1};
        if (m != 0) {
            typename cx<T>::t c = make_c<T>((T)cr[m], (T)ci[m]);
            v = cmul_tw<T, CONJ>(v, make_twv_const<T>(c));
        }
        return cmul_tw<T, CONJ>(v, pt);
    }
    template <typename TT>
    __device__ __forceinline__ static Tw<TT> make_twv_const(typename cx<TT>::t c)
    {
        Tw<TT> r;
        r.lo = c;
        r.hi = make_c<TT>(-c.y, c.x);
        return r;
    }
};

// Fill the per-stage twiddle table (w_N^{r * jm * N/(Ns p)}) and the phase
// table P_k = exp(-i pi k/N) from the operator's double-accurate root/phase
// tables (global) into shared memory.
template <typename T, int N>
__device__ void fill_tables(typename tw4<T>::t* tw, typename tw4<T>::t* ph,
                            const typename cx<T>::t* __restrict__ roots,
                            const typename cx<T>::t* __restrict__ phase)
{
    using P = Plan<N>;
#pragma unroll
    for (int s = 1; s < P::NST; ++s) {
        const int p = P::radix(s), ns = P::ns(s);
        const int cnt = ns * (p - 1);
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const int jm = e / (p - 1), r = e % (p - 1) + 1;
            tw[P::tw_off(s) + e] = make_tw<T>(ldg_c(roots + (r * jm * (N / (ns * p))) % N));
        }
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x)
        ph[k] = make_tw<T>(ldg_c(phase + k));
}

// One radix-p butterfly on registers v[i + r*(8/p)], r < p, compile-time p.
template <typename T, int P, bool INV>
__device__ __forceinline__ void butterfly(typename cx<T>::t (&v)[8], int i)
{
    using T2 = typename cx<T>::t;
    constexpr int G = 8 / P;
    if constexpr (P == 8) {
        dft_small<T, 8, INV>(v, nullptr, 0);
    } else if constexpr (P == 4) {
        dft4<T, INV>(v[i], v[i + G], v[i + 2 * G], v[i + 3 * G]);
    } else {
        const T2 a = v[i], b = v[i + G];
        v[i] = cadd(a, b);
        v[i + G] = csub(a, b);
    }
}

// K simultaneous length-N transforms of the row pattern held in v[k][8].
// buf0/buf1: ping-pong exchange buffers; sidx(k, pos) gives the element index
// of (transform k, position pos) inside one buffer. xc counts exchanges across
// calls so consecutive exchanges alternate buffers (one __syncthreads each).
struct SyncCta {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// Threads of one fiber only: a named barrier over `count` threads, or a warp
// barrier when the fiber lives inside one warp.
struct SyncGroup {
    int id, count;
    __device__ __forceinline__ void operator()() const
    {
        if (count <= 32)
            __syncwarp();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
    }
};

// wreg (optional): per-thread twiddle bases, slot(s, i) = w_N^{jm N/(Ns p)};
// when given, powers are formed in registers instead of reading the table.
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f)
{
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// Stage S of K simultaneous length-N transforms (compile-time stage, radix
// and butterfly indices, so every register/twiddle index is a constant).
template <typename T, int N, bool INV, int K, bool REGTW, int S, class SIdx, class Sync, class WReg,
          bool SINGLE = false>
__device__ __forceinline__ void fft_stage(typename cx<T>::t (&v)[K][8], typename cx<T>::t* buf0,
                                          typename cx<T>::t* buf1, const SIdx& sidx,
                                          const typename tw4<T>::t* tw, int t, int& xc,
                                          const Sync& sync, const WReg& wreg)
{
    using T2 = typename cx<T>::t;
    using PL = Plan<N>;
    constexpr int TF = PL::TF;
    constexpr int p = PL::radix(S);
    constexpr int ns = PL::ns(S);
    constexpr int G = 8 / p;
    if constexpr (S > 0) {
        static_for<0, G>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if constexpr (REGTW && S == PL::NST - 1) {
                // last stage (a distinct base per thread): powers of a register
                // base instead of table reads
                Tw<T> b = wreg[i];
                T2 pw[8];
                pw[1] = b.lo;
                if constexpr (p > 2)
                    pw[2] = cmul_tw<T, false>(b.lo, b);
                if constexpr (p > 3)
                    pw[3] = cmul_tw<T, false>(pw[2], b);
                if constexpr (p > 4) {
                    const Tw<T> b2 = make_twv<T>(pw[2]);
                    pw[4] = cmul_tw<T, false>(pw[2], b2);
                    pw[5] = cmul_tw<T, false>(pw[4], b);
                    pw[6] = cmul_tw<T, false>(pw[4], b2);
                    pw[7] = cmul_tw<T, false>(pw[4], make_twv<T>(pw[3]));
                }
#pragma unroll
                for (int r = 1; r < p; ++r) {
                    const Tw<T> w = make_twv<T>(pw[r]);
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        v[k][i + r * G] = cmul_tw<T, INV>(v[k][i + r * G], w);
                }
            } else {
                const int jm = (t + i * TF) % ns;
#pragma unroll
                for (int r = 1; r < p; ++r) {
                    const Tw<T> w = load_tw<T>(tw + PL::tw_off(S) + jm * (p - 1) + (r - 1));
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        v[k][i + r * G] = cmul_tw<T, INV>(v[k][i + r * G], w);
                }
            }
        });
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if constexpr (p == 8)
            butterfly<T, 8, INV>(v[k], 0);
        else if constexpr (p == 4) {
            butterfly<T, 4, INV>(v[k], 0);
            butterfly<T, 4, INV>(v[k], 1);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                butterfly<T, 2, INV>(v[k], i);
        }
    }
    if constexpr (S < PL::NST - 1) {
        T2* buf = (SINGLE || !(xc++ & 1)) ? buf0 : buf1;
        static_for<0, G>([&](auto I) {
            constexpr int i = decltype(I)::value;
            const int j = t + i * TF;
            const int jm = j % ns;
            const int base = (j - jm) * p + jm;
#pragma unroll
            for (int q = 0; q < p; ++q)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    buf[sidx(k, base + q * ns)] = v[k][i + q * G];
        });
        sync();
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int k = 0; k < K; ++k)
                v[k][m] = buf[sidx(k, t + m * TF)];
        if constexpr (SINGLE)
            sync();  // single buffer: all reads done before the next writes
        fft_stage<T, N, INV, K, REGTW, S + 1, SIdx, Sync, WReg, SINGLE>(v, buf0, buf1, sidx, tw, t, xc,
                                                                         sync, wreg);
    }
}

// leaf pass: last-stage twiddles from register powers (true) or the table
#ifndef LEAF_REGTW
#define LEAF_REGTW false
#endif

struct NoWReg {
    template <typename I>
    __device__ int operator[](I) const { return 0; }
};

// K simultaneous length-N transforms of the row pattern held in v[k][8].
// buf0/buf1: ping-pong exchange buffers; sidx(k, pos) gives the element index
// of (transform k, position pos) inside one buffer. xc counts exchanges across
// calls so consecutive exchanges alternate buffers (one barrier each). wreg
// (REGTW): per-thread twiddle bases indexed by Plan::slot(stage, butterfly).
template <typename T, int N, bool INV, int K, class SIdx, class Sync = SyncCta, bool REGTW = false,
          class WReg = NoWReg, bool SINGLE = false>
__device__ __forceinline__ void fft_rows(typename cx<T>::t (&v)[K][8], typename cx<T>::t* buf0,
                                         typename cx<T>::t* buf1, const SIdx& sidx,
                                         const typename tw4<T>::t* tw, int t, int& xc,
                                         const Sync& sync = Sync(), const WReg& wreg = WReg())
{
    fft_stage<T, N, INV, K, REGTW, 0, SIdx, Sync, WReg, SINGLE>(v, buf0, buf1, sidx, tw, t, xc, sync,
                                                                 wreg);
}

// Shared-memory index maps (bank-conflict-free for the three access patterns
// of an exchange: row-pattern reads t + m*TF, stage-0 writes 8t + q, stage-1
// writes 64(t/8) + t%8 + 8q; checked per 128-byte wavefront).
//
// Strided tiles, W columns per row. With 8-byte elements and W = 8 a
// half-warp touches two rows; rows r and r' of one access must sit in
// different 64-byte halves of a 128-byte bank line: row r lives in line r/2,
// half (r ^ r>>3) & 1. Otherwise rows are plain (one row per wavefront).
template <int N, int W, int ES>
struct StridedIdx {
    int w;
    __device__ __forceinline__ int operator()(int k, int pos) const
    {
        if constexpr (ES == 8 && W == 8)
            return k * N * W + (pos >> 1) * 16 + (((pos ^ (pos >> 3)) & 1) << 3) + w;
        else
            return (k * N + pos) * W + w;
    }
};
// Contiguous fibers: position pos of transform k of fiber f at
// (k*F + f)*N + swz(pos); swz XORs the bank-selecting low bits with higher
// position bits (8-byte: 16 elements per line; 16-byte: 8 per line).
template <int N, int ES>
struct FiberIdx {
    int base;  // f * N
    int kstride;
    __device__ __forceinline__ int operator()(int k, int pos) const
    {
        int sw;
        if constexpr (ES == 8)
            sw = pos ^ (((pos >> 4) & 7) | ((pos >> 3) & 8));
        else
            sw = pos ^ ((pos >> 3) & 7);
        return k * kstride + base + (N >= 16 ? sw : pos);
    }
};

template <typename T, int N>
constexpr int strided_w()
{
    return (N / 8) >= 32 ? 8 : 256 / (N / 8);
}

// ------------------------------------------------------------------- K1/K3

template <typename T>
__device__ __forceinline__ typename cx<T>::t cscale(typename cx<T>::t v, T s)
{
    if constexpr (sizeof(T) == 4)
        return mul2(v, make_float2(s, s));
    else
        return make_c<T>(v.x * s, v.y * s);
}

// MODE 0: K1 forward split (even/odd by use flags); MODE 1: K3 inverse merge.
// Persistent CTAs; the next tile's loads are issued before the current tile's
// transforms so HBM reads overlap the shared-memory exchanges.
template <typename T, int N, int W, int MODE>
__global__ void __launch_bounds__(N / 8 * W) k_strided(tsk_axis p)
{
    using T2 = typename cx<T>::t;
    using T4 = typename tw4<T>::t;
    using PL = Plan<N>;
    constexpr int TF = PL::TF;
    constexpr int NIN = MODE == 0 ? 1 : 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T4* tw = reinterpret_cast<T4*>(smem_raw);
    T4* ph = tw + PL::TW;
    T2* buf0 = reinterpret_cast<T2*>(ph + N);
    T2* buf1 = buf0 + 2 * N * W;
    fill_tables<T, N>(tw, ph, static_cast<const T2*>(p.roots), static_cast<const T2*>(p.phase));
    __syncthreads();

    const int w = threadIdx.x % W;
    const int t = threadIdx.x / W;
    const int64_t inner = p.inner;
    const int64_t cols = inner / W;
    const int64_t tiles_per_comp = p.outer * cols;
    const int64_t ntiles = tiles_per_comp * p.ncomp;
    const bool ue = p.use_even, uo = p.use_odd;
    const T scale = (T)p.scale;
    StridedIdx<N, W, sizeof(T2)> sidx{w};
    const T2* s0 = static_cast<const T2*>(p.src0);
    const T2* s1 = static_cast<const T2*>(p.src1);
    const bool ld0 = MODE == 0 || ue, ld1 = MODE == 1 && uo;
    const int64_t rstride = (int64_t)TF * inner;  // element stride between m and m+1

    const FastDiv div_tpc((uint32_t)tiles_per_comp), div_cols((uint32_t)cols);
    auto tile_base = [&](int64_t tile) {
        // launcher guarantees ntiles < 2^31
        const uint32_t t32 = (uint32_t)tile;
        const uint32_t c32 = div_tpc.div(t32);
        const uint32_t r32 = t32 - c32 * (uint32_t)tiles_per_comp;
        const uint32_t o32 = div_cols.div(r32);
        const int64_t c = c32, o = o32;
        const int64_t i0 = (int64_t)(r32 - o32 * (uint32_t)cols) * W;
        return c * p.cstride + o * (int64_t)N * inner + i0 + w + (int64_t)t * inner;
    };
    T2 nx[NIN][8];
    int xc = 0;
    int64_t tile = blockIdx.x;
    if (tile < ntiles) {
        const int64_t b = tile_base(tile);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            nx[0][m] = ld0 ? s0[b + m * rstride] : make_c<T>(0, 0);
            if (NIN == 2)
                nx[NIN - 1][m] = ld1 ? s1[b + m * rstride] : make_c<T>(0, 0);
        }
    }
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile_base(tile);
        T2 v[2][8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            v[0][m] = nx[0][m];
            if (MODE == 0)
                v[1][m] = cmul_tw<T, false>(nx[0][m], load_tw<T>(ph + t + m * TF));
            else
                v[1][m] = nx[NIN - 1][m];
        }
        const int64_t nt = tile + gridDim.x;
        if (nt < ntiles) {
            const int64_t b = tile_base(nt);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                nx[0][m] = ld0 ? s0[b + m * rstride] : make_c<T>(0, 0);
                if (NIN == 2)
                    nx[NIN - 1][m] = ld1 ? s1[b + m * rstride] : make_c<T>(0, 0);
            }
        }
        if (MODE == 0) {
            fft_rows<T, N, false, 2>(v, buf0, buf1, sidx, tw, t, xc);
            T2* de = static_cast<T2*>(p.dst0) + base;
            T2* dodd = static_cast<T2*>(p.dst1) + base;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (ue)
                    de[m * rstride] = v[0][m];
                if (uo)
                    dodd[m * rstride] = v[1][m];
            }
        } else {
            fft_rows<T, N, true, 2>(v, buf0, buf1, sidx, tw, t, xc);
            T2* dst = static_cast<T2*>(p.dst0) + base;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const T2 acc = cadd(v[0][m], cmul_tw<T, true>(v[1][m], load_tw<T>(ph + t + m * TF)));
                dst[m * rstride] = cscale<T>(acc, scale);
            }
        }
    }
}

// --------------------------------------------------------------------- K2

// Mirror orbit of a stored index s along one axis: the full indices that the
// compressed layout maps to s (ref kernel.cpp:25-37): s itself and, when it
// exists, its mirrored partner.
__device__ __forceinline__ int orbit_members(int64_t n, int odd, int64_t s, int64_t& partner)
{
    const int64_t kp = odd ? n - 1 - s : n - s;
    partner = kp;
    if (kp >= 0 && kp < n && kp != s) {
        bool m;
        if (mirror_src(n, odd, kp, m) == s && m)
            return 2;
    }
    return 1;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T2>
__device__ __forceinline__ T2 flip_sign(T2 v, bool neg)
{
    if (neg) {
        v.x = -v.x;
        v.y = -v.y;
    }
    return v;
}

// y_i = sum_j T_map(i,j) x_j for the block-symmetric 3x3 map
// [[0,1,2],[1,3,4],[2,4,5]] (complex64: packed MACs, 21 instructions).
template <typename T>
__device__ __forceinline__ void matvec3(typename cx<T>::t (&x)[3], const typename cx<T>::t (&sv)[6])
{
    constexpr int cmap[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
    using T2 = typename cx<T>::t;
    T2 y[3];
    if constexpr (sizeof(T) == 4) {
        float2 xn[3];
#pragma unroll
        for (int j = 0; j < 3; ++j)
            xn[j] = mul2(bc_y(x[j]), make_float2(-1.f, 1.f));  // (-x.y, x.y)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            float2 a = mul2(bc_x(x[0]), sv[cmap[i * 3]]);
            a = fma2(xn[0], swz(sv[cmap[i * 3]]), a);
#pragma unroll
            for (int j = 1; j < 3; ++j) {
                a = fma2(bc_x(x[j]), sv[cmap[i * 3 + j]], a);
                a = fma2(xn[j], swz(sv[cmap[i * 3 + j]]), a);
            }
            y[i] = a;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T2 a = make_c<T>(0, 0);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const T2 s = sv[cmap[i * 3 + j]];
                a.x = fma(x[j].x, s.x, fma(-x[j].y, s.y, a.x));
                a.y = fma(x[j].x, s.y, fma(x[j].y, s.x, a.y));
            }
            y[i] = a;
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
        x[i] = y[i];
}

// Leaf pair on the contiguous last axis. A CTA processes G work units of up
// to 4 fibers each. With mirror-compressed spectra a unit is the mirror orbit
// of one stored spectra row over the last two outer axes (+-k_{d-3},
// +-k_{d-2}), so the row is fetched from HBM once and reused from L1 by all
// members (with per-member signs); with full spectra a unit is 4 consecutive
// fibers. Components are transformed one after another through a single pair
// of exchange buffers; the m x m multiply happens in registers. The leaf
// parities along the last axis are even (beta 0) and odd (beta 1).
template <typename T, int N, int M, int G>
__global__ void __launch_bounds__(N / 8 * 4 * G, sizeof(T) == 4 ? 2 : 1) k_leaf(tsk_axis p, tsk_spectra sp)
{
    using T2 = typename cx<T>::t;
    using T4 = typename tw4<T>::t;
    using PL = Plan<N>;
    constexpr int TF = PL::TF;
    constexpr int S = 4 * G;  // fiber slots per CTA
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T4* twt = reinterpret_cast<T4*>(smem_raw);
    T2* buf0 = reinterpret_cast<T2*>(twt + PL::TW);
    T2* buf1 = buf0 + S * N;
    T2* stash = buf1 + S * N;  // M x S x N: x during the even branch, e' during the odd
    // compressed spectra: one branch's stored row of every unique component,
    // per unit, staged with cp.async while the forward transforms run
    constexpr int LROW = N / 2 + 1;
    constexpr int UM = M == 1 ? 1 : 6;
    T2* sstage = stash + M * S * N;  // G x UM x LROW
    {
        // stage tables only (the phase comes from registers)
#pragma unroll
        for (int s = 1; s < PL::NST; ++s) {
            const int pr = PL::radix(s), ns = PL::ns(s);
            for (int e = threadIdx.x; e < ns * (pr - 1); e += blockDim.x) {
                const int jm = e / (pr - 1), r = e % (pr - 1) + 1;
                twt[PL::tw_off(s) + e] =
                    make_tw<T>(ldg_c(static_cast<const T2*>(p.roots) + (r * jm * (N / (ns * pr))) % N));
            }
        }
        __syncthreads();
    }

    const int slot = threadIdx.x / TF;
    const int gi = slot / 4, f = slot % 4;
    const int t = threadIdx.x % TF;
    // per-thread twiddle bases and split phase, loaded once (no table reads
    // inside the transforms)
    // per-thread twiddle bases of the last stage (powers in registers)
    constexpr int SL = PL::NST - 1;
    constexpr int NWR = SL > 0 ? 8 / PL::radix(SL) : 1;
    Tw<T> wreg[NWR];
    if constexpr (SL > 0) {
        const T2* roots = static_cast<const T2*>(p.roots);
        constexpr int pr = PL::radix(SL), ns = PL::ns(SL);
#pragma unroll
        for (int i = 0; i < NWR; ++i) {
            const int jm = (t + i * TF) % ns;
            wreg[i] = make_twv<T>(ldg_c(roots + jm * (N / (ns * pr))));
        }
    }
    PhaseReg<T> phr;
    phr.pt = make_twv<T>(ldg_c(static_cast<const T2*>(p.phase) + t));
    const typename tw4<T>::t* tw = twt;
    constexpr int FT = TF;  // threads per fiber; exchanges sync only those
    const SyncGroup fsync{1 + (int)(threadIdx.x / (FT >= 32 ? FT : 32)), FT >= 32 ? FT : 32};
    const int ut = threadIdx.x - gi * 4 * TF;  // thread index within the unit
    const T scale = (T)p.scale;
    const T2* src = static_cast<const T2*>(p.src0);
    T2* dst = static_cast<T2*>(p.dst0);
    FiberIdx<N, sizeof(T2)> sidx{slot * N, 0};
    const int d = sp.d;
    const int U = sp.n_unique;
    const bool compressed = sp.compressed;
    const uint32_t bits = sp.branch_bits[0];  // outer-axis parities (shared by both leaves)
    uint32_t lastneg = 0;                     // components skew along the leaf axis
    for (int uu = 0; uu < U; ++uu)
        lastneg |= ((sp.skew_mask[uu] >> (d - 1)) & 1u) << uu;
    // orbit axes (last two outer axes) and unit count
    const int A2 = d - 2, A1 = d - 3;
    int64_t n1 = 1, n2 = 1, st1 = 1, st2 = 1, rest = 1;
    if (A2 >= 0) {
        n2 = sp.levels[A2];
        st2 = compressed ? stored_len(n2, (bits >> A2) & 1u) : n2;
    }
    if (A1 >= 0) {
        n1 = sp.levels[A1];
        st1 = compressed ? stored_len(n1, (bits >> A1) & 1u) : n1;
    }
    for (int a = 0; a < A1; ++a)
        rest *= sp.levels[a];
    const int64_t units = compressed ? rest * st1 * st2 : (p.outer + 3) / 4;
    T2* stash_me = stash + slot * N + t;
    int xc = 0;

    for (int64_t tile = blockIdx.x; tile * G < units; tile += gridDim.x) {
        const int64_t u = tile * G + gi;
        bool valid = false;
        int64_t g = 0, off[2] = {0, 0};
        uint32_t neg = 0;
        if (u < units) {
            if (!compressed) {
                g = u * 4 + f;
                valid = g < p.outer;
                off[0] = off[1] = g * N;
            } else {
                // unit -> (rest, s1, s2): 32-bit (units < 2^31), no 64-bit division
                const uint32_t u32 = (uint32_t)u, st2u = (uint32_t)st2, st1u = (uint32_t)st1;
                const uint32_t q2 = u32 / st2u;
                const int64_t s2 = u32 - q2 * st2u;
                const uint32_t q1 = q2 / st1u;
                const int64_t s1 = q2 - q1 * st1u;
                const int64_t r = q1;
                int64_t p1 = 0, p2 = 0;
                const int c1 = A1 >= 0 ? orbit_members(n1, (bits >> A1) & 1u, s1, p1) : 1;
                const int c2 = A2 >= 0 ? orbit_members(n2, (bits >> A2) & 1u, s2, p2) : 1;
                {
                    valid = f < c1 * c2;
                    const int i1 = (f % (c1 * c2)) / c2, i2 = f % c2;
                    const int64_t kk1 = A1 < 0 ? 0 : (i1 ? p1 : s1);
                    const int64_t kk2 = A2 < 0 ? 0 : (i2 ? p2 : s2);
                    for (int uu = 0; uu < U; ++uu) {
                        if (A1 >= 0 && i1)
                            neg ^= ((sp.skew_mask[uu] >> A1) & 1u) << uu;
                        if (A2 >= 0 && i2)
                            neg ^= ((sp.skew_mask[uu] >> A2) & 1u) << uu;
                    }
                    // rest axes (0 .. d-4): plain per-fiber mirror remap
                    int64_t rsrc = 0, rstride_elems = 1, gr = r, rfull = 0, rmul = 1;
                    for (int a = A1 - 1; a >= 0; --a) {
                        const int64_t na = sp.levels[a];
                        const int64_t ka = gr % na;
                        gr /= na;
                        const int odd = (bits >> a) & 1u;
                        bool mm;
                        rsrc += mirror_src(na, odd, ka, mm) * rstride_elems;
                        rstride_elems *= stored_len(na, odd);
                        rfull += ka * rmul;
                        rmul *= na;
                        if (mm)
                            for (int uu = 0; uu < U; ++uu)
                                neg ^= ((sp.skew_mask[uu] >> a) & 1u) << uu;
                    }
                    g = (rfull * n1 + kk1) * n2 + kk2;
                    const int64_t row = (rsrc * st1 + s1) * st2 + s2;
                    off[0] = row * (N / 2 + 1);
                    off[1] = row * (N / 2);
                }
            }
        }
        const T2* xin = src + g * N + t;
        T2* stg = sstage + gi * UM * LROW;
        auto stage = [&](int beta) {
            if (!compressed || u >= units)
                return;
            const int L = beta ? N / 2 : N / 2 + 1;
            const T2* row = static_cast<const T2*>(sp.data) + sp.branch_base[beta] + off[beta];
            for (int e = ut; e < UM * L; e += 4 * TF) {
                const int uu = e / L, kk = e - uu * L;
                if constexpr (sizeof(T2) == 8)
                    cp_async8(stg + uu * LROW + kk, row + uu * sp.block_elems[beta] + kk);
                else
                    cp_async16(stg + uu * LROW + kk, row + uu * sp.block_elems[beta] + kk);
            }
            cp_async_commit();
        };
        // every member thread computed the same unit row; slot-0 threads hold it
        // whether or not their own fiber is valid (row offsets depend on the unit)
        stage(p.use_even ? 0 : 1);
        T2 v[M][8];
#pragma unroll
        for (int beta = 0; beta < 2; ++beta) {
            const bool use = beta ? p.use_odd : p.use_even;
            if (!use)
                continue;
#pragma unroll
            for (int c = 0; c < M; ++c)
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    T2* sl = stash_me + c * S * N + m * TF;
                    if (beta == 0) {
                        T2 x = make_c<T>(0, 0);
                        if (valid)
                            x = xin[c * p.cstride + m * TF];
                        if (p.use_odd)
                            *sl = x;
                        v[c][m] = x;
                    } else if (!p.use_even) {
                        T2 x = make_c<T>(0, 0);
                        if (valid)
                            x = xin[c * p.cstride + m * TF];
                        v[c][m] = phr.template apply<false>(x, m);
                    } else {
                        const T2 x = *sl;
                        *sl = v[c][m];  // e' of the even branch
                        v[c][m] = phr.template apply<false>(x, m);
                    }
                }
#pragma unroll
            for (int c = 0; c < M; ++c)
                fft_rows<T, N, false, 1, FiberIdx<N, sizeof(T2)>, SyncGroup, LEAF_REGTW, Tw<T>[NWR]>(
                    *reinterpret_cast<T2(*)[1][8]>(&v[c]), buf0, buf1, sidx, tw, t, xc, fsync, wreg);
            const T2* sb = static_cast<const T2*>(sp.data) + sp.branch_base[beta] + off[beta];
            const int64_t bst = sp.block_elems[beta];
            if (compressed) {
                cp_async_wait_all();
                __syncthreads();  // the staged row is complete and visible
            }
            constexpr int MB = 1;  // frequencies per spectra batch
#pragma unroll
            for (int mb = 0; mb < 8; mb += MB) {
                int kidx[MB];
                uint32_t ngs[MB];
#pragma unroll
                for (int mm = 0; mm < MB; ++mm) {
                    const int k = t + (mb + mm) * TF;
                    int ki = k;
                    bool mir = false;
                    if (compressed) {
                        // beta 0: even parity (stores 0..N/2), beta 1: odd (0..N/2-1)
                        if (beta == 0) {
                            mir = k > N / 2;
                            ki = mir ? N - k : k;
                        } else {
                            mir = k >= N / 2;
                            ki = mir ? N - 1 - k : k;
                        }
                    }
                    kidx[mm] = ki;
                    ngs[mm] = neg ^ (mir ? lastneg : 0u);
                }
                if (M == 1) {
                    T2 sv[MB];
#pragma unroll
                    for (int mm = 0; mm < MB; ++mm) {
                        sv[mm] = make_c<T>(0, 0);
                        if (compressed)
                            sv[mm] = stg[kidx[mm]];
                        else if (valid)
                            sv[mm] = ldg_c(sb + kidx[mm]);
                    }
#pragma unroll
                    for (int mm = 0; mm < MB; ++mm)
                        v[0][mb + mm] = cmul(v[0][mb + mm], flip_sign(sv[mm], ngs[mm] & 1u));
                } else {
                    // 4 frequencies x 6 unique components loaded together, then
                    // four 3x3 products
                    T2 sv[MB][6];
#pragma unroll
                    for (int mm = 0; mm < MB; ++mm)
#pragma unroll
                        for (int uu = 0; uu < 6; ++uu) {
                            T2 sx = make_c<T>(0, 0);
                            if (compressed)
                                sx = stg[uu * LROW + kidx[mm]];
                            else if (valid)
                                sx = ldg_c(sb + uu * bst + kidx[mm]);
                            sv[mm][uu] = sx;
                        }
#pragma unroll
                    for (int mm = 0; mm < MB; ++mm) {
#pragma unroll
                        for (int uu = 0; uu < 6; ++uu)
                            sv[mm][uu] = flip_sign(sv[mm][uu], (ngs[mm] >> uu) & 1u);
                        T2 x[3] = {v[0][mb + mm], v[1][mb + mm], v[2][mb + mm]};
                        matvec3<T>(x, sv[mm]);
#pragma unroll
                        for (int c = 0; c < 3; ++c)
                            v[c][mb + mm] = x[c];
                    }
                }
                // compiler barrier between the two halves: bounds the number of
                // spectra values held in registers (all 48 at once spills)
                asm volatile("" ::: "memory");
            }
            if (compressed) {
                __syncthreads();  // everyone is done with the staged row
                if (beta == 0 && p.use_odd)
                    stage(1);  // lands while this branch's inverse transforms run
            }
#pragma unroll
            for (int c = 0; c < M; ++c)
                fft_rows<T, N, true, 1, FiberIdx<N, sizeof(T2)>, SyncGroup, LEAF_REGTW, Tw<T>[NWR]>(
                    *reinterpret_cast<T2(*)[1][8]>(&v[c]), buf0, buf1, sidx, tw, t, xc, fsync, wreg);
        }
        if (valid) {
            T2* yout = dst + g * N + t;
#pragma unroll
            for (int c = 0; c < M; ++c)
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    T2 a;
                    if (p.use_odd) {
                        a = phr.template apply<true>(v[c][m], m);
                        if (p.use_even)
                            a = cadd(a, stash_me[c * S * N + m * TF]);
                    } else {
                        a = v[c][m];
                    }
                    yout[c * p.cstride + m * TF] = cscale<T>(a, scale);
                }
        }
    }
}

// ---------------------------------------------------------------- launchers

static int sm_count()
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

// Per-kernel one-time setup: opt in to the dynamic shared memory and cache
// the occupancy-derived persistent grid (resident CTAs per SM x SMs).
template <typename K>
static int prep(K kernel, size_t smem, int threads, int& grid_cap)
{
    static thread_local struct {
        const void* k = nullptr;
        int dev = -1;
        int cap = 0;
    } cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    const void* key = reinterpret_cast<const void*>(kernel);
    for (auto& c : cache)
        if (c.k == key && c.dev == dev) {
            grid_cap = c.cap;
            return 0;
        }
    int e = (int)cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e)
        return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    grid_cap = sm_count() * std::max(per_sm, 1);
    for (auto& c : cache)
        if (!c.k) {
            c.k = key;
            c.dev = dev;
            c.cap = grid_cap;
            break;
        }
    return 0;
}

template <typename T, int N, int MODE>
static int launch_strided(const tsk_axis& a, cudaStream_t st)
{
    constexpr int W = strided_w<T, N>();
    using T2 = typename cx<T>::t;
    const size_t smem = 2 * sizeof(T2) * (Plan<N>::TW + N) + sizeof(T2) * 2 * 2 * N * W;
    if (smem > 227 * 1024)
        return -1;
    auto kern = k_strided<T, N, W, MODE>;
    int cap = 0;
    if (int e = prep(kern, smem, N / 8 * W, cap))
        return e;
    const int64_t ntiles = a.outer * (a.inner / W) * a.ncomp;
    if (ntiles >= (int64_t(1) << 31))
        return -1;  // 32-bit tile decomposition
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, cap));
    kern<<<(unsigned)grid, N / 8 * W, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <typename T, int N, int M>
static int launch_leaf(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    constexpr int G = (N / 8 * 4 >= 256) ? 1 : 256 / (N / 8 * 4);
    constexpr int S = 4 * G;
    using T2 = typename cx<T>::t;
    const size_t smem = 2 * sizeof(T2) * Plan<N>::TW + sizeof(T2) * (2 + M) * S * N +
                        sizeof(T2) * G * (M == 1 ? 1 : 6) * (N / 2 + 1);
    if (smem > 227 * 1024)
        return -1;
    auto kern = k_leaf<T, N, M, G>;
    int cap = 0;
    if (int e = prep(kern, smem, N / 8 * S, cap))
        return e;
    // work units: mirror orbits (compressed) or groups of 4 fibers
    int64_t units;
    if (sp.compressed) {
        const int d = sp.d;
        units = 1;
        for (int ax = 0; ax < d - 1; ++ax) {
            const bool orbit_axis = ax >= d - 3;
            units *= orbit_axis ? stored_len(sp.levels[ax], (sp.branch_bits[0] >> ax) & 1u)
                                : sp.levels[ax];
        }
    } else {
        units = (a.outer + 3) / 4;
    }
    const int64_t ntiles = (units + G - 1) / G;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, cap));
    kern<<<(unsigned)grid, N / 8 * S, smem, st>>>(a, sp);
    return (int)cudaGetLastError();
}

template <typename T, int MODE>
static int dispatch_strided(const tsk_axis& a, cudaStream_t st)
{
    switch (a.n) {
    case 8: return launch_strided<T, 8, MODE>(a, st);
    case 16: return launch_strided<T, 16, MODE>(a, st);
    case 32: return launch_strided<T, 32, MODE>(a, st);
    case 64: return launch_strided<T, 64, MODE>(a, st);
    case 128: return launch_strided<T, 128, MODE>(a, st);
    case 256: return launch_strided<T, 256, MODE>(a, st);
    case 512: return launch_strided<T, 512, MODE>(a, st);
    default: return -1;
    }
}

template <typename T, int M>
static int dispatch_leaf(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    switch (a.n) {
    case 8: return launch_leaf<T, 8, M>(a, sp, st);
    case 16: return launch_leaf<T, 16, M>(a, sp, st);
    case 32: return launch_leaf<T, 32, M>(a, sp, st);
    case 64: return launch_leaf<T, 64, M>(a, sp, st);
    case 128: return launch_leaf<T, 128, M>(a, sp, st);
    case 256: return launch_leaf<T, 256, M>(a, sp, st);
    case 512: return launch_leaf<T, 512, M>(a, sp, st);
    default: return -1;
    }
}

}  // namespace fast
}  // namespace tsk

using namespace tsk::fast;

// Return -1 when the pass shape is not covered (caller falls back to the
// generic kernels), otherwise the cudaError_t of the launch.
static int64_t strided_w_rt(int64_t n)
{
    return (n / 8) >= 32 ? 8 : 256 / (n / 8 > 0 ? n / 8 : 1);
}

extern "C" int tsk_fast_fwd_split(const tsk_axis* a, void* stream)
{
    const int64_t W = strided_w_rt(a->n);
    if (a->inner < W || a->inner % W != 0)
        return -1;
    return a->prec ? dispatch_strided<float, 0>(*a, (cudaStream_t)stream)
                   : dispatch_strided<double, 0>(*a, (cudaStream_t)stream);
}

extern "C" int tsk_fast_inv_merge(const tsk_axis* a, void* stream)
{
    const int64_t W = strided_w_rt(a->n);
    if (a->inner < W || a->inner % W != 0)
        return -1;
    return a->prec ? dispatch_strided<float, 1>(*a, (cudaStream_t)stream)
                   : dispatch_strided<double, 1>(*a, (cudaStream_t)stream);
}

extern "C" int tsk_fast_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    if (a->inner != 1)
        return -1;
    auto st = (cudaStream_t)stream;
    if (sp->m == 1)
        return a->prec ? dispatch_leaf<float, 1>(*a, *sp, st) : dispatch_leaf<double, 1>(*a, *sp, st);
    static const int8_t canon[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
    bool canonical = sp->n_unique == 6;
    for (int i = 0; i < 9 && canonical; ++i)
        canonical = sp->comp_map[i] == canon[i];
    if (sp->m == 3 && canonical)
        return a->prec ? dispatch_leaf<float, 3>(*a, *sp, st) : dispatch_leaf<double, 3>(*a, *sp, st);
    return -1;
}
