// Leaf-pair pass (K2) with one component per thread and R = N/16..N/8
// elements per thread: a length-N transform is two in-register stages (radix
// R, then N/R) and ONE shared-memory exchange among the TF = N/R threads of a
// (fiber, component) — a half or quarter warp, synchronised with __syncwarp.
// The m x m spectra multiply couples the components once per branch: through
// tensor memory (the component warps of a (fiber, t) share a TMEM lane; see
// MIXT) with compressed storage, through shared memory otherwise. Tensor memory
// also holds, per lane, the stage-B twiddles and the split phase (TWT), and
// the even branch's output e' while the odd branch runs; the odd branch
// re-reads x (an L1 hit). The pass is bound by the FP32 and L1/shared pipes,
// not HBM, so TMEM serves as a second on-chip datapath (3x the shared-memory
// read bandwidth, tools/micro/pipes.cu). A unit is one mirror orbit of 4
// fibers (compressed spectra rows fetched once, cp.async-staged) or, with full
// storage, 4 consecutive fibers (spectra read straight from global memory,
// each element once), m components each.
//
// Reference semantics (relative to /root/reference/proj): leaf multiply
// src/core/kernel.cpp:126-219, leaf FFT/IFFT and deepest merge
// src/core/engine_split.cpp:67-99, mirror remap kernel.cpp:17-37.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "tsk_common.cuh"
#include "tsk_tmem.cuh"
#include "tsk_wide.cuh"

namespace tsk {
namespace leaf {

using wide::Dft;
using wide::Plan;
using wide::Tw;

// Members of the mirror orbit of stored index s along an axis of length n
// (1 or 2) and the partner index; 32-bit (every axis length fits).
__device__ __forceinline__ int orbit_members(int n, int odd, int s, int& partner)
{
    const int kp = odd ? n - 1 - s : n - s;
    partner = kp;
    // kp mirrors back onto s (ref kernel.cpp:25-37) iff it lies past the
    // stored half: odd parity stores [0, (n+1)/2), even [0, n/2]
    const bool mirrored = odd ? kp >= (n + 1) / 2 : kp > n / 2;
    return kp < n && kp != s && mirrored ? 2 : 1;
}


__device__ __forceinline__ void cp_async_bytes8(void* smem, const void* gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_bytes16(void* smem, const void* gmem)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

template <typename T2>
__device__ __forceinline__ T2 neg_if(T2 v, bool neg)
{
    if (neg) {
        v.x = -v.x;
        v.y = -v.y;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ Tw<T> twv(typename cx<T>::t w)
{
    Tw<T> r;
    r.lo = w;
    if constexpr (sizeof(T) == 4)
        r.hi = mul2(swz(w), make_float2(-1.f, 1.f));
    else
        r.hi = make_c<T>(-w.y, w.x);
    return r;
}

// v * P_k at k = t + TF m: P_t (register) times exp(-i pi m / R) (constant)
template <typename T, int R, bool CONJ>
struct PhaseR {
    template <int Mi>
    __device__ __forceinline__ static typename cx<T>::t apply(typename cx<T>::t v, const Tw<T>& pt)
    {
        // exp(-+ 2 pi i Mi / (2R)); CONJ flips the sign
        v = wide::cmul_const<T, 2 * R, Mi, CONJ>(v);
        return wide::cmul_tw<T, CONJ>(v, pt);
    }
};

// Exchange-buffer layout: one pad element per R, so a thread's R-run
// (t R + q) and the row pattern (t + TF m) are both bank-conflict free and
// affine in t (addresses are a base register plus immediates).
template <int N, int R>
struct Pad {
    static constexpr int TF = N / R;
    static constexpr int NP = N + N / R;  // buffer pitch
    __device__ __forceinline__ static int wr(int t, int q) { return t * (R + 1) + q; }
    __device__ __forceinline__ static int rd(int t, int m) { return t + TF * m + (TF * m) / R; }
};

// s with both parts' sign bits flipped when neg (integer pipe, not FMA)
template <typename T>
__device__ __forceinline__ typename cx<T>::t flip_bits(typename cx<T>::t s, uint32_t neg)
{
    if constexpr (sizeof(T) == 4) {
        const uint32_t b = neg << 31;
        return make_float2(__uint_as_float(__float_as_uint(s.x) ^ b),
                           __uint_as_float(__float_as_uint(s.y) ^ b));
    } else {
        const long long b = (long long)neg << 63;
        return make_double2(__longlong_as_double(__double_as_longlong(s.x) ^ b),
                            __longlong_as_double(__double_as_longlong(s.y) ^ b));
    }
}

// acc (+)= x * s; packed f32x2: x s = s.x x + s.y (i x)
template <typename T>
__device__ __forceinline__ typename cx<T>::t cmac(typename cx<T>::t acc, typename cx<T>::t x,
                                                  typename cx<T>::t s, bool first)
{
    if constexpr (sizeof(T) == 4) {
        const float2 a = first ? mul2(x, bc_x(s)) : fma2(x, bc_x(s), acc);
        return fma2(make_float2(-x.y, x.x), bc_y(s), a);
    } else {
        const typename cx<T>::t pr = cmul(x, s);
        return first ? pr : cadd(acc, pr);
    }
}

// acc (+)= -x * s
template <typename T>
__device__ __forceinline__ typename cx<T>::t cmac_neg(typename cx<T>::t acc, typename cx<T>::t x,
                                                      typename cx<T>::t s, bool first)
{
    if constexpr (sizeof(T) == 4) {
        const float2 nx = make_float2(-x.x, -x.y);
        const float2 a = first ? mul2(nx, bc_x(s)) : fma2(nx, bc_x(s), acc);
        return fma2(make_float2(x.y, -x.x), bc_y(s), a);
    } else {
        const typename cx<T>::t pr = cmul(x, s);
        return first ? make_c<T>(-pr.x, -pr.y) : csub(acc, pr);
    }
}

// e + o conj(w); packed f32x2: e rides on the first FFMA2 (w.x o + e, then
// - w.y (i o)), one instruction fewer than a product and a sum
template <typename T>
__device__ __forceinline__ typename cx<T>::t cmulc_add(typename cx<T>::t o, typename cx<T>::t w,
                                                       typename cx<T>::t e)
{
    if constexpr (sizeof(T) == 4)
        return fma2(make_float2(o.y, -o.x), bc_y(w), fma2(o, bc_x(w), e));
    else
        return cadd(cmulc(o, w), e);
}

// a + e * scale
template <typename T>
__device__ __forceinline__ typename cx<T>::t fma_s(typename cx<T>::t e, T scale, typename cx<T>::t a)
{
    if constexpr (sizeof(T) == 4)
        return fma2(e, make_float2(scale, scale), a);
    else
        return make_c<T>(e.x * scale + a.x, e.y * scale + a.y);
}

// acc (+)= sgn * x * s; packed f32x2: x s = x.x s + x.y (i s)
template <typename T>
__device__ __forceinline__ typename cx<T>::t cmac_sgn(typename cx<T>::t acc, typename cx<T>::t x,
                                                      typename cx<T>::t s, T sgn, bool first)
{
    if constexpr (sizeof(T) == 4) {
        const float2 ss = mul2(s, make_float2(sgn, sgn));
        const float2 rs = mul2(swz(s), make_float2(-sgn, sgn));
        const float2 a = first ? mul2(bc_x(x), ss) : fma2(bc_x(x), ss, acc);
        return fma2(bc_y(x), rs, a);
    } else {
        const typename cx<T>::t ss = make_c<T>(s.x * sgn, s.y * sgn);
        const typename cx<T>::t pr = cmul(x, ss);
        return first ? pr : cadd(acc, pr);
    }
}

template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f)
{
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        sfor<B + 1, E>(f);
    }
}

// One length-N transform of this thread's row pattern v[m] = x[t + TF m].
// TWT: the stage-B twiddles of this thread's two butterflies come from its
// TMEM lane (32 columns per butterfly at twt) instead of the shared table.
template <typename T, int N, int R, bool INV, bool TWT = false>
__device__ __forceinline__ void fft_one(typename cx<T>::t (&v)[R], typename cx<T>::t* buf,
                                        const typename cx<T>::t* tw, int t, uint32_t twt = 0)
{
    using T2 = typename cx<T>::t;
    constexpr int TF = N / R;
    constexpr int P2 = N / R;
    constexpr int G2 = R / P2;
    static_assert(P2 <= R, "two-stage plan needs N <= R^2");
    // stage A: radix R, butterfly j = t (Ns = 1) -> positions t*R + q
    Dft<T, R, INV>::run(v);
#pragma unroll
    for (int q = 0; q < R; ++q)
        buf[Pad<N, R>::wr(t, q)] = v[q];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < R; ++m)
        v[m] = buf[Pad<N, R>::rd(t, m)];
    __syncwarp();
    // stage B: radix P2, Ns = R, butterflies j = t + i TF (i < G2), twiddle w_N^{r j}
#pragma unroll
    for (int i = 0; i < G2; ++i) {
        const int j = t + i * TF;
        T2 a[P2];
        a[0] = v[i];
        if constexpr (TWT) {
            static_assert(sizeof(T2) == 8 && P2 == 16, "TMEM twiddles: complex64, radix 16");
            uint32_t r32[32];
            tmem_ld32(twt + 32 * i, r32);  // waits
#pragma unroll
            for (int r = 1; r < P2; ++r) {
                Tw<T> w;
                w.lo = Words<T2>::make(r32 + 2 * (r - 1));
                w.hi = w.lo;
                a[r] = wide::cmul_tw<T, INV>(v[i + r * G2], w);
            }
        } else {
#pragma unroll
            for (int r = 1; r < P2; ++r) {
                const Tw<T> w = wide::load_tw<T>(tw + j * (P2 - 1) + (r - 1));
                a[r] = wide::cmul_tw<T, INV>(v[i + r * G2], w);
            }
        }
        Dft<T, P2, INV>::run(a);
#pragma unroll
        for (int q = 0; q < P2; ++q)
            v[i + q * G2] = a[q];
        asm volatile("" ::: "memory");  // bound the twiddle loads in flight
    }
}

// Components meet in tensor memory (MIXT): the threads of one (unit, fiber,
// t) in the M component warps share a TMEM lane (warps q, q+4, q+8), so each
// writes its transform to its own column block of that lane and reads the
// others' — the exchange uses the TMEM datapath instead of the shared-memory
// pipe, which the FFT exchanges and the spectra reads keep busy.
#ifndef TSK_LEAF_MIXT
#define TSK_LEAF_MIXT 1
#endif
#ifndef TSK_LEAF_XS
#define TSK_LEAF_XS 1
#endif
// Streaming (st.global.cs, evict-first) output stores: K2 0.346 -> 0.341 ms at
// 256^3, neutral at 512^3 (profiles/r02_ab_stcs.txt)
#ifndef TSK_LEAF_STCS
#define TSK_LEAF_STCS 1
#endif
// TSK_LEAF_LDEF=1 (A/B): the x-row bulk copies carry an L2 evict-first policy
#ifndef TSK_LEAF_LDEF
#define TSK_LEAF_LDEF 0
#endif
#ifndef TSK_LEAF_XC
#define TSK_LEAF_XC 0
#endif
// (Compressed storage only: with full storage the leaf reads each fiber's own
// spectra from global memory and the extra registers of the TMEM chunks spill,
// measured 3.83 -> 4.33 ms per launch at 512^3.)
template <typename T, int R, int M, bool CMP>
constexpr bool leaf_mixt()
{
    return TSK_LEAF_MIXT && CMP && M > 1 && (R * (int)sizeof(typename cx<T>::t) / 4) % 32 == 0;
}
#ifndef TSK_LEAF_TWT
#define TSK_LEAF_TWT 1
#endif
#ifndef TSK_LEAF_FS512
#define TSK_LEAF_FS512 1
#endif
// Stage-B twiddles (32 columns per radix-16 butterfly of a thread, R / 16 of
// them) and the split phase (2R columns) in TMEM after the exchange blocks:
// complex64, radix-16 stage B (N = 512 at R = 32, N = 256 at R = 16).
template <typename T, int N, int R, int M, bool CMP, int NW>
constexpr bool leaf_twt()
{
    constexpr int EW = R * (int)sizeof(typename cx<T>::t) / 4;
    return TSK_LEAF_TWT && leaf_mixt<T, R, M, CMP>() && sizeof(T) == 4 && N / R == 16 && R % 16 == 0 &&
           2 * EW * ((NW + 3) / 4) + 64 * (R / 16) <= 512;
}
// TMEM columns per CTA: e' park (+ component exchange, + twiddles and phase)
template <typename T, int N, int R, int M, bool CMP, int NW>
constexpr int leaf_tcols()
{
    constexpr int EW = R * (int)sizeof(typename cx<T>::t) / 4;
    return tmem_cols_pow2(EW * ((NW + 3) / 4) * (leaf_mixt<T, R, M, CMP>() ? 2 : 1) +
                          (leaf_twt<T, N, R, M, CMP, NW>() ? 64 * (R / 16) : 0));
}

// units (orbits) per CTA: warps per CTA a multiple of 4 (even split over the
// SM sub-partitions' register files)
constexpr int gcd_i(int a, int b) { return b == 0 ? a : gcd_i(b, a % b); }
template <int N, int R, int M>
constexpr int leaf1_g()
{
    return 128 / gcd_i(128, 4 * M * (N / R));
}

// FS (factorised signs; 3x3, d = 3, compressed, with the dyadic sign
// structure skew_mask(i, j) = axis i XOR axis j): the mirror sign of block
// (C, c') under the mirrored axis set F is s_C(F) s_c'(F), s_c(F) = -1 iff
// axis c is in F. Component c's thread flips its transform by s_c once (c = 0,
// 1: a per-fiber sign; c = 2: the leaf axis, known per element at compile
// time), and y_C = s_C sum_c' T_Cc' (s_c' x_c'): the output sign folds into
// the output scale (C = 0, 1) or into the partner terms (C = 2). No per-value
// sign flips on the spectra reads.
template <typename T, int N, int R, int M, bool CMP, bool MRHS, bool FS = false, int G = leaf1_g<N, R, M>()>
// 16 elements per thread fit two 384-thread CTAs per SM (80 registers, 24
// warps): the 256-point leaf 0.41 -> 0.365 ms at 256^3
#ifndef TSK_LEAF256_2CTA
#define TSK_LEAF256_2CTA 1
#endif
// Short leaves (N = 64, complex64, 3x3: 384 threads) at two CTAs per SM as
// well: their passes are a wave or two of tiles (configs[1]: 256 tiles), so a
// second resident CTA per SM removes the second round
#ifndef TSK_LEAF_SHORT_2CTA
#define TSK_LEAF_SHORT_2CTA 1
#endif
__global__ void __launch_bounds__(G * 4 * M * (N / R), sizeof(T) == 4 && G * 4 * M * (N / R) < 384 ? 384 / (G * 4 * M * (N / R)) : (TSK_LEAF256_2CTA && sizeof(T) == 4 && R == 16 && N == 256 ? 2 : (TSK_LEAF_SHORT_2CTA && sizeof(T) == 4 && N <= 64 ? 2 : 1))) k_leaf1(tsk_axis p, tsk_spectra sp)
{
    using T2 = typename cx<T>::t;
    constexpr int TF = N / R;
    constexpr int P2 = N / R;
    constexpr int CF = 4 * M;  // (fiber, component) groups per CTA
    constexpr int UT = CF * TF;  // threads per unit
    constexpr int NT = G * UT;
    constexpr int NP = Pad<N, R>::NP;
    constexpr int LROW = N / 2 + 1;
    constexpr int UM = M == 1 ? 1 : 6;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T2* tw = reinterpret_cast<T2*>(smem_raw);         // R x (P2 - 1) stage-B twiddles
    T2* bufs = tw + R * (P2 - 1);                      // G x CF x NP exchange / mix buffers
    T2* stg0 = bufs + G * CF * NP;                     // G x UM x LROW staged spectra rows
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t xbar[G];          // XS: x rows landed

    for (int e = threadIdx.x; e < R * (P2 - 1); e += NT) {
        const int j = e / (P2 - 1), r = e % (P2 - 1) + 1;
        tw[e] = ldg_c(static_cast<const T2*>(p.roots) + (r * j) % N);
    }

    // thread layout [component][unit][fiber][t]: the component is warp-uniform
    // (the spectra multiply is specialised per component, no divergence)
    const int c = threadIdx.x / (G * 4 * TF);
    const int fs = (threadIdx.x / TF) % (G * 4);
    const int gi = fs / 4, f = fs % 4;
    const int t = threadIdx.x % TF;
    const int lt = (c * 4 + f) * TF + t;  // index among this unit's threads
    const int cf = f * M + c;
    T2* buf = bufs + (gi * CF + cf) * NP;
    T2* fbufs = bufs + gi * CF * NP;  // this unit's component buffers
    T2* stg = stg0 + gi * UM * LROW;
    // each unit (6 warps for m = 3) synchronises on its own named barrier, so
    // the units of a CTA drift apart and overlap memory with arithmetic
    auto unit_sync = [gi]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "n"(UT) : "memory"); };
    const Tw<T> pt = twv<T>(ldg_c(static_cast<const T2*>(p.phase) + t));
    // output scale 1/(2n) folded into the odd branch's conj phase and the
    // merge FMA (the spectra multiply only flips signs)
    const T scale = (T)p.scale;
    const Tw<T> pts = twv<T>(make_c<T>(pt.lo.x * scale, pt.lo.y * scale));

    // e' parked in TMEM when it is a multiple of 32 words, else in registers
    constexpr int EW = R * (int)sizeof(T2) / 4;
    constexpr bool TM = EW % 32 == 0;
    constexpr int NW = NT / 32 > 0 ? NT / 32 : 1;
    constexpr int TCOLS = leaf_tcols<T, N, R, M, CMP, NW>();
    constexpr bool MIXT = leaf_mixt<T, R, M, CMP>();
    constexpr int MIXOFF = EW * ((NW + 3) / 4);  // first column of the exchange blocks
    // stage-B twiddles in TMEM (after the exchange blocks; 64 columns)
    constexpr bool TWT = leaf_twt<T, N, R, M, CMP, NW>();
    constexpr int TWOFF = 2 * MIXOFF;
    static_assert(!FS || (TWT && M == 3 && CMP), "factorised signs: 3x3, compressed, TMEM twiddles");
    constexpr int PHOFF = TWOFF + 32 * (R / 16);  // phase table (TWT: 2R columns)
    uint32_t tbase = 0, lane_base = 0;
    if constexpr (TM) {
        tbase = tmem_alloc(&tmem_slot, TCOLS);
        lane_base = tbase + ((uint32_t)(32 * ((threadIdx.x / 32) % 4)) << 16) +
                    (uint32_t)(EW * ((threadIdx.x / 32) / 4));
        if constexpr (TWT) {
            // the first warp of each lane quadrant writes its lanes' twiddles
            // w_N^{r j}, j = t + i TF (the component warps of a lane share t)
            if ((threadIdx.x / 32) / 4 == 0) {
                const int tl = threadIdx.x % TF;
                const uint32_t q = tbase + ((uint32_t)(32 * ((threadIdx.x / 32) % 4)) << 16) + TWOFF;
#pragma unroll
                for (int i = 0; i < R / 16; ++i) {
                    uint32_t r32[32];
#pragma unroll
                    for (int r = 1; r < 16; ++r) {
                        const T2 w = ldg_c(static_cast<const T2*>(p.roots) + (r * (tl + i * TF)) % N);
                        r32[2 * (r - 1)] = __float_as_uint(w.x);
                        r32[2 * (r - 1) + 1] = __float_as_uint(w.y);
                    }
                    r32[30] = r32[31] = 0u;
                    tmem_st32(q + 32 * i, r32);
                }
                // split phase P_k = exp(-i pi k / N) at this lane's k = t + TF m
#pragma unroll
                for (int h = 0; h < R / 16; ++h) {
                    uint32_t r32[32];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const T2 w = ldg_c(static_cast<const T2*>(p.phase) + tl + TF * (16 * h + i));
                        r32[2 * i] = __float_as_uint(w.x);
                        r32[2 * i + 1] = __float_as_uint(w.y);
                    }
                    tmem_st32(q + 32 * (R / 16) + 32 * h, r32);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
    } else {
        __syncthreads();
    }

    // lane quadrant of this warp (its partners' exchange blocks, the twiddles)
    const uint32_t quad = tbase + ((uint32_t)(32 * ((threadIdx.x / 32) % 4)) << 16);
    const int d = sp.d;
    const int U = sp.n_unique;
    const bool ue = p.use_even, uo = p.use_odd, both = ue && uo;
    const uint32_t bits = sp.branch_bits[0];
    uint32_t lastneg = 0;
    for (int uu = 0; uu < U; ++uu)
        lastneg |= ((sp.skew_mask[uu] >> (d - 1)) & 1u) << uu;
    // orbit axes: the last two outer axes (A1, A2); unit = (rest, s1, s2)
    const int A2 = d - 2, A1 = d - 3;
    int64_t n1 = 1, n2 = 1, st1 = 1, st2 = 1;
    if (A2 >= 0) {
        n2 = sp.levels[A2];
        st2 = stored_len(n2, (bits >> A2) & 1u);
    }
    if (A1 >= 0) {
        n1 = sp.levels[A1];
        st1 = stored_len(n1, (bits >> A1) & 1u);
    }
    int64_t rest = 1;
    for (int a = 0; a < A1; ++a)
        rest *= sp.levels[a];
    // per-axis masks of the unique components that are skew along the axis
    auto axis_mask = [&](int a) {
        uint32_t mk = 0;
        for (int uu = 0; uu < U; ++uu)
            mk |= ((sp.skew_mask[uu] >> a) & 1u) << uu;
        return mk;
    };
    const uint32_t mask1 = A1 >= 0 ? axis_mask(A1) : 0u, mask2 = A2 >= 0 ? axis_mask(A2) : 0u;
    const FastDiv div2((uint32_t)st2), div1((uint32_t)st1);
    // compressed: one unit = one mirror orbit; full storage: 4 consecutive
    // fibers; times nrhs right-hand sides, the RHS index fastest so that the
    // units sharing a spectra row run side by side (one HBM fetch per row)
    // (MRHS: a separate instantiation, so the single-vector pass keeps its
    // register budget)
    const int64_t nrhs = MRHS && p.nrhs > 1 ? p.nrhs : 1;
    const FastDiv divr((uint32_t)nrhs);
    const int64_t units = (CMP ? rest * st1 * st2 : (p.outer + 3) / 4) * nrhs;
    const T2* src0 = static_cast<const T2*>(p.src0);
    T2* dst0 = static_cast<T2*>(p.dst0);
    const T2* spec = static_cast<const T2*>(sp.data);
    T2 ekeep[TM ? 1 : R];

    // ---- unit geometry: fiber g of orbit member f, spectra row offsets,
    // signs. Members past the orbit size alias a real member (loads stay in
    // range) and skip the store.
    auto geometry = [&](int64_t u, bool uvalid, bool& valid, int64_t& g, int64_t& off0, int64_t& off1,
                        uint32_t& neg) {
        neg = 0;
        if constexpr (!CMP) {
            g = u * 4 + f;
            valid = uvalid && g < p.outer;
            if (g >= p.outer)
                g = p.outer - 1;
            off0 = off1 = g * N;
        } else if constexpr (FS && N == 512) {
            // d = 3 (FS): orbit axes 0 and 1, no rest axes (units = st1 st2)
            // (at N = 256 the 80-register pass spills with this variant)
            const uint32_t u32 = (uint32_t)u;
            const uint32_t q2 = div2.div(u32);
            const int s2 = (int)(u32 - q2 * (uint32_t)st2), s1 = (int)q2;
            int p1 = 0, p2 = 0;
            const int c1 = orbit_members((int)n1, bits & 1u, s1, p1);
            const int c2 = orbit_members((int)n2, (bits >> 1) & 1u, s2, p2);
            valid = uvalid && f < c1 * c2;
            const int i1 = c2 == 2 ? (f >> 1) & (c1 - 1) : f & (c1 - 1), i2 = f & (c2 - 1);
            neg = (i1 ? mask1 : 0u) ^ (i2 ? mask2 : 0u);
            g = (int64_t)((i1 ? p1 : s1) * (int)n2 + (i2 ? p2 : s2));
            const int row = s1 * (int)st2 + s2;
            off0 = (int64_t)row * (N / 2 + 1);
            off1 = (int64_t)row * (N / 2);
        } else {
            // units < 2^31 (stored elements per component fit int32 here)
            const uint32_t u32 = (uint32_t)u;
            const uint32_t q2 = div2.div(u32), q1 = div1.div(q2);
            const int s2 = (int)(u32 - q2 * (uint32_t)st2), s1 = (int)(q2 - q1 * (uint32_t)st1);
            const int64_t r = q1;
            int p1 = 0, p2 = 0;
            const int c1 = A1 >= 0 ? orbit_members((int)n1, (bits >> A1) & 1u, s1, p1) : 1;
            const int c2 = A2 >= 0 ? orbit_members((int)n2, (bits >> A2) & 1u, s2, p2) : 1;
            valid = uvalid && f < c1 * c2;
            const int i1 = c2 == 2 ? (f >> 1) & (c1 - 1) : f & (c1 - 1), i2 = f & (c2 - 1);
            const int64_t kk1 = A1 < 0 ? 0 : (i1 ? p1 : s1);
            const int64_t kk2 = A2 < 0 ? 0 : (i2 ? p2 : s2);
            if (i1)
                neg ^= mask1;
            if (i2)
                neg ^= mask2;
            int64_t rsrc = 0, rstr = 1, gr = r, rfull = 0, rmul = 1;
            for (int a = A1 - 1; a >= 0; --a) {
                const int64_t na = sp.levels[a];
                const int64_t ka = gr % na;
                gr /= na;
                const int odd = (bits >> a) & 1u;
                bool mm;
                rsrc += mirror_src(na, odd, ka, mm) * rstr;
                rstr *= stored_len(na, odd);
                rfull += ka * rmul;
                rmul *= na;
                if (mm)
                    for (int uu = 0; uu < U; ++uu)
                        neg ^= ((sp.skew_mask[uu] >> a) & 1u) << uu;
            }
            g = (rfull * n1 + kk1) * n2 + kk2;
            const int64_t row = (rsrc * st1 + s1) * st2 + s2;
            off0 = row * (N / 2 + 1);
            off1 = row * (N / 2);
        }
    };
    // XS (C3's 512-point 3x3 leaf): each unit's 12 x rows (4 fibers x 3
    // components, 4 KB each) arrive in shared memory by bulk copies issued one
    // unit ahead — while the current unit's odd branch computes — instead of
    // per-thread global loads at the start of every unit (their latency was
    // the largest stall); the odd branch re-reads x from the same rows.
    constexpr bool XS = TSK_LEAF_XS && CMP && M == 3 && N == 512 && sizeof(T) == 4;
    T2* xsu = stg0 + G * UM * LROW + (XS ? gi * CF * N : 0);  // this unit's rows
    uint32_t xphase = 0;
    auto issue_x = [&](int64_t tile_n) {
        // warp-uniform: one component's warps issue for their fibers.
        // TSK_LEAF_XC: which one (A/B; with factorised signs the last
        // component's warps have no per-fiber flips to apply)
        if (c != (TSK_LEAF_XC < M ? TSK_LEAF_XC : 0))
            return;
        int64_t un = tile_n * G + gi;
        if (un >= units)
            un = units - 1;
        const T2* srcn = src0;
        if (MRHS && nrhs > 1) {
            const uint32_t ur = divr.div((uint32_t)un);
            srcn += (un - (int64_t)ur * nrhs) * p.rstride;
            un = ur;
        }
        bool vn;
        int64_t gn, o0, o1;
        uint32_t ng;
        geometry(un, true, vn, gn, o0, o1, ng);
        if (t == 0) {
            const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&xbar[gi]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(M * N * 8)
                         : "memory");
#if TSK_LEAF_LDEF
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
#pragma unroll
            for (int cc = 0; cc < M; ++cc) {
                const uint32_t dsts = (uint32_t)__cvta_generic_to_shared(xsu + (f * M + cc) * N);
#if TSK_LEAF_LDEF
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                    "[%3], %4;" ::"r"(dsts),
                    "l"(srcn + cc * p.cstride + gn * N), "r"(N * 8), "r"(bar), "l"(pol)
                    : "memory");
#else
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        dsts),
                    "l"(srcn + cc * p.cstride + gn * N), "r"(N * 8), "r"(bar)
                    : "memory");
#endif
            }
        }
    };
    // N >= 256: one or two CTAs per SM holding most of the shared memory, so
    // the next pass's CTAs cannot co-reside; they may be released at once.
    // Smaller leaves release them on their last tile (a co-resident waiter
    // would take issue slots from the pass).
    if constexpr (N >= 256)
        pdl_trigger();
    pdl_wait();  // the previous pass's output is this pass's input
    if constexpr (XS) {
        if (threadIdx.x < G) {
            const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&xbar[threadIdx.x]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(4) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncthreads();
        if ((int64_t)blockIdx.x * G < units)
            issue_x(blockIdx.x);
    }

    for (int64_t tile = blockIdx.x; tile * G < units; tile += gridDim.x) {
        if constexpr (N < 256) {
            if ((tile + gridDim.x) * G >= units)
                pdl_trigger();  // last tile: the next pass may start its prologue
        }
        int64_t u = tile * G + gi;
        const bool uvalid = u < units;
        if (!uvalid)
            u = units - 1;  // runs in lockstep (barriers), stores nothing
        const T2* src = src0;
        T2* dst = dst0;
        if (MRHS && nrhs > 1) {  // units < 2^31 (checked by the launcher)
            const uint32_t ur = divr.div((uint32_t)u);
            const int64_t r = u - (int64_t)ur * nrhs;
            src += r * p.rstride;
            dst += r * p.rstride;
            u = ur;
        }
        if constexpr (XS) {  // this unit's x rows (issued one unit ahead)
            const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&xbar[gi]);
            asm volatile(
                "{\n .reg .pred p;\n XW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra XW;\n}" ::"r"(
                    bar),
                "r"(xphase)
                : "memory");
            xphase ^= 1u;
        }
        bool valid;
        int64_t g, off0, off1;
        uint32_t neg;
        geometry(u, uvalid, valid, g, off0, off1, neg);
        // sign masks per unique component: bit uu of neg (unmirrored k) and
        // of neg ^ lastneg (mirrored k)
        const uint32_t neg0 = neg, neg1 = neg ^ lastneg;
        // FS: this thread's per-fiber sign s_c (c = 0: axis 0 mirrored, the
        // sign of block (0, 2); c = 1: axis 1, block (1, 2)); the output scale
        // carries it
        const uint32_t sgx = FS && c < 2 ? (neg >> (c == 0 ? 2 : 4)) & 1u : 0u;
        const T sscale = sgx ? -scale : scale;
        auto stage_row = [&](int beta) {
            if constexpr (!CMP)
                return;
            const int L = beta ? N / 2 : N / 2 + 1;
            const T2* rowp = spec + sp.branch_base[beta] + (beta ? off1 : off0);
            const int64_t be = sp.block_elems[beta];
#pragma unroll
            for (int uu = 0; uu < UM; ++uu) {
#pragma unroll
                for (int k0 = 0; k0 < LROW; k0 += UT) {
                    const int kk = k0 + lt;
                    if (kk < L) {
                        if constexpr (sizeof(T2) == 8)
                            cp_async_bytes8(stg + uu * LROW + kk, rowp + uu * be + kk);
                        else
                            cp_async_bytes16(stg + uu * LROW + kk, rowp + uu * be + kk);
                    }
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        stage_row(ue ? 0 : 1);
        const T2* xin = src + c * p.cstride + g * N + t;

#pragma unroll
        for (int beta = 0; beta < 2; ++beta) {
            if (beta == 0 ? !ue : !uo)
                continue;
            // x: from the unit's shared-memory rows (XS), else global memory
            // (the odd branch's re-read then hits L1)
            T2 v[R];
            if constexpr (XS) {
                const T2* xr = xsu + (f * M + c) * N + t;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = xr[m * TF];
            } else {
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = xin[m * TF];
            }
            if constexpr (FS) {
                if (c < 2)
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        v[m] = flip_bits<T>(v[m], sgx);
            }
            if (beta == 1) {
                if constexpr (TWT) {
                    // P_k from this lane's TMEM table: one complex product
#pragma unroll
                    for (int h = 0; h < R / 16; ++h) {
                        uint32_t r32[32];
                        tmem_ld32(quad + PHOFF + 32 * h, r32);
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            Tw<T> w;
                            w.lo = Words<T2>::make(r32 + 2 * i);
                            w.hi = w.lo;
                            v[16 * h + i] = wide::cmul_tw<T, false>(v[16 * h + i], w);
                        }
                    }
                } else {
                    sfor<0, R>([&](auto I) {
                        constexpr int mi = decltype(I)::value;
                        v[mi] = PhaseR<T, R, false>::template apply<mi>(v[mi], pt);
                    });
                }
            }
            fft_one<T, N, R, false, TWT>(v, buf, tw, t, quad + TWOFF);

            // ---- spectra multiply y_c = sum_c' T_{c c'} x_c' (components meet in smem)
            if constexpr (MIXT) {
                tmem_park<T, R>(quad + MIXOFF + EW * c, v);
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            } else if (M > 1) {
#pragma unroll
                for (int m = 0; m < R; ++m)
                    buf[Pad<N, R>::rd(t, m)] = v[m];
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            unit_sync();
            if constexpr (MIXT)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // stored half-spectrum index: k = t + TF m below N/2, mirrored
            // (N - beta - k) from N/2 up; k = N/2 (t = 0, even) maps to itself
            auto mix = [&](auto CI) {
                constexpr int C = decltype(CI)::value;
                const T2* sA = stg + t;
                const T2* sB = stg + (N - beta - t);
                const bool t0 = t == 0;
                // 8-column reads at R = 32 (16 fewer live registers at the mix:
                // the 168-register pass otherwise spills), 16 below
                constexpr int WPC = R >= 32 ? 8 : 16;  // words per TMEM read
                constexpr int XCH = WPC / Words<T2>::W;        // partner values per read
                T2 xo[M][XCH];          // partners' values of the current chunk
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    if constexpr (MIXT) {
                        if (m % XCH == 0) {
                            uint32_t r[M][WPC];
#pragma unroll
                            for (int cc = 0; cc < M; ++cc)
                                if (cc != C) {
                                    if constexpr (WPC == 8)
                                        tmem_ld8(quad + MIXOFF + EW * cc + (m / XCH) * WPC, r[cc]);
                                    else
                                        tmem_ld16(quad + MIXOFF + EW * cc + (m / XCH) * WPC, r[cc]);
                                }
                            tmem_wait_ld();
#pragma unroll
                            for (int cc = 0; cc < M; ++cc)
                                if (cc != C)
#pragma unroll
                                    for (int i = 0; i < XCH; ++i)
                                        xo[cc][i] = Words<T2>::make(r[cc] + i * Words<T2>::W);
                        }
                    }
                    const bool mirm = 2 * m >= R;
                    const T2* sp_ = mirm ? sB - TF * m : sA + TF * m;
                    (void)sp_;  // unused with full storage
                    T2 acc;
                    sfor<0, M>([&](auto CC) {
                        constexpr int cc = decltype(CC)::value;
                        constexpr int lo = C < cc ? C : cc, hi = C < cc ? cc : C;
                        constexpr int uu = M == 1 ? 0 : 3 * lo - (lo * (lo - 1)) / 2 + (hi - lo);
                        // sign: unmirrored neg0, mirrored neg1 (k = N/2 at t = 0 unmirrored)
                        uint32_t ng;
                        if (!mirm)
                            ng = neg0;
                        else if (beta == 0 && 2 * m == R)
                            ng = t0 ? neg0 : neg1;
                        else
                            ng = neg1;
                        T2 s_;
                        if constexpr (FS)
                            s_ = sp_[uu * LROW];
                        else if constexpr (CMP)
                            s_ = flip_bits<T>(sp_[uu * LROW], (ng >> uu) & 1u);
                        else  // full storage: this fiber's own row, read once
                            s_ = ldg_c(spec + sp.branch_base[beta] + (beta ? off1 : off0) +
                                       uu * sp.block_elems[beta] + t + TF * m);
                        T2 xv;
                        if constexpr (cc == C)
                            xv = v[m];
                        else if constexpr (MIXT)
                            xv = xo[cc][m % XCH];
                        else
                            xv = fbufs[(f * M + cc) * NP + Pad<N, R>::rd(t, m)];
                        // FS: the term is negated on the mirrored leaf half iff
                        // exactly one of C, cc is the leaf-axis component 2
                        if constexpr (FS && ((C == 2) != (cc == 2))) {
                            if (beta == 0 && 2 * m == R)  // k = N/2: unmirrored at t = 0
                                acc = cmac<T>(acc, xv, flip_bits<T>(s_, t0 ? 0u : 1u), cc == 0);
                            else if (mirm)
                                acc = cmac_neg<T>(acc, xv, s_, cc == 0);
                            else
                                acc = cmac<T>(acc, xv, s_, cc == 0);
                        } else {
                            acc = cmac<T>(acc, xv, s_, cc == 0);
                        }
                    });
                    v[m] = acc;
                    if (m % 2 == 1)
                        asm volatile("" ::: "memory");  // bound the loads in flight
                }
            };
            if constexpr (M == 1) {
                mix(std::integral_constant<int, 0>{});
            } else {
                if (c == 0)
                    mix(std::integral_constant<int, 0>{});
                else if (c == 1)
                    mix(std::integral_constant<int, 1>{});
                else
                    mix(std::integral_constant<int, 2>{});
            }
            if constexpr (MIXT)
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            unit_sync();  // staged row and mix buffers free
            if constexpr (MIXT)
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (beta == 0 && uo)
                stage_row(1);
            if constexpr (XS) {  // every thread of the unit has read its x rows
                if ((beta == 1 || !uo) && (tile + gridDim.x) * G < units)
                    issue_x(tile + gridDim.x);
            }
            fft_one<T, N, R, true, TWT>(v, buf, tw, t, quad + TWOFF);

            if (beta == 0 && both) {
                if constexpr (TM)
                    tmem_park<T, R, false>(lane_base, v);  // waited before the restore
                else
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        ekeep[m] = v[m];
            } else {
                // e' comes back from TMEM 32 words at a time (bounded registers);
                // the branch conditions are resolved once, outside the element loop
                constexpr int EPC = TWT ? 8 : TM ? 32 / ((int)sizeof(T2) / 4) : R;
                T2* yout = dst + c * p.cstride + g * N + t;
                auto emit = [&](auto ODD, auto BOTH) {
                    constexpr bool odd = decltype(ODD)::value, bth = decltype(BOTH)::value;
                    if constexpr (bth && TM)
                        tmem_wait_st();  // e' park (usually long complete)
                    sfor<0, R / EPC>([&](auto C) {
                        constexpr int c0 = decltype(C)::value * EPC;
                        T2 e[EPC], ph[TWT ? EPC : 1];
                        if constexpr (TWT && odd) {
                            uint32_t r[16];
                            tmem_ld16(quad + PHOFF + c0 * 2, r);
                            if constexpr (bth) {
                                uint32_t re[16];
                                tmem_ld16(lane_base + c0 * 2, re);
                                tmem_wait_ld();
#pragma unroll
                                for (int i = 0; i < EPC; ++i)
                                    e[i] = Words<T2>::make(re + 2 * i);
                            } else {
                                tmem_wait_ld();
                            }
#pragma unroll
                            for (int i = 0; i < EPC; ++i)
                                ph[i] = Words<T2>::make(r + 2 * i);
                        } else if constexpr (bth) {
                            if constexpr (TM) {
                                uint32_t r[32];
                                tmem_ld32(lane_base + c0 * ((int)sizeof(T2) / 4), r);
#pragma unroll
                                for (int i = 0; i < EPC; ++i)
                                    e[i] = Words<T2>::make(r + i * Words<T2>::W);
                            } else {
#pragma unroll
                                for (int i = 0; i < EPC; ++i)
                                    e[i] = ekeep[c0 + i];
                            }
                        }
                        sfor<0, EPC>([&](auto I) {
                            constexpr int mi = c0 + decltype(I)::value;
                            T2 a;
                            if constexpr (odd && TWT) {
                                // scale (conj(P) o + e): the table holds P unscaled
                                Tw<T> w;
                                w.lo = ph[decltype(I)::value];
                                w.hi = w.lo;
                                // (fused at R = 32 only: the 80-register 256-point
                                // pass spills 64 B with it)
                                if constexpr (bth && R >= 32) {
                                    a = cmulc_add<T>(v[mi], w.lo, e[decltype(I)::value]);
                                } else {
                                    a = wide::cmul_tw<T, true>(v[mi], w);
                                    if constexpr (bth)
                                        a = cadd(a, e[decltype(I)::value]);
                                }
                                a = scale_c<T>(a, FS ? sscale : scale);
                            } else if constexpr (odd) {
                                a = PhaseR<T, R, true>::template apply<mi>(v[mi], pts);
                                if constexpr (bth)
                                    a = fma_s<T>(e[decltype(I)::value], scale, a);
                            } else {
                                a = scale_c<T>(v[mi], FS ? sscale : scale);
                            }
                            if (valid) {
                                // (short leaves: their vectors are often L2-resident)
                                if constexpr (TSK_LEAF_STCS && N >= 256)
                                    __stcs(yout + mi * TF, a);
                                else
                                    yout[mi * TF] = a;
                            }
                        });
                    });
                };
                using B0 = std::false_type;
                using B1 = std::true_type;
                if (beta == 0)
                    emit(B0{}, B0{});
                else if (both)
                    emit(B1{}, B1{});
                else
                    emit(B1{}, B0{});
            }
        }
    }
    if constexpr (TM)
        tmem_free(tbase, TCOLS);
}

static int sm_count()
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

template <typename T, int N, int R, int M, bool CMP, bool MRHS, bool FS = false>
static int launch(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    using T2 = typename cx<T>::t;
    constexpr int TF = N / R;
    constexpr int NP = Pad<N, R>::NP;
    constexpr int G = leaf1_g<N, R, M>();
    constexpr int NT = G * 4 * M * TF;
    constexpr bool XS = TSK_LEAF_XS && CMP && M == 3 && N == 512 && sizeof(T) == 4;
    const size_t smem = sizeof(T2) * (R * (N / R - 1) + G * 4 * M * NP + G * (M == 1 ? 1 : 6) * (N / 2 + 1) +
                                      (XS ? G * 4 * M * N : 0));
    if (smem > 227 * 1024)
        return -1;
    auto kern = k_leaf1<T, N, R, M, CMP, MRHS, FS>;
    static thread_local int cached_dev = -1, cap = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        if (int e = (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem))
            return e;
        if (const char* cv = getenv("TSK_LEAF_CARVEOUT"))  // A/B: shared-memory carveout (%)
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
        int per_sm = 0;
        // TMEM: every resident CTA allocates its columns (the occupancy API
        // undercounts tcgen05 kernels; tmem_occupancy counts the resources)
        constexpr int EW = R * (int)sizeof(T2) / 4;
        constexpr int NW = NT / 32 > 0 ? NT / 32 : 1;
        constexpr int TC = leaf_tcols<T, N, R, M, CMP, NW>();
        if (EW % 32 == 0)
            per_sm = tmem_occupancy(kern, NT, smem, TC);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
        if (getenv("TSK_DEBUG_OCC")) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kern);
            fprintf(stderr, "k_leaf1<%d,%d,%d,%d,%d>: %d CTAs/SM, %zu B smem (+%zu static), %d threads, %d regs\n",
                    (int)sizeof(T), N, R, M, (int)CMP, per_sm, smem, fa.sharedSizeBytes, NT, fa.numRegs);
        }
        cap = sm_count() * (per_sm > 0 ? per_sm : 1);
        cached_dev = dev;
    }
    int64_t units = 1;
    if (CMP) {
        for (int ax = 0; ax < sp.d - 1; ++ax)
            units *= ax >= sp.d - 3 ? stored_len(sp.levels[ax], (sp.branch_bits[0] >> ax) & 1u)
                                    : sp.levels[ax];
        if (units >= (int64_t(1) << 31))
            return -1;  // FastDiv / 32-bit orbit indices
    } else {
        units = (a.outer + 3) / 4;
    }
    units *= a.nrhs > 1 ? a.nrhs : 1;
    if (units >= (int64_t(1) << 31))
        return -1;
    const int64_t tiles = (units + G - 1) / G;
    const int64_t grid = tiles < cap ? tiles : cap;
    const cudaError_t e = launch_pdl(pdl_for(a), kern, (unsigned)(grid > 0 ? grid : 1), NT, smem, st, a, sp);
    return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

// The dyadic sign structure (FS above): d = 3 and skew_mask(i, j) = axis i
// XOR axis j for the canonical 6-unique 3x3 map. TSK_LEAF_NO_FS=1 (A/B)
// keeps the per-value sign flips; TSK_LEAF_FS512=0 (build flag) keeps them at
// n = 512.
static bool dyadic_signs(const tsk_spectra& sp)
{
    static const bool off = [] {
        const char* e = getenv("TSK_LEAF_NO_FS");
        return e && e[0] == '1';
    }();
    static const uint32_t want[6] = {0u, 3u, 5u, 0u, 6u, 0u};
    if (off || sp.d != 3 || sp.m != 3 || sp.n_unique != 6 || !sp.compressed)
        return false;
    for (int u = 0; u < 6; ++u)
        if (sp.skew_mask[u] != want[u])
            return false;
    return true;
}

template <typename T, int M, bool CMP, bool MRHS>
static int dispatch_n(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    constexpr bool FSOK = sizeof(T) == 4 && M == 3 && CMP;
    const bool fs = FSOK && (a.n == 256 || TSK_LEAF_FS512) && dyadic_signs(sp);
    switch (a.n) {
    case 64: return launch<T, 64, 8, M, CMP, MRHS>(a, sp, st);
    case 128: return launch<T, 128, 16, M, CMP, MRHS>(a, sp, st);
    case 256:
        if constexpr (FSOK)
            if (fs)
                return launch<T, 256, 16, M, CMP, MRHS, true>(a, sp, st);
        return launch<T, 256, 16, M, CMP, MRHS>(a, sp, st);
    case 512:  // complex128 at R = 32 spills; the 8-point kernel handles it
        // (factorised signs at R = 32 fit the 168-register cap only with the
        // 8-column partner reads of the mix; with 16-column reads they spilled,
        // K2 2.77 -> 3.06 ms at 512^3, profiles/r02_ab_fs.txt; with 8-column
        // reads 2.81 -> 2.70 ms, profiles/r02_ab_fs512.txt. At R = 16, 80
        // registers: 0.367 -> 0.350 ms at 256^3)
        if constexpr (sizeof(T) == 4) {
#if TSK_LEAF_FS512
            if constexpr (FSOK)
                if (fs)
                    return launch<T, 512, 32, M, CMP, MRHS, true>(a, sp, st);
#endif
            return launch<T, 512, 32, M, CMP, MRHS>(a, sp, st);
        } else {
            return -1;
        }
    default: return -1;
    }
}

template <typename T, int M, bool CMP>
static int dispatch_s(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    return a.nrhs > 1 ? dispatch_n<T, M, CMP, true>(a, sp, st) : dispatch_n<T, M, CMP, false>(a, sp, st);
}

template <typename T, int M>
static int dispatch(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    return sp.compressed ? dispatch_s<T, M, true>(a, sp, st) : dispatch_s<T, M, false>(a, sp, st);
}

// ---- plain transforms along a contiguous axis (inner = 1, no split / no
// merge partner): the full-embedding engine's last axis and the spectra
// precompute. One fiber per TF = N/R threads (a warp or half warp), R
// elements per thread, one shared-memory exchange (fft_one); out = F(x) or
// scale * F^{-1}(x), natural order, in place allowed.
template <typename T, int N, int R, bool INV>
__global__ void __launch_bounds__(256) k_contig(tsk_axis p)
{
    using T2 = typename cx<T>::t;
    constexpr int TF = N / R;
    constexpr int P2 = N / R;
    constexpr int FPC = 256 / TF;  // fibers per CTA
    constexpr int NP = Pad<N, R>::NP;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T2* tw = reinterpret_cast<T2*>(smem_raw);
    T2* bufs = tw + R * (P2 - 1);
    for (int e = threadIdx.x; e < R * (P2 - 1); e += blockDim.x) {
        const int j = e / (P2 - 1), r = e % (P2 - 1) + 1;
        tw[e] = ldg_c(static_cast<const T2*>(p.roots) + (r * j) % N);
    }
    __syncthreads();
    const int fi = threadIdx.x / TF, t = threadIdx.x % TF;
    T2* buf = bufs + fi * NP;
    const int64_t nfib = p.outer * p.ncomp;
    const T scale = (T)p.scale;
    const T2* src0 = static_cast<const T2*>(p.src0);
    T2* dst0 = static_cast<T2*>(p.dst0);
    // fibers are whole warps or half warps: the loop bound is uniform per
    // fiber group, and fft_one synchronises with __syncwarp only
    for (int64_t f0 = (int64_t)blockIdx.x * FPC; f0 < nfib; f0 += (int64_t)gridDim.x * FPC) {
        const int64_t f = f0 + fi;
        if (f >= nfib)
            continue;
        const int64_t c = f / p.outer, o = f - c * p.outer;
        const int64_t off = c * p.cstride + o * N + t;
        T2 v[R];
#pragma unroll
        for (int m = 0; m < R; ++m)
            v[m] = src0[off + m * TF];
        fft_one<T, N, R, INV>(v, buf, tw, t);
#pragma unroll
        for (int m = 0; m < R; ++m)
            dst0[off + m * TF] = INV ? scale_c<T>(v[m], scale) : v[m];
    }
}

template <typename T, int N, int R, bool INV>
static int launch_contig(const tsk_axis& a, cudaStream_t st)
{
    using T2 = typename cx<T>::t;
    constexpr int TF = N / R;
    constexpr int FPC = 256 / TF;
    const size_t smem = sizeof(T2) * (R * (N / R - 1) + FPC * Pad<N, R>::NP);
    auto kern = k_contig<T, N, R, INV>;
    static thread_local int cached_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        if (int e = (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))
            return e;
        cached_dev = dev;
    }
    const int64_t nfib = a.outer * a.ncomp;
    const int64_t blocks = (nfib + FPC - 1) / FPC;
    const int64_t grid = blocks < sm_count() * 8 ? blocks : sm_count() * 8;
    kern<<<(unsigned)(grid > 0 ? grid : 1), 256, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <typename T, bool INV>
static int dispatch_contig(const tsk_axis& a, cudaStream_t st)
{
    switch (a.n) {
    case 256: return launch_contig<T, 256, 16, INV>(a, st);
    case 512: return launch_contig<T, 512, 32, INV>(a, st);
    case 1024: return launch_contig<T, 1024, 32, INV>(a, st);
    default: return -1;
    }
}

}  // namespace leaf
}  // namespace tsk

// Plain (even-only) transform along a contiguous axis; -1: not covered.
extern "C" int tsk_contig_pass(const tsk_axis* a, int inv, void* stream)
{
    if (a->inner != 1 || a->use_odd || !a->use_even || !a->prec || a->src1)
        return -1;
    auto st = (cudaStream_t)stream;
    return inv ? tsk::leaf::dispatch_contig<float, true>(*a, st)
               : tsk::leaf::dispatch_contig<float, false>(*a, st);
}

// -1: not covered (caller falls back), else the launch cudaError_t.
extern "C" int tsk_leaf1_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    if (a->inner != 1)
        return -1;
    static const int8_t canon[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
    auto st = (cudaStream_t)stream;
    if (sp->m == 1)
        return a->prec ? tsk::leaf::dispatch<float, 1>(*a, *sp, st)
                       : tsk::leaf::dispatch<double, 1>(*a, *sp, st);
    if (sp->m == 3 && sp->n_unique == 6) {
        for (int i = 0; i < 9; ++i)
            if (sp->comp_map[i] != canon[i])
                return -1;
        return a->prec ? tsk::leaf::dispatch<float, 3>(*a, *sp, st)
                       : tsk::leaf::dispatch<double, 3>(*a, *sp, st);
    }
    return -1;
}
