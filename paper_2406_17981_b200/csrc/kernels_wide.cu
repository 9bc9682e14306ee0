// Wide-tile sm_100a kernels for the strided passes (K1 fwd_split, K3
// inv_merge) on power-of-two axes.
//
// Why wide tiles: a strided pass reads/writes, per tile, one contiguous row
// segment per position along the axis. Measured on B200 (tools/micro/
// strided_copy2.cu / strided_copy3.cu, pure 1R/2W copies of 512-row tiles):
// 64-byte segments reach 2.3 TB/s, 128-byte 4.4-5.2 TB/s at two CTAs per SM,
// 256-byte 5.7-5.8 TB/s at one. Every warp memory instruction covers one
// row segment of W columns; the default is 128 bytes (W = 16 complex64) with
// two CTAs per SM, so one CTA's memory phase overlaps the other's arithmetic.
//
// Each thread holds R = 16..32 elements of one column in registers ("row
// pattern" k = t + m*TF, TF = N/R threads per column): N = 512 is 32 x 16, one
// shared-memory exchange per transform.
//  K1: odd = F(P x) is transformed and stored (to the child buffer), then
//      even = F(x) from x parked in tensor memory (thread-private lane) when
//      the load arrived — the even child may overwrite x in place.
//  K3: out = scale * (B(e) + conj(P) B(o)); B(e) is parked in tensor memory
//      while B(o) is computed, so registers hold one transform at a time.
// Both allocate TMEM, so the launcher counts CTAs per SM from registers,
// shared memory and columns (the occupancy API reports one for tcgen05
// kernels).
// Reference semantics as in kernels_generic.cu (fft.cpp:65-87,
// tensor.cpp:227-254, engine_split.cpp:13-37).
#include <cuda_runtime.h>

#include <cstdlib>

#include <utility>

#include "tsk_common.cuh"
#include "tsk_tmem.cuh"
#include "tsk_wide.cuh"

namespace tsk {
namespace wide {

template <typename T, int N, int R>
__device__ void fill_tables(typename cx<T>::t* tw, typename cx<T>::t* ph,
                            const typename cx<T>::t* __restrict__ roots,
                            const typename cx<T>::t* __restrict__ phase)
{
    using P = Plan<N, R>;
#pragma unroll
    for (int s = 1; s < P::NST; ++s) {
        const int p = P::radix(s), ns = P::ns(s);
        for (int e = threadIdx.x; e < ns * (p - 1); e += blockDim.x) {
            const int jm = e / (p - 1), r = e % (p - 1) + 1;
            tw[P::tw_off(s) + e] = ldg_c(roots + (r * jm * (N / (ns * p))) % N);
        }
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x)
        ph[k] = ldg_c(phase + k);
}

// One length-N transform of the row pattern v[m] = x[t + m TF] (m < R) of one
// column w; exchanges through the [N][W] tile buffer (a warp covers one row,
// conflict free), two barriers per exchange (single buffer).
template <typename T, int N, int R, int W, bool INV>
__device__ __forceinline__ void fft_col(typename cx<T>::t (&v)[R], typename cx<T>::t* buf,
                                        const typename cx<T>::t* tw, int t, int w)
{
    using T2 = typename cx<T>::t;
    using PL = Plan<N, R>;
    constexpr int TF = PL::TF;
#pragma unroll
    for (int s = 0; s < PL::NST; ++s) {
        constexpr int dummy = 0;
        (void)dummy;
        const int p = PL::radix(s);
        const int ns = PL::ns(s);
        const int G = R / p;
        if (s > 0) {
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int jm = (t + i * TF) % ns;
#pragma unroll
                for (int r = 1; r < p; ++r) {
                    const Tw<T> wv = load_tw<T>(tw + PL::tw_off(s) + jm * (p - 1) + (r - 1));
                    v[i + r * G] = cmul_tw<T, INV>(v[i + r * G], wv);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < G; ++i) {
            T2 a[R];
#pragma unroll
            for (int r = 0; r < p; ++r)
                a[r] = v[i + r * G];
            switch (p) {
            case 2: Dft<T, 2, INV>::run(a); break;
            case 4: Dft<T, 4, INV>::run(a); break;
            case 8: Dft<T, 8, INV>::run(a); break;
            case 16: Dft<T, 16, INV>::run(a); break;
            case 32: Dft<T, 32, INV>::run(a); break;
            default: break;
            }
#pragma unroll
            for (int r = 0; r < p; ++r)
                v[i + r * G] = a[r];
        }
        if (s == PL::NST - 1)
            break;
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const int j = t + i * TF;
            const int jm = j % ns;
            const int base = (j - jm) * p + jm;
#pragma unroll
            for (int q = 0; q < p; ++q)
                buf[(base + q * ns) * W + w] = v[i + q * G];
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < R; ++m)
            v[m] = buf[(t + m * TF) * W + w];
        __syncthreads();
    }
}

// ---- K1 / K3 ------------------------------------------------------------------

template <typename T, int N, int R, int W, int MODE>
__global__ void __launch_bounds__(N / R * W, sizeof(T) == 4 && (N / R * W) < 512 ? 512 / (N / R * W) : 1) k_wide(tsk_axis p)
{
    using T2 = typename cx<T>::t;
    using T4 = typename tw4<T>::t;
    using PL = Plan<N, R>;
    constexpr int TF = PL::TF;
    constexpr int NT = TF * W;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T2* tw = reinterpret_cast<T2*>(smem_raw);
    T2* ph = tw + PL::TW;
    T2* buf = ph + N;
    __shared__ uint32_t tmem_slot;
    fill_tables<T, N, R>(tw, ph, static_cast<const T2*>(p.roots), static_cast<const T2*>(p.phase));
    __syncthreads();

    const int w = threadIdx.x % W;
    const int t = threadIdx.x / W;
    const int64_t inner = p.inner;
    const int64_t cols = inner / W;
    const int64_t tiles_per_comp = p.outer * cols;
    const int64_t ntiles = tiles_per_comp * p.ncomp;
    const bool ue = p.use_even, uo = p.use_odd;
    const T scale = (T)p.scale;
    const int64_t rs = (int64_t)TF * inner;  // element stride between m and m+1

    // K3 with both inputs parks B(e) in tensor memory: warps sharing a lane
    // quadrant (w % 4) take disjoint column ranges
    constexpr int PWORDS = R * (int)sizeof(T2) / 4;
    constexpr int NW = NT / 32;
    constexpr int TCOLS_RAW = PWORDS * ((NW + 3) / 4);
    constexpr int TCOLS = TCOLS_RAW <= 32 ? 32 : TCOLS_RAW <= 64 ? 64 : TCOLS_RAW <= 128 ? 128
                                                                        : TCOLS_RAW <= 256 ? 256 : 512;
    constexpr bool TM = PWORDS % 32 == 0;  // small R keeps B(e) in registers
// K1 keeps x in tensor memory for the even child instead of re-reading it
// through L2 (with two CTAs per SM: K1 2.35/2.05 -> 2.09/1.94 ms at 512^3;
// measured slower only while the occupancy API held tcgen05 kernels to one
// CTA per SM)
#ifndef WIDE_K1_XTMEM
#define WIDE_K1_XTMEM 1
#endif
    const bool park = TM && (MODE == 1 || WIDE_K1_XTMEM) && ue && uo;
    uint32_t tbase = 0, lane_base = 0;
    if constexpr (MODE == 1 || WIDE_K1_XTMEM) {
        if (park) {
            tbase = tmem_alloc(&tmem_slot, TCOLS);
            const int warp = threadIdx.x / 32;
            lane_base = tbase + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)(PWORDS * (warp / 4));
        }
    }

    pdl_wait();  // the previous pass's output is this pass's input
    // tile -> (component, outer, column block) by multiply-high (the
    // launcher guarantees ntiles < 2^31)
    const FastDiv div_tpc((uint32_t)tiles_per_comp), div_cols((uint32_t)cols);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (tile + gridDim.x >= ntiles)
            pdl_trigger();  // last tile: the next pass may start its prologue
        const uint32_t t32 = (uint32_t)tile;
        const uint32_t c32 = div_tpc.div(t32);
        const uint32_t r32 = t32 - c32 * (uint32_t)tiles_per_comp;
        const uint32_t o32 = div_cols.div(r32);
        const int64_t c = c32, o = o32;
        const int64_t i0 = (int64_t)(r32 - o32 * (uint32_t)cols) * W;
        const int64_t base = c * p.cstride + o * (int64_t)N * inner + i0 + w + (int64_t)t * inner;
        T2 v[R];
        T2 ekeep[TM ? 1 : R];
        if (MODE == 0) {
            // odd first: even may be written in place over the input (dst0 ==
            // src0 below the root), and the odd child needs the input again
            const T2* src = static_cast<const T2*>(p.src0) + base;
            if (uo) {
#if WIDE_K1_XTMEM
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = src[m * rs];
                if constexpr (TM) {
                    if (park)
                        tmem_park<T, R, false>(lane_base, v);  // waited before the restore
                }
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = cmul_tw<T, false>(v[m], load_tw<T>(ph + t + m * TF));
#else
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = cmul_tw<T, false>(src[m * rs], load_tw<T>(ph + t + m * TF));
#endif
                fft_col<T, N, R, W, false>(v, buf, tw, t, w);
                T2* dd = static_cast<T2*>(p.dst1) + base;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    dd[m * rs] = v[m];
            }
            if (ue) {
                // x again: from TMEM (WIDE_K1_XTMEM), else an L1/L2 hit
                bool have = false;
#if WIDE_K1_XTMEM
                if constexpr (TM) {
                    if (park) {
                        tmem_wait_st();
                        tmem_restore<T, R>(lane_base, v);
                        have = true;
                    }
                }
#endif
                if (!have)
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        v[m] = src[m * rs];
                fft_col<T, N, R, W, false>(v, buf, tw, t, w);
                T2* de = static_cast<T2*>(p.dst0) + base;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    de[m * rs] = v[m];
            }
        } else {
            T2* dst = static_cast<T2*>(p.dst0) + base;
            if (ue) {
                const T2* se = static_cast<const T2*>(p.src0) + base;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = se[m * rs];
                fft_col<T, N, R, W, true>(v, buf, tw, t, w);
                if (!uo) {
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        dst[m * rs] = scale_c<T>(v[m], scale);
                    continue;
                }
                if constexpr (MODE == 1 && TM)
                    tmem_park<T, R, false>(lane_base, v);  // waited before the restore
                else
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        ekeep[m] = v[m];
            }
            if (uo) {
                const T2* so = static_cast<const T2*>(p.src1) + base;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = so[m * rs];
                fft_col<T, N, R, W, true>(v, buf, tw, t, w);
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = cmul_tw<T, true>(v[m], load_tw<T>(ph + t + m * TF));
                if (ue) {
                    T2 e[R];
                    if constexpr (MODE == 1 && TM) {
                        tmem_wait_st();
                        tmem_restore<T, R>(lane_base, e);
                    }
                    else
#pragma unroll
                        for (int m = 0; m < R; ++m)
                            e[m] = ekeep[m];
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        v[m] = cadd(v[m], e[m]);
                }
#pragma unroll
                for (int m = 0; m < R; ++m)
                    dst[m * rs] = scale_c<T>(v[m], scale);
            }
        }
    }
    if constexpr (MODE == 1 || WIDE_K1_XTMEM) {
        if (park)
            tmem_free(tbase, TCOLS);
    }
}

template <typename T, int N, int SEG = 256>
struct Geom {
    // SEG-byte row segments; R elements per thread
    static constexpr int W = SEG / (int)sizeof(typename cx<T>::t);
    static constexpr int R = N >= 512 ? 32 : (N >= 128 ? 16 : 8);
    static constexpr int NT = N / R * W;
};

static int sm_count()
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

template <typename T, int N, int MODE, int SEG>
static int launch(const tsk_axis& a, cudaStream_t st)
{
    using G = Geom<T, N, SEG>;
    using T2 = typename cx<T>::t;
    if (G::NT > 1024 || a.inner % G::W != 0)
        return -1;
    const size_t smem = sizeof(T2) * (Plan<N, G::R>::TW + N) + sizeof(T2) * N * G::W;
    if (smem > 227 * 1024)
        return -1;
    auto kern = k_wide<T, N, G::R, G::W, MODE>;
    static thread_local int cached_dev = -1, cap = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        if (int e = (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem))
            return e;
        int per_sm = 0;
        // K3 parks B(e) in TMEM: the occupancy API undercounts tcgen05
        // kernels, so count the resources (TMEM columns included)
        constexpr int PWORDS = G::R * (int)sizeof(T2) / 4;
        constexpr int NW = G::NT / 32;
        constexpr int TCR = PWORDS * ((NW + 3) / 4);
        constexpr int TC = TCR <= 32 ? 32 : TCR <= 64 ? 64 : TCR <= 128 ? 128 : TCR <= 256 ? 256 : 512;
        if ((MODE == 1 || WIDE_K1_XTMEM) && PWORDS % 32 == 0)
            per_sm = tmem_occupancy(kern, G::NT, smem, TC);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NT, smem);
        cap = sm_count() * (per_sm > 0 ? per_sm : 1);
        cached_dev = dev;
    }
    const int64_t ntiles = a.outer * (a.inner / G::W) * a.ncomp;
    if (ntiles >= (int64_t(1) << 31))
        return -1;  // 32-bit tile decomposition
    const int64_t grid = ntiles < cap ? ntiles : cap;
    const cudaError_t e = launch_pdl(pdl_for(a), kern, (unsigned)(grid > 0 ? grid : 1), G::NT, smem, st, a);
    return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

// Row segment per tile: 128 bytes, two CTAs per SM for K1 and K3 (with the
// TMEM-aware occupancy: K3 at 512^3 1.89 -> 1.69 ms on axis 1 against one
// 256-byte-wide CTA per SM); for axes whose row stride is >= 1 MB (axis 0 at
// 512^3: 2 MB) one 256-byte CTA per SM is a little faster (K1 2.10 -> 2.05 ms,
// K3 1.92 -> 1.88 ms). TSK_WIDE_SEG=128|256 overrides both (A/B).
static int seg_bytes(int mode, int64_t stride_bytes)
{
    static const int v = [] {
        const char* e = getenv("TSK_WIDE_SEG");
        return e ? atoi(e) : 0;
    }();
    if (v == 128 || v == 256)
        return v;
    (void)mode;
    return stride_bytes >= (int64_t(1) << 20) ? 256 : 128;
}

template <typename T, int MODE, int SEG>
static int dispatch_seg(const tsk_axis& a, cudaStream_t st)
{
    switch (a.n) {
    case 64: return launch<T, 64, MODE, SEG>(a, st);
    case 128: return launch<T, 128, MODE, SEG>(a, st);
    case 256: return launch<T, 256, MODE, SEG>(a, st);
    case 512: return launch<T, 512, MODE, SEG>(a, st);
    // 1024 (the full-embedding engine's (2n)^d axes at n = 512): 128-byte
    // rows (a 256-byte tile would need 256 KB of shared memory), complex64
    case 1024:
        if constexpr (sizeof(T) == 4)
            return launch<T, 1024, MODE, 128>(a, st);
        else
            return -1;
    default: return -1;
    }
}

template <typename T, int MODE>
static int dispatch(const tsk_axis& a, cudaStream_t st)
{
    const int64_t stride_bytes = a.inner * (int64_t)sizeof(typename cx<T>::t);
    return seg_bytes(MODE, stride_bytes) == 128 ? dispatch_seg<T, MODE, 128>(a, st)
                                                : dispatch_seg<T, MODE, 256>(a, st);
}

}  // namespace wide
}  // namespace tsk

// -1: shape not covered (the caller falls back), else the launch cudaError_t.
extern "C" int tsk_wide_fwd_split(const tsk_axis* a, void* stream)
{
    return a->prec ? tsk::wide::dispatch<float, 0>(*a, (cudaStream_t)stream)
                   : tsk::wide::dispatch<double, 0>(*a, (cudaStream_t)stream);
}

extern "C" int tsk_wide_inv_merge(const tsk_axis* a, void* stream)
{
    return a->prec ? tsk::wide::dispatch<float, 1>(*a, (cudaStream_t)stream)
                   : tsk::wide::dispatch<double, 1>(*a, (cudaStream_t)stream);
}
