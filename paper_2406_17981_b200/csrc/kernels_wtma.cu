// Strided passes (K1 fwd_split, K3 inv_merge) at n = 512 and 256, complex64,
// with the input tiles brought in by the Tensor Memory Accelerator.
//
// Why: a strided pass reads one 512-row x W-column tile per step. The DRAM
// side wants wide row segments (256 B rows: 5.7-5.8 TB/s for the K1 pattern
// against 4.4-5.2 at 128 B, tools/micro/strided_copy3.cu), but a 256 B tile
// (128 KB) held by per-thread loads leaves room for one CTA per SM, whose
// memory phase then idles while it computes (k_wide, kernels_wide.cu). Here
// one CTA per SM keeps a single 128 KB landing buffer busy all the time: the
// tile is copied from shared memory into registers (one 256 B row per warp
// instruction, conflict free), and right after that copy the next tile's two
// 256-row boxes are issued (cp.async.bulk.tensor, mbarrier completion) while
// the current tile is transformed. The column FFT (R = n/16 elements per
// thread, radix R x 16) exchanges through shared memory (at n = 512 a 64 KB
// half buffer in two rounds);
// K1 parks x and K3 parks B(e) in tensor memory between their two
// transforms; results go out as per-warp 256 B row stores.
//
// Same arithmetic, in the same order, as k_wide<float, n, n/16, W, MODE>
// (bit-identical outputs); reference semantics as there (fft.cpp:65-87,
// tensor.cpp:227-254, engine_split.cpp:13-37, relative to
// /root/reference/proj/src/core).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "tsk_common.cuh"
#include "tsk_tmem.cuh"
#include "tsk_wide.cuh"

namespace tsk {
namespace wtma {

using wide::cmul_tw;
using wide::Dft;
using wide::load_tw;
using wide::Plan;
using wide::Tw;

// N = 512 (R = 32, radix 32 x 16) or 256 (R = 16, radix 16 x 16); TF = 16
// threads per column
// rows per TMA box (<= 256; TSK_WTMA_BOX_ROWS: A/B of smaller boxes)
#ifndef TSK_WTMA_BOX_ROWS
#define TSK_WTMA_BOX_ROWS 256
#endif
// W columns per tile: 32 (256 B rows, 512 threads, one CTA per SM) everywhere
// except the merge pass at N = 256, which runs 16 columns (128 B rows, 256
// threads) at two CTAs per SM — one CTA's stores then overlap the other's
// transforms: K3 0.219 -> 0.201 ms (axis 1) and 0.224 -> 0.212 ms (axis 0) at
// 256^3, while K1 there (0.205 -> 0.248 ms) and both passes at N = 512 (K1
// 1.69 -> 2.14, K3 1.56 -> 1.87 ms) lose more DRAM efficiency to the shorter
// row segments than the overlap returns (profiles/r02_ab_w16.txt).
// TSK_WTMA_W3_256 (A/B): the merge pass's width at N = 256.
#ifndef TSK_WTMA_W3_256
#define TSK_WTMA_W3_256 16
#endif
constexpr int TF = 16, BOX_ROWS = TSK_WTMA_BOX_ROWS;
template <int N, int W>
struct Geo {
    static_assert(W == 32 || W == 16, "256 B or 128 B rows");
    static constexpr int NT = TF * W;
    static constexpr int CTAS_PER_SM = W == 32 ? 1 : 2;
    static constexpr int R = N / TF;
    static constexpr int TILE_BYTES = N * W * 8;  // 128 / 64 KB at W = 32
    // exchange buffer: half a tile at N = 512 (two rounds), a whole one below
    static constexpr int XROWS = N == 512 ? N / 2 : N;
    using PL = Plan<N, R>;
    static_assert(PL::NST == 2 && PL::radix(1) == 16, "two stages, radix R x 16");
    static constexpr size_t SMEM = TILE_BYTES + XROWS * W * 8 + (PL::TW + N) * 8;
    static constexpr int PW = 2 * R;   // TMEM words parked per thread
    static constexpr int TCOLS = (NT / 128) * PW;  // NT / 128 warps per lane quadrant
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Radix-R stage, exchange, radix-16 stage with twiddles: the arithmetic of
// wide::fft_col<float, N, R, W, INV>. The exchange writes the stage-A outputs
// (rows t R + q) and reads the row pattern (rows t + 16 m); at N = 512 through
// a buffer of half the tile: round 0 moves q < 16 / even m (rows with r % 32 <
// 16), round 1 q >= 16 / odd m.
template <int N, int W, bool INV>
__device__ __forceinline__ void fft_col(float2 (&v)[Geo<N, W>::R], float2* xb, const float2* tw, int t, int w)
{
    constexpr int R = Geo<N, W>::R;
    using PL = typename Geo<N, W>::PL;
    Dft<float, R, INV>::run(v);
    if constexpr (N == 512) {
        float2 ev[R / 2];
#pragma unroll
        for (int q = 0; q < R / 2; ++q)
            xb[(t * 16 + q) * W + w] = v[q];
        __syncthreads();
#pragma unroll
        for (int h = 0; h < R / 2; ++h)
            ev[h] = xb[(h * 16 + t) * W + w];  // m = 2h
        __syncthreads();
#pragma unroll
        for (int q = R / 2; q < R; ++q)
            xb[(t * 16 + q - 16) * W + w] = v[q];
        __syncthreads();
#pragma unroll
        for (int h = 0; h < R / 2; ++h) {
            v[2 * h] = ev[h];
            v[2 * h + 1] = xb[(h * 16 + t) * W + w];  // m = 2h + 1
        }
    } else {
        // rows t R + q out, rows t + 16 m in (whole tile)
#pragma unroll
        for (int q = 0; q < R; ++q)
            xb[(t * R + q) * W + w] = v[q];
        __syncthreads();
#pragma unroll
        for (int m = 0; m < R; ++m)
            v[m] = xb[(t + m * TF) * W + w];
    }
    __syncthreads();
    // stage B: radix 16, Ns = R, butterflies j = t + 16 i (i < R / 16)
    constexpr int P = 16, G = R / P;
#pragma unroll
    for (int i = 0; i < G; ++i) {
        const int jm = (t + i * TF) % PL::ns(1);
#pragma unroll
        for (int r = 1; r < P; ++r) {
            const Tw<float> wv = load_tw<float>(tw + PL::tw_off(1) + jm * (P - 1) + (r - 1));
            v[i + r * G] = cmul_tw<float, INV>(v[i + r * G], wv);
        }
    }
#pragma unroll
    for (int i = 0; i < G; ++i) {
        float2 a[P];
#pragma unroll
        for (int r = 0; r < P; ++r)
            a[r] = v[i + r * G];
        Dft<float, P, INV>::run(a);
#pragma unroll
        for (int r = 0; r < P; ++r)
            v[i + r * G] = a[r];
    }
}

struct Maps {
    CUtensorMap m[2];
};

// Output stores of the forward-split pass (one read, two writes) are marked
// streaming (st.global.cs, evict-first): K1 1.70 -> 1.67 ms at 512^3; the merge
// pass (two reads, one write) lost 1% with them and keeps plain stores
// (profiles/r02_ab_stcs.txt). TSK_WTMA_STCS: bit 0 = K1, bit 1 = K3.
#ifndef TSK_WTMA_STCS
#define TSK_WTMA_STCS 1
#endif
// TSK_WTMA_LDEF=1 (A/B): the TMA tile loads carry an L2 evict-first policy
#ifndef TSK_WTMA_LDEF
#define TSK_WTMA_LDEF 0
#endif
// L2 promotion of the tile loads (CUtensorMapL2promotion: 0 none, 1 64 B, 2 128 B,
// 3 256 B = one row segment; A/B)
#ifndef TSK_WTMA_L2PROMO
#define TSK_WTMA_L2PROMO 3
#endif
template <int MODE>
__device__ __forceinline__ void st_out(float2* p, float2 v)
{
    if constexpr (((TSK_WTMA_STCS) >> MODE) & 1)
        __stcs(p, v);
    else
        *p = v;
}

template <int N, int MODE, int W>
__global__ void __launch_bounds__(Geo<N, W>::NT, Geo<N, W>::CTAS_PER_SM)
    k_wtma(tsk_axis p, const __grid_constant__ Maps maps)
{
    using GE = Geo<N, W>;
    constexpr int R = GE::R, NT = GE::NT;
    using PL = typename GE::PL;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float2* land = reinterpret_cast<float2*>(smem_raw);     // N x W landing tile
    float2* xb = land + N * W;                               // exchange rows
    float2* tw = xb + GE::XROWS * W;                     // stage-B twiddles
    float2* ph = tw + PL::TW;                                // split phase
    __shared__ __align__(8) uint64_t full;
    __shared__ uint32_t tmem_slot;

    const float2* roots = static_cast<const float2*>(p.roots);
    for (int e = threadIdx.x; e < PL::ns(1) * 15; e += NT) {
        const int jm = e / 15, r = e % 15 + 1;
        tw[PL::tw_off(1) + e] = ldg_c(roots + (r * jm * (N / (PL::ns(1) * 16))) % N);
    }
    for (int k = threadIdx.x; k < N; k += NT)
        ph[k] = ldg_c(static_cast<const float2*>(p.phase) + k);

    const int w = threadIdx.x % W;
    const int t = threadIdx.x / W;
    const int64_t inner = p.inner;
    const int64_t cols = inner / W;
    const int64_t tpc = p.outer * cols;
    const int64_t ntiles = tpc * p.ncomp;
    const bool ue = p.use_even, uo = p.use_odd;
    const float scale = (float)p.scale;
    const int64_t rs = (int64_t)TF * inner;
    // inputs per tile: K1 x; K3 B(e) and/or B(o)
    const int nin = MODE == 0 ? 1 : (int)ue + (int)uo;
    const int64_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nloads = mine * nin;

    // x (K1, both children) or B(e) (K3, both inputs) parked in tensor memory:
    // 2R columns per thread, four warps per lane quadrant
    const bool park = ue && uo;
    uint32_t tbase = 0, lane_base = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (park) {
        tbase = tmem_alloc(&tmem_slot, GE::TCOLS);
        const int warp = threadIdx.x / 32;
        lane_base = tbase + ((uint32_t)(32 * (warp % 4)) << 16) + (uint32_t)(GE::PW * (warp / 4));
    } else {
        __syncthreads();
    }

    const FastDiv div_tpc((uint32_t)tpc), div_cols((uint32_t)cols);
    auto coords = [&](int64_t tile, int64_t& c, int64_t& o, int64_t& cb) {
        const uint32_t t32 = (uint32_t)tile;
        const uint32_t c32 = div_tpc.div(t32);
        const uint32_t r32 = t32 - c32 * (uint32_t)tpc;
        const uint32_t o32 = div_cols.div(r32);
        c = c32;
        o = o32;
        cb = r32 - o32 * (uint32_t)cols;
    };
    // load g of this CTA: tile blockIdx.x + (g / nin) gridDim.x, input g % nin
    auto issue = [&](int64_t g) {
        const int64_t tile = blockIdx.x + (g / nin) * gridDim.x;
        const int k = (int)(g % nin);
        const int map = MODE == 0 ? 0 : (ue ? k : 1);
        int64_t c, o, cb;
        coords(tile, c, o, cb);
        const int x = (int)(cb * W), z = (int)(c * p.outer + o);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full)),
                     "r"(GE::TILE_BYTES)
                     : "memory");
#if TSK_WTMA_LDEF
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
        for (int r = 0; r < N; r += BOX_ROWS)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
                "{%3, %4, %5}], [%2], %6;" ::"r"(sa(land + r * W)),
                "l"(&maps.m[map]), "r"(sa(&full)), "r"(x), "r"(r), "r"(z), "l"(pol)
                : "memory");
#else
#pragma unroll
        for (int r = 0; r < N; r += BOX_ROWS)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
                "[%2];" ::"r"(sa(land + r * W)),
                "l"(&maps.m[map]), "r"(sa(&full)), "r"(x), "r"(r), "r"(z)
                : "memory");
#endif
    };
    // one CTA per SM with 130-200 KB of shared memory: the next pass's CTAs
    // cannot co-reside, so they may be released at once (they are scheduled as
    // these retire)
    pdl_trigger();
    pdl_wait();  // the previous pass's output is this pass's input
    if (threadIdx.x == 0 && nloads > 0)
        issue(0);
    int64_t g = 0;
    // take load g into registers, then hand the landing buffer to load g + 1
    auto take = [&](float2(&v)[R]) {
        asm volatile(
            "{\n .reg .pred p;\n WT: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WT;\n}" ::"r"(
                sa(&full)),
            "r"((uint32_t)(g & 1))
            : "memory");
#pragma unroll
        for (int m = 0; m < R; ++m)
            v[m] = land[(t + m * TF) * W + w];
        __syncthreads();
        if (threadIdx.x == 0 && g + 1 < nloads)
            issue(g + 1);
        ++g;
    };

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int64_t c, o, cb;
        coords(tile, c, o, cb);
        const int64_t base = c * p.cstride + o * (int64_t)N * inner + cb * W + w + (int64_t)t * inner;
        float2 v[R];
        if constexpr (MODE == 0) {
            take(v);
            if (uo) {
                if (park)
                    tmem_park<float, R, false>(lane_base, v);  // waited before the restore
#pragma unroll
                for (int m = 0; m < R; ++m)
                    v[m] = cmul_tw<float, false>(v[m], load_tw<float>(ph + t + m * TF));
                fft_col<N, W, false>(v, xb, tw, t, w);
                float2* dd = static_cast<float2*>(p.dst1) + base;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    st_out<MODE>(dd + m * rs, v[m]);
                if (park) {
                    tmem_wait_st();
                    tmem_restore<float, R>(lane_base, v);
                }
            }
            if (ue) {
                fft_col<N, W, false>(v, xb, tw, t, w);
                float2* de = static_cast<float2*>(p.dst0) + base;
#pragma unroll
                for (int m = 0; m < R; ++m)
                    st_out<MODE>(de + m * rs, v[m]);
            }
        } else {
            float2* dst = static_cast<float2*>(p.dst0) + base;
            if (ue) {
                take(v);
                fft_col<N, W, true>(v, xb, tw, t, w);
                if (!uo) {
#pragma unroll
                    for (int m = 0; m < R; ++m)
                        st_out<MODE>(dst + m * rs, scale_c<float>(v[m], scale));
                    continue;
                }
                tmem_park<float, R, false>(lane_base, v);  // waited before the restore
            }
            take(v);
            fft_col<N, W, true>(v, xb, tw, t, w);
#pragma unroll
            for (int m = 0; m < R; ++m)
                v[m] = cmul_tw<float, true>(v[m], load_tw<float>(ph + t + m * TF));
            if (ue) {
                // B(e) back 16 values at a time (the 128-register budget of
                // 512 threads holds v and one chunk)
                tmem_wait_st();
#pragma unroll
                for (int h = 0; h < R / 16; ++h) {
                    uint32_t r32[32];
                    tmem_ld32(lane_base + 32 * h, r32);
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        v[16 * h + i] = cadd(v[16 * h + i], Words<float2>::make(r32 + 2 * i));
                }
            }
#pragma unroll
            for (int m = 0; m < R; ++m)
                st_out<MODE>(dst + m * rs, scale_c<float>(v[m], scale));
        }
    }
    if (park)
        tmem_free(tbase, GE::TCOLS);
}

// ---- host side ------------------------------------------------------------

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder()
{
    static const EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

// [outer * ncomp][n][inner] complex64 tensor as 8-byte elements; box W x 256 x 1
static bool make_map(CUtensorMap* m, const void* base, const tsk_axis& a, int W)
{
    EncodeFn enc = encoder();
    if (!enc)
        return false;
    const cuuint64_t dims[3] = {(cuuint64_t)a.inner, (cuuint64_t)a.n, (cuuint64_t)(a.outer * a.ncomp)};
    const cuuint64_t strides[2] = {(cuuint64_t)a.inner * 8, (cuuint64_t)(a.inner * a.n * 8)};
    const cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)BOX_ROWS, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, W == 32 ? (CUtensorMapL2promotion)TSK_WTMA_L2PROMO : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool disabled()
{
    static const bool v = [] {
        const char* e = getenv("TSK_NO_WTMA");
        return e && e[0] == '1';
    }();
    return v;
}

static int sm_count()
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

template <int N, int MODE, int W>
static int launch(const tsk_axis& a, cudaStream_t st)
{
    using GE = Geo<N, W>;
    if (a.inner % W != 0 || a.cstride != a.outer * N * a.inner || !(a.use_even || a.use_odd))
        return -1;
    const int64_t ntiles = a.outer * (a.inner / W) * a.ncomp;
    if (ntiles >= (int64_t(1) << 31) || a.outer * a.ncomp >= (int64_t(1) << 31) || a.inner >= (int64_t(1) << 31))
        return -1;
    const void* in0 = MODE == 0 ? a.src0 : (a.use_even ? a.src0 : a.src1);
    if ((reinterpret_cast<uintptr_t>(in0) & 15) || (MODE == 1 && (reinterpret_cast<uintptr_t>(a.src1) & 15)))
        return -1;
    Maps maps;
    std::memset(&maps, 0, sizeof(maps));
    if (!make_map(&maps.m[0], in0, a, W))
        return -1;
    if (MODE == 1 && a.use_even && a.use_odd && !make_map(&maps.m[1], a.src1, a, W))
        return -1;
    if (MODE == 1 && !a.use_even)
        maps.m[1] = maps.m[0];
    auto kern = k_wtma<N, MODE, W>;
    constexpr size_t SMEM = GE::SMEM;
    static thread_local int cached_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        if (int e = (int)cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM))
            return e;
        cached_dev = dev;
    }
    const int64_t cap = (int64_t)sm_count() * GE::CTAS_PER_SM;
    const int64_t grid = ntiles < cap ? ntiles : cap;
    const cudaError_t e = launch_pdl(pdl_for(a), kern, (unsigned)(grid > 0 ? grid : 1), GE::NT, SMEM, st, a, maps);
    return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

template <int MODE>
static int dispatch(const tsk_axis& a, cudaStream_t st)
{
    if (disabled() || !a.prec)
        return -1;
    switch (a.n) {
    case 256: return launch<256, MODE, MODE == 1 ? TSK_WTMA_W3_256 : 32>(a, st);
    case 512: return launch<512, MODE, 32>(a, st);
    default: return -1;
    }
}

}  // namespace wtma
}  // namespace tsk

// -1: shape not covered (the caller falls back), else the launch cudaError_t.
extern "C" int tsk_wtma_fwd_split(const tsk_axis* a, void* stream)
{
    return tsk::wtma::dispatch<0>(*a, (cudaStream_t)stream);
}

extern "C" int tsk_wtma_inv_merge(const tsk_axis* a, void* stream)
{
    return tsk::wtma::dispatch<1>(*a, (cudaStream_t)stream);
}
