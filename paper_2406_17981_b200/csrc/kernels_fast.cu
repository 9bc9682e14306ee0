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
};

// Fill the per-stage twiddle table (w_N^{r * jm * N/(Ns p)}) and the phase
// table P_k = exp(-i pi k/N) from the operator's double-accurate root/phase
// tables (global) into shared memory.
template <typename T, int N>
__device__ void fill_tables(typename cx<T>::t* tw, typename cx<T>::t* ph,
                            const typename cx<T>::t* __restrict__ roots,
                            const typename cx<T>::t* __restrict__ phase)
{
    using P = Plan<N>;
#pragma unroll
    for (int s = 1; s < P::NST; ++s) {
        constexpr int dummy = 0;
        (void)dummy;
        const int p = P::radix(s), ns = P::ns(s);
        const int cnt = ns * (p - 1);
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const int jm = e / (p - 1), r = e % (p - 1) + 1;
            tw[P::tw_off(s) + e] = ldg_c(roots + (r * jm * (N / (ns * p))) % N);
        }
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x)
        ph[k] = ldg_c(phase + k);
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
// sbuf: two ping-pong buffers; sidx(k, pos) gives the element index of
// (transform k, position pos) inside one buffer.
template <typename T, int N, bool INV, int K, class SIdx>
__device__ __forceinline__ void fft_rows(typename cx<T>::t (&v)[K][8], typename cx<T>::t* buf0,
                                         typename cx<T>::t* buf1, const SIdx& sidx,
                                         const typename cx<T>::t* tw, int t)
{
    using T2 = typename cx<T>::t;
    using PL = Plan<N>;
    constexpr int TF = PL::TF;
#pragma unroll
    for (int s = 0; s < PL::NST; ++s) {
        const int p = PL::radix(s);
        const int ns = PL::ns(s);
        const int G = 8 / p;
        // twiddles (stage > 0): input r of butterfly j scaled by w^{r jm ...}
        if (s > 0) {
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int j = t + i * TF;
                const int jm = j % ns;
#pragma unroll
                for (int r = 1; r < p; ++r) {
                    T2 w = tw[PL::tw_off(s) + jm * (p - 1) + (r - 1)];
                    if (INV)
                        w.y = -w.y;
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        v[k][i + r * G] = cmul(v[k][i + r * G], w);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (p == 8)
                butterfly<T, 8, INV>(v[k], 0);
            else if (p == 4) {
#pragma unroll
                for (int i = 0; i < 2; ++i)
                    butterfly<T, 4, INV>(v[k], i);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    butterfly<T, 2, INV>(v[k], i);
            }
        }
        if (s == PL::NST - 1)
            break;  // last stage outputs are already in the row pattern
        T2* buf = (s & 1) ? buf1 : buf0;
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const int j = t + i * TF;
            const int jm = j % ns;
            const int base = (j - jm) * p + jm;
#pragma unroll
            for (int q = 0; q < p; ++q)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    buf[sidx(k, base + q * ns)] = v[k][i + q * G];
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int k = 0; k < K; ++k)
                v[k][m] = buf[sidx(k, t + m * TF)];
    }
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

// MODE 0: K1 forward split (even/odd by use flags); MODE 1: K3 inverse merge.
// Persistent CTAs; the next tile's loads are issued before the current tile's
// transforms so HBM reads overlap the shared-memory exchanges.
template <typename T, int N, int W, int MODE>
__global__ void __launch_bounds__(N / 8 * W) k_strided(tsk_axis p)
{
    using T2 = typename cx<T>::t;
    using PL = Plan<N>;
    constexpr int TF = PL::TF;
    constexpr int NIN = MODE == 0 ? 1 : 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T2* tw = reinterpret_cast<T2*>(smem_raw);
    T2* ph = tw + PL::TW;
    T2* buf0 = ph + N;
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

    auto tile_base = [&](int64_t tile) {
        const int64_t c = tile / tiles_per_comp;
        const int64_t r = tile - c * tiles_per_comp;
        const int64_t o = r / cols;
        const int64_t i0 = (r - o * cols) * W;
        return c * p.cstride + o * (int64_t)N * inner + i0 + w;
    };
    T2 nx[NIN][8];
    int64_t tile = blockIdx.x;
    if (tile < ntiles) {
        const int64_t b = tile_base(tile);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int64_t a = b + (int64_t)(t + m * TF) * inner;
            nx[0][m] = ld0 ? s0[a] : make_c<T>(0, 0);
            if (NIN == 2)
                nx[NIN - 1][m] = ld1 ? s1[a] : make_c<T>(0, 0);
        }
    }
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile_base(tile);
        T2 v[2][8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (MODE == 0) {
                v[0][m] = nx[0][m];
                v[1][m] = cmul(nx[0][m], ph[t + m * TF]);
            } else {
                v[0][m] = nx[0][m];
                v[1][m] = nx[NIN - 1][m];
            }
        }
        const int64_t nt = tile + gridDim.x;
        if (nt < ntiles) {
            const int64_t b = tile_base(nt);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int64_t a = b + (int64_t)(t + m * TF) * inner;
                nx[0][m] = ld0 ? s0[a] : make_c<T>(0, 0);
                if (NIN == 2)
                    nx[NIN - 1][m] = ld1 ? s1[a] : make_c<T>(0, 0);
            }
        }
        if (MODE == 0) {
            fft_rows<T, N, false, 2>(v, buf0, buf1, sidx, tw, t);
            T2* de = static_cast<T2*>(p.dst0);
            T2* dodd = static_cast<T2*>(p.dst1);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int64_t a = base + (int64_t)(t + m * TF) * inner;
                if (ue)
                    de[a] = v[0][m];
                if (uo)
                    dodd[a] = v[1][m];
            }
        } else {
            fft_rows<T, N, true, 2>(v, buf0, buf1, sidx, tw, t);
            T2* dst = static_cast<T2*>(p.dst0);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const T2 acc = cadd(v[0][m], cmulc(v[1][m], ph[t + m * TF]));
                dst[base + (int64_t)(t + m * TF) * inner] = make_c<T>(scale * acc.x, scale * acc.y);
            }
        }
        // the next tile's first exchange reuses buf0; with two or more
        // exchanges the later __syncthreads already orders it
        if (PL::NST - 1 < 2)
            __syncthreads();
    }
}

// --------------------------------------------------------------------- K2

// Leaf pair on the contiguous last axis; F fibers per CTA, M components
// multiplied by the m x m spectra in registers.
template <typename T, int N, int M, int F>
__global__ void __launch_bounds__(N / 8 * F) k_leaf(tsk_axis p, tsk_spectra sp)
{
    using T2 = typename cx<T>::t;
    using PL = Plan<N>;
    constexpr int TF = PL::TF;
    constexpr int FP = N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T2* tw = reinterpret_cast<T2*>(smem_raw);
    T2* ph = tw + PL::TW;
    T2* buf0 = ph + N;
    T2* buf1 = buf0 + M * F * FP;
    T2* stash = buf1 + M * F * FP;  // the tile's input, reused by the odd branch
    fill_tables<T, N>(tw, ph, static_cast<const T2*>(p.roots), static_cast<const T2*>(p.phase));
    __syncthreads();

    const int f = threadIdx.x / TF;
    const int t = threadIdx.x % TF;
    const int64_t nfib = p.outer;
    const int64_t ntiles = (nfib + F - 1) / F;
    const T scale = (T)p.scale;
    const T2* src = static_cast<const T2*>(p.src0);
    T2* dst = static_cast<T2*>(p.dst0);
    const T2* spec = static_cast<const T2*>(sp.data);
    FiberIdx<N, sizeof(T2)> sidx{f * FP, F * FP};
    const int d = sp.d;
    const int U = sp.n_unique;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t g = tile * F + f;
        const bool valid = g < nfib;
        const int64_t gv = valid ? g : nfib - 1;
        T2 acc[M][8];
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
                    // each thread stashes and re-reads only its own elements
                    T2* sl = stash + (c * F + f) * FP + t + m * TF;
                    if (beta == 0 || !p.use_even) {
                        const T2 x = src[c * p.cstride + gv * N + t + m * TF];
                        if (beta == 0 && p.use_odd)
                            *sl = x;
                        v[c][m] = beta ? cmul(x, ph[t + m * TF]) : x;
                    } else {
                        v[c][m] = cmul(*sl, ph[t + m * TF]);
                    }
                }
            fft_rows<T, N, false, M>(v, buf0, buf1, sidx, tw, t);
            // spectra offset of this fiber (mirror remap of the outer axes)
            const uint32_t bits = sp.branch_bits[beta];
            int64_t off = 0;
            uint32_t neg = 0;
            int odd_last = (bits >> (d - 1)) & 1u;
            if (!sp.compressed) {
                off = gv * N;
            } else {
                int64_t gg = gv;
                int64_t stride = stored_len(N, odd_last);
                for (int a = d - 2; a >= 0; --a) {
                    const int64_t na = sp.levels[a];
                    const int64_t ka = gg % na;
                    gg /= na;
                    const int odd = (bits >> a) & 1u;
                    bool mir;
                    off += mirror_src(na, odd, ka, mir) * stride;
                    stride *= stored_len(na, odd);
                    if (mir)
                        for (int u = 0; u < U; ++u)
                            neg ^= ((sp.skew_mask[u] >> a) & 1u) << u;
                }
            }
            const T2* sb = spec + sp.branch_base[beta];
            const int64_t bst = sp.block_elems[beta];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int k = t + m * TF;
                int64_t idx = off;
                uint32_t ng = neg;
                if (sp.compressed) {
                    bool mir;
                    idx += mirror_src(N, odd_last, k, mir);
                    if (mir)
                        for (int u = 0; u < U; ++u)
                            ng ^= ((sp.skew_mask[u] >> (d - 1)) & 1u) << u;
                } else {
                    idx += k;
                }
                if (M == 1) {
                    T2 s = ldg_c(sb + idx);
                    if (ng & 1u)
                        s = make_c<T>(-s.x, -s.y);
                    v[0][m] = cmul(v[0][m], s);
                } else {
                    // block-symmetric 3x3, canonical map [[0,1,2],[1,3,4],[2,4,5]]
                    T2 sv[6];
#pragma unroll
                    for (int u = 0; u < 6; ++u) {
                        T2 s = ldg_c(sb + u * bst + idx);
                        if ((ng >> u) & 1u)
                            s = make_c<T>(-s.x, -s.y);
                        sv[u] = s;
                    }
                    constexpr int cmap[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
                    T2 x[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        x[c] = v[c][m];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        T2 a = make_c<T>(0, 0);
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            const T2 s = sv[cmap[i * 3 + j]];
                            a.x = fma(x[j].x, s.x, fma(-x[j].y, s.y, a.x));
                            a.y = fma(x[j].x, s.y, fma(x[j].y, s.x, a.y));
                        }
                        v[i][m] = a;
                    }
                }
            }
            // the forward transform's last exchange buffer is free once every
            // thread passed it; order the inverse's first exchange after it
            __syncthreads();
            fft_rows<T, N, true, M>(v, buf0, buf1, sidx, tw, t);
#pragma unroll
            for (int c = 0; c < M; ++c)
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (beta == 0)
                        acc[c][m] = v[c][m];
                    else if (p.use_even)
                        acc[c][m] = cadd(acc[c][m], cmulc(v[c][m], ph[t + m * TF]));
                    else
                        acc[c][m] = cmulc(v[c][m], ph[t + m * TF]);
                }
            __syncthreads();
        }
        if (valid) {
#pragma unroll
            for (int c = 0; c < M; ++c)
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    dst[c * p.cstride + g * N + t + m * TF] =
                        make_c<T>(scale * acc[c][m].x, scale * acc[c][m].y);
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
    const size_t smem = sizeof(T2) * (Plan<N>::TW + N + 2 * 2 * N * W);
    if (smem > 227 * 1024)
        return -1;
    auto kern = k_strided<T, N, W, MODE>;
    int cap = 0;
    if (int e = prep(kern, smem, N / 8 * W, cap))
        return e;
    const int64_t ntiles = a.outer * (a.inner / W) * a.ncomp;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, cap));
    kern<<<(unsigned)grid, N / 8 * W, smem, st>>>(a);
    return (int)cudaGetLastError();
}

template <typename T, int N, int M>
static int launch_leaf(const tsk_axis& a, const tsk_spectra& sp, cudaStream_t st)
{
    constexpr int F = (N / 8 >= 128) ? 1 : 128 / (N / 8);
    using T2 = typename cx<T>::t;
    const size_t smem = sizeof(T2) * (Plan<N>::TW + N + 3 * M * F * N);
    if (smem > 227 * 1024)
        return -1;
    auto kern = k_leaf<T, N, M, F>;
    int cap = 0;
    if (int e = prep(kern, smem, N / 8 * F, cap))
        return e;
    const int64_t ntiles = (a.outer + F - 1) / F;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, cap));
    kern<<<(unsigned)grid, N / 8 * F, smem, st>>>(a, sp);
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
