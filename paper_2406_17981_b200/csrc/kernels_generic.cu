// Generic sm_100a kernels for the split-FFT block-Toeplitz MVM: any axis
// length (mixed radix 2/3/4/5/7/8 + direct prime butterflies), any d, c64 or
// c128, 1x1 or m x m blocks, full or mirror-compressed spectra. Tiles of W
// fibers are staged through shared memory; every FFT stage is a Stockham
// autosort pass between two shared buffers (natural order in and out, so the
// spectra and phases are indexed exactly like the reference's tensors).
//
// These are the correctness backbone (every shape the reference accepts);
// the power-of-two sizes of the headline configs get register-resident fast
// kernels in kernels_fast.cu.
//
// Reference behaviour mirrored (paths relative to /root/reference/proj):
//   forward DFT kernel exp(-2 pi i lk/N), inverse with 1/N  src/core/fft.hpp:7-10
//   split phase P_k = exp(-i pi k/n)                        src/core/tensor.cpp:227-254
//   merge  even = (even + exp(+i pi k/n) odd)/2             src/core/engine_split.cpp:13-37
//   leaf multiply, full / mirror remap                      src/core/kernel.cpp:126-219
#include <cuda_runtime.h>

#include "tsk_common.cuh"

namespace tsk {

// One Stockham stage with compile-time radix R over nf rows of length n.
template <typename T, int R, bool INV>
__device__ __forceinline__ void stage_reg(const typename cx<T>::t* __restrict__ a,
                                          typename cx<T>::t* __restrict__ b, int nf, int pitch,
                                          int n, int ns, const typename cx<T>::t* __restrict__ roots)
{
    using T2 = typename cx<T>::t;
    const int m = n / R;
    const int tstep = n / (ns * R);
    const int total = nf * m;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int f = t / m;
        const int j = t - f * m;
        const int jm = j % ns;
        const T2* x = a + (int64_t)f * pitch;
        T2* y = b + (int64_t)f * pitch;
        T2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
            v[r] = x[j + r * m];
        if (jm > 0) {
#pragma unroll
            for (int r = 1; r < R; ++r)
                v[r] = cmul(v[r], twiddle<T, INV>(roots, r * jm * tstep));
        }
        dft_small<T, R, INV>(v, roots, m);
        const int base = (j - jm) * R + jm;
#pragma unroll
        for (int q = 0; q < R; ++q)
            y[base + q * ns] = v[q];
    }
}

// Direct stage for a large prime radix: one output per thread.
template <typename T, bool INV>
__device__ void stage_direct(const typename cx<T>::t* __restrict__ a,
                             typename cx<T>::t* __restrict__ b, int nf, int pitch, int n, int ns,
                             int R, const typename cx<T>::t* __restrict__ roots)
{
    using T2 = typename cx<T>::t;
    const int m = n / R;
    const int tstep = n / (ns * R);
    const int total = nf * n;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int f = t / n;
        const int rem = t - f * n;
        const int q = rem / m;
        const int j = rem - q * m;
        const int jm = j % ns;
        const T2* x = a + (int64_t)f * pitch;
        T2 acc = make_c<T>(0, 0);
        for (int r = 0; r < R; ++r) {
            T2 xv = x[j + r * m];
            if (jm > 0 && r > 0)
                xv = cmul(xv, twiddle<T, INV>(roots, r * jm * tstep));
            acc = cadd(acc, cmul(xv, twiddle<T, INV>(roots, ((r * q) % R) * m)));
        }
        b[(int64_t)f * pitch + (j - jm) * R + jm + q * ns] = acc;
    }
}

// Full mixed-radix FFT of nf rows; returns the buffer holding the result.
template <typename T, bool INV>
__device__ typename cx<T>::t* fft_rows(typename cx<T>::t* a, typename cx<T>::t* b, int nf,
                                       int pitch, const tsk_axis& p,
                                       const typename cx<T>::t* __restrict__ roots)
{
    const int n = (int)p.n;
    int ns = 1;
    for (int s = 0; s < p.nrad; ++s) {
        const int R = p.rad[s];
        switch (R) {
        case 2: stage_reg<T, 2, INV>(a, b, nf, pitch, n, ns, roots); break;
        case 3: stage_reg<T, 3, INV>(a, b, nf, pitch, n, ns, roots); break;
        case 4: stage_reg<T, 4, INV>(a, b, nf, pitch, n, ns, roots); break;
        case 5: stage_reg<T, 5, INV>(a, b, nf, pitch, n, ns, roots); break;
        case 7: stage_reg<T, 7, INV>(a, b, nf, pitch, n, ns, roots); break;
        case 8: stage_reg<T, 8, INV>(a, b, nf, pitch, n, ns, roots); break;
        default: stage_direct<T, INV>(a, b, nf, pitch, n, ns, R, roots); break;
        }
        __syncthreads();
        typename cx<T>::t* t = a;
        a = b;
        b = t;
        ns *= R;
    }
    return a;
}

struct TileGeom {
    int64_t g0;  // first fiber of the tile
    int nfib;    // valid fibers in the tile
};

// Element e of a tile (component c, fiber f, position k): coalesced mapping.
template <typename T>
__device__ __forceinline__ bool tile_elem(const tsk_axis& p, int W, const TileGeom& tg, int e,
                                          int& c, int& f, int& k, int64_t& addr)
{
    const int n = (int)p.n;
    const int per = W * n;
    c = e / per;
    const int r = e - c * per;
    if (p.inner == 1) {
        f = r / n;
        k = r - f * n;
    } else {
        k = r / W;
        f = r - k * W;
    }
    if (f >= tg.nfib)
        return false;
    const int64_t g = tg.g0 + f;
    const int64_t o = g / p.inner;
    const int64_t i = g - o * p.inner;
    addr = (int64_t)c * p.cstride + (o * p.n + k) * p.inner + i;
    return true;
}

template <typename T>
__global__ void __launch_bounds__(256) k_fwd_split(tsk_axis p, int W)
{
    using T2 = typename cx<T>::t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = (int)p.n;
    const int pitch = n | 1;
    const int rows = p.ncomp * W;
    T2* A = reinterpret_cast<T2*>(smem_raw);
    T2* B = A + (int64_t)rows * pitch;
    T2* Cb = B + (int64_t)rows * pitch;
    const T2* src = static_cast<const T2*>(p.src0);
    T2* de = static_cast<T2*>(p.dst0);
    T2* dodd = static_cast<T2*>(p.dst1);
    const T2* __restrict__ roots = static_cast<const T2*>(p.roots);
    const T2* __restrict__ phase = static_cast<const T2*>(p.phase);
    const int64_t nfibers = p.outer * p.inner;
    const int64_t ntiles = (nfibers + W - 1) / W;
    const int nelem = rows * n;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        TileGeom tg{tile * W, (int)(nfibers - tile * W < W ? nfibers - tile * W : W)};
        for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
            int c, f, k;
            int64_t addr;
            if (!tile_elem<T>(p, W, tg, e, c, f, k, addr))
                continue;
            const T2 v = src[addr];
            const int64_t s = (int64_t)(c * W + f) * pitch + k;
            if (p.use_even)
                A[s] = v;
            if (p.use_odd)
                Cb[s] = cmul(v, phase[k]);
        }
        __syncthreads();
        if (p.use_even) {
            T2* R = fft_rows<T, false>(A, B, rows, pitch, p, roots);
            for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
                int c, f, k;
                int64_t addr;
                if (tile_elem<T>(p, W, tg, e, c, f, k, addr))
                    de[addr] = R[(int64_t)(c * W + f) * pitch + k];
            }
            __syncthreads();
        }
        if (p.use_odd) {
            T2* R = fft_rows<T, false>(Cb, B, rows, pitch, p, roots);
            for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
                int c, f, k;
                int64_t addr;
                if (tile_elem<T>(p, W, tg, e, c, f, k, addr))
                    dodd[addr] = R[(int64_t)(c * W + f) * pitch + k];
            }
            __syncthreads();
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_inv_merge(tsk_axis p, int W)
{
    using T2 = typename cx<T>::t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = (int)p.n;
    const int pitch = n | 1;
    const int rows = p.ncomp * W;
    T2* A = reinterpret_cast<T2*>(smem_raw);
    T2* B = A + (int64_t)rows * pitch;
    T2* Cb = B + (int64_t)rows * pitch;
    const T2* se = static_cast<const T2*>(p.src0);
    const T2* so = static_cast<const T2*>(p.src1);
    T2* dst = static_cast<T2*>(p.dst0);
    const T2* __restrict__ roots = static_cast<const T2*>(p.roots);
    const T2* __restrict__ phase = static_cast<const T2*>(p.phase);
    const int64_t nfibers = p.outer * p.inner;
    const int64_t ntiles = (nfibers + W - 1) / W;
    const int nelem = rows * n;
    const T scale = (T)p.scale;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        TileGeom tg{tile * W, (int)(nfibers - tile * W < W ? nfibers - tile * W : W)};
        for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
            int c, f, k;
            int64_t addr;
            if (!tile_elem<T>(p, W, tg, e, c, f, k, addr))
                continue;
            const int64_t s = (int64_t)(c * W + f) * pitch + k;
            if (p.use_even)
                A[s] = se[addr];
            if (p.use_odd)
                Cb[s] = so[addr];
        }
        __syncthreads();
        T2* Re = nullptr;
        T2* Ro = nullptr;
        if (p.use_even)
            Re = fft_rows<T, true>(A, B, rows, pitch, p, roots);
        if (p.use_odd)
            Ro = fft_rows<T, true>(Cb, Re == A ? B : A, rows, pitch, p, roots);
        for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
            int c, f, k;
            int64_t addr;
            if (!tile_elem<T>(p, W, tg, e, c, f, k, addr))
                continue;
            const int64_t s = (int64_t)(c * W + f) * pitch + k;
            T2 acc = make_c<T>(0, 0);
            if (Re)
                acc = Re[s];
            if (Ro)
                acc = cadd(acc, cmulc(Ro[s], phase[k]));
            dst[addr] = make_c<T>(scale * acc.x, scale * acc.y);
        }
        __syncthreads();
    }
}

// Mirror-remap bookkeeping of one fiber (all axes but the leaf axis d-1).
__device__ __forceinline__ void fiber_prefix(const tsk_spectra& sp, int beta, int64_t g,
                                             int64_t& off, uint32_t& neg)
{
    const uint32_t bits = sp.branch_bits[beta];
    const int d = sp.d;
    off = 0;
    neg = 0;
    if (!sp.compressed) {
        off = g * sp.levels[d - 1];
        return;
    }
    int64_t stride = stored_len(sp.levels[d - 1], (bits >> (d - 1)) & 1u);
    for (int a = d - 2; a >= 0; --a) {
        const int64_t na = sp.levels[a];
        const int64_t ka = g % na;
        g /= na;
        const int odd = (bits >> a) & 1u;
        bool mirrored;
        const int64_t src = mirror_src(na, odd, ka, mirrored);
        off += src * stride;
        stride *= stored_len(na, odd);
        if (mirrored)
            for (int u = 0; u < sp.n_unique; ++u)
                neg ^= ((sp.skew_mask[u] >> a) & 1u) << u;
    }
}

// y_i = sum_j T[b](map(i,j)) x_j at every (fiber, k) of the tile, in place.
template <typename T>
__device__ void leaf_multiply(typename cx<T>::t* Rb, int W, int pitch, int nfib, int n,
                              const tsk_spectra& sp, int beta, const int64_t* fib_off,
                              const uint32_t* fib_neg)
{
    using T2 = typename cx<T>::t;
    const T2* __restrict__ spec = static_cast<const T2*>(sp.data) + sp.branch_base[beta];
    const int64_t bstride = sp.block_elems[beta];
    const int m = sp.m;
    const int d = sp.d;
    const int odd_last = (sp.branch_bits[beta] >> (d - 1)) & 1u;
    const int total = nfib * n;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int f = t / n;
        const int k = t - f * n;
        int64_t idx = fib_off[f];
        uint32_t neg = fib_neg[f];
        if (sp.compressed) {
            bool mirrored;
            idx += mirror_src(n, odd_last, k, mirrored);
            if (mirrored)
                for (int u = 0; u < sp.n_unique; ++u)
                    neg ^= ((sp.skew_mask[u] >> (d - 1)) & 1u) << u;
        } else {
            idx += k;
        }
        T2 x[TSK_MAX_M];
        for (int j = 0; j < m; ++j)
            x[j] = Rb[(int64_t)(j * W + f) * pitch + k];
        for (int i = 0; i < m; ++i) {
            T2 acc = make_c<T>(0, 0);
            for (int j = 0; j < m; ++j) {
                const int u = sp.comp_map[i * m + j];
                T2 tv = ldg_c(spec + (int64_t)u * bstride + idx);
                if ((neg >> u) & 1u)
                    tv = make_c<T>(-tv.x, -tv.y);
                acc = cadd(acc, cmul(x[j], tv));
            }
            Rb[(int64_t)(i * W + f) * pitch + k] = acc;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_leaf_pair(tsk_axis p, tsk_spectra sp, int W)
{
    using T2 = typename cx<T>::t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = (int)p.n;
    const int pitch = n | 1;
    const int rows = p.ncomp * W;
    T2* A = reinterpret_cast<T2*>(smem_raw);
    T2* B = A + (int64_t)rows * pitch;
    T2* Cb = B + (int64_t)rows * pitch;
    int64_t* fib_off = reinterpret_cast<int64_t*>(Cb + (int64_t)rows * pitch);  // [2][W]
    uint32_t* fib_neg = reinterpret_cast<uint32_t*>(fib_off + 2 * W);           // [2][W]
    const T2* src = static_cast<const T2*>(p.src0);
    T2* dst = static_cast<T2*>(p.dst0);
    const T2* __restrict__ roots = static_cast<const T2*>(p.roots);
    const T2* __restrict__ phase = static_cast<const T2*>(p.phase);
    const int64_t nfibers = p.outer * p.inner;
    const int64_t ntiles = (nfibers + W - 1) / W;
    const int nelem = rows * n;
    const T scale = (T)p.scale;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        TileGeom tg{tile * W, (int)(nfibers - tile * W < W ? nfibers - tile * W : W)};
        for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
            int c, f, k;
            int64_t addr;
            if (!tile_elem<T>(p, W, tg, e, c, f, k, addr))
                continue;
            const T2 v = src[addr];
            const int64_t s = (int64_t)(c * W + f) * pitch + k;
            if (p.use_even)
                A[s] = v;
            if (p.use_odd)
                Cb[s] = cmul(v, phase[k]);
        }
        for (int t = threadIdx.x; t < 2 * W; t += blockDim.x) {
            const int beta = t / W;
            const int f = t - beta * W;
            int64_t off = 0;
            uint32_t neg = 0;
            if (f < tg.nfib)
                fiber_prefix(sp, beta, tg.g0 + f, off, neg);
            fib_off[t] = off;
            fib_neg[t] = neg;
        }
        __syncthreads();
        T2* Re = nullptr;
        T2* Ro = nullptr;
        if (p.use_even) {
            T2* r = fft_rows<T, false>(A, B, rows, pitch, p, roots);
            leaf_multiply<T>(r, W, pitch, tg.nfib, n, sp, 0, fib_off, fib_neg);
            __syncthreads();
            Re = fft_rows<T, true>(r, r == A ? B : A, rows, pitch, p, roots);
        }
        if (p.use_odd) {
            T2* S = Re ? (Re == A ? B : A) : B;
            T2* r = fft_rows<T, false>(Cb, S, rows, pitch, p, roots);
            leaf_multiply<T>(r, W, pitch, tg.nfib, n, sp, 1, fib_off + W, fib_neg + W);
            __syncthreads();
            Ro = fft_rows<T, true>(r, r == Cb ? S : Cb, rows, pitch, p, roots);
        }
        for (int e = threadIdx.x; e < nelem; e += blockDim.x) {
            int c, f, k;
            int64_t addr;
            if (!tile_elem<T>(p, W, tg, e, c, f, k, addr))
                continue;
            const int64_t s = (int64_t)(c * W + f) * pitch + k;
            T2 acc = make_c<T>(0, 0);
            if (Re)
                acc = Re[s];
            if (Ro)
                acc = cadd(acc, cmulc(Ro[s], phase[k]));
            dst[addr] = make_c<T>(scale * acc.x, scale * acc.y);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launchers

static int elem_size(int prec) { return prec ? 8 : 16; }

static size_t tile_smem(const tsk_axis& a, int W, bool leaf)
{
    const size_t pitch = (size_t)(a.n | 1);
    size_t b = 3 * (size_t)a.ncomp * W * pitch * elem_size(a.prec);
    if (leaf)
        b += (size_t)2 * W * (sizeof(int64_t) + sizeof(uint32_t));
    return b;
}

// Dynamic shared memory these kernels may use. The opt-in attribute is set to this
// one value at every launch: a per-launch value would race between host threads
// launching axes of different length (one lowers it under the other's launch).
static constexpr size_t kSmemLimit = 200 * 1024;

static int choose_w(const tsk_axis& a, bool leaf, int& W, size_t& smem)
{
    const size_t limit = kSmemLimit;
    const int64_t nfib = a.outer * a.inner;
    const int target = a.prec ? 4096 : 2048;  // complex elements per tile
    int w = (int)std::max<int64_t>(1, target / (a.ncomp * a.n));
    if (a.inner > 1)
        w = std::max(w, a.prec ? 16 : 8);
    w = (int)std::min<int64_t>(w, std::max<int64_t>(nfib, 1));
    while (w > 1 && tile_smem(a, w, leaf) > limit)
        --w;
    if (tile_smem(a, w, leaf) > limit)
        return -1;  // axis too long to stage a fiber: the long-axis passes take it
    W = w;
    smem = tile_smem(a, w, leaf);
    return 0;
}

static int grid_for(int64_t ntiles)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sms * 8));
}

template <typename K>
static int launch(K kernel, size_t smem, int64_t ntiles, cudaStream_t st, const tsk_axis& a,
                  int W)
{
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemLimit);
    if (e != cudaSuccess)
        return (int)e;
    kernel<<<grid_for(ntiles), 256, smem, st>>>(a, W);
    return (int)cudaGetLastError();
}

}  // namespace tsk

using namespace tsk;

extern "C" int tsk_generic_fwd_split(const tsk_axis* a, void* stream)
{
    int W;
    size_t smem;
    if (int e = choose_w(*a, false, W, smem))
        return e;
    const int64_t nt = (a->outer * a->inner + W - 1) / W;
    auto st = static_cast<cudaStream_t>(stream);
    return a->prec ? launch(k_fwd_split<float>, smem, nt, st, *a, W)
                   : launch(k_fwd_split<double>, smem, nt, st, *a, W);
}

extern "C" int tsk_generic_inv_merge(const tsk_axis* a, void* stream)
{
    int W;
    size_t smem;
    if (int e = choose_w(*a, false, W, smem))
        return e;
    const int64_t nt = (a->outer * a->inner + W - 1) / W;
    auto st = static_cast<cudaStream_t>(stream);
    return a->prec ? launch(k_inv_merge<float>, smem, nt, st, *a, W)
                   : launch(k_inv_merge<double>, smem, nt, st, *a, W);
}

extern "C" int tsk_generic_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream)
{
    int W;
    size_t smem;
    if (a->inner != 1)
        return (int)cudaErrorInvalidValue;
    if (int e = choose_w(*a, true, W, smem))
        return e;
    const int64_t nt = (a->outer + W - 1) / W;
    auto st = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (a->prec) {
        e = cudaFuncSetAttribute(k_leaf_pair<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemLimit);
        if (e != cudaSuccess)
            return (int)e;
        k_leaf_pair<float><<<grid_for(nt), 256, smem, st>>>(*a, *sp, W);
    } else {
        e = cudaFuncSetAttribute(k_leaf_pair<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemLimit);
        if (e != cudaSuccess)
            return (int)e;
        k_leaf_pair<double><<<grid_for(nt), 256, smem, st>>>(*a, *sp, W);
    }
    return (int)cudaGetLastError();
}
