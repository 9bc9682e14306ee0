// Microbenchmark (not product code): the K1/K3 strided-tile pattern moved by
// TMA (cp.async.bulk.tensor) instead of per-thread loads/stores. A persistent
// CTA per SM streams tiles of `rows` x W complex64 (one fiber of a strided
// axis, W columns wide) through S shared-memory stages; K1 pattern = each
// tile stored twice (even + odd child), K3 pattern = two tiles loaded, one
// stored. Reports GB/s of (reads + writes).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase)
{
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(sa(b)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load2(const CUtensorMap* m, void* dst, uint64_t* bar, int x, int y)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            sa(dst)),
        "l"(m), "r"(sa(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tma_store2(const CUtensorMap* m, const void* src, int x, int y)
{
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m), "r"(sa(src)),
                 "r"(x), "r"(y)
                 : "memory");
}

// tile = 512 rows x W cols (c64 = 8-byte elements), loaded as 512/BR boxes of BR rows
template <int W, int S, int MODE>
__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap ms, const __grid_constant__ CUtensorMap ms2,
                                      const __grid_constant__ CUtensorMap md0, const __grid_constant__ CUtensorMap md1,
                                      long inner, long outer)
{
    constexpr int BR = 256;
    constexpr int TB = 512 * W * 8;  // tile bytes
    constexpr int NIN = MODE == 0 ? 1 : 2;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full[S];
    const long cols = inner / W, ntiles = outer * cols;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0)
        return;
    long mine = 0;
    for (long t = blockIdx.x; t < ntiles; t += gridDim.x)
        ++mine;
    auto issue = [&](long i) {
        const long t = blockIdx.x + i * gridDim.x;
        const int s = (int)(i % S);
        const int o = (int)(t / cols), c0 = (int)((t % cols) * W);
        mbar_expect(&full[s], NIN * TB);
        for (int in = 0; in < NIN; ++in)
            for (int r = 0; r < 512; r += BR)
                tma_load2(in ? &ms2 : &ms, sm + (size_t)(s * NIN + in) * TB + (size_t)r * W * 8, &full[s], c0,
                          o * 512 + r);
    };
    for (long i = 0; i < S && i < mine; ++i)
        issue(i);
    for (long i = 0; i < mine; ++i) {
        const long t = blockIdx.x + i * gridDim.x;
        const int s = (int)(i % S);
        mbar_wait(&full[s], (uint32_t)((i / S) & 1));
        const int o = (int)(t / cols), c0 = (int)((t % cols) * W);
        for (int r = 0; r < 512; r += BR) {
            tma_store2(&md0, sm + (size_t)(s * NIN) * TB + (size_t)r * W * 8, c0, o * 512 + r);
            if (MODE == 0)
                tma_store2(&md1, sm + (size_t)(s * NIN) * TB + (size_t)r * W * 8, c0, o * 512 + r);
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // stage s is reused by tile i + S: its stores must have read the smem
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (i + S < mine)
            issue(i + S);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static EncodeFn get_encode()
{
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (EncodeFn)fn;
}

static CUtensorMap make_map(EncodeFn enc, void* base, long inner, long rows, int W, int BR)
{
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)inner * 8};
    cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)BR};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        printf("encode failed %d\n", (int)r);
    return m;
}

template <int W, int S, int MODE>
void run(EncodeFn enc, float2* a, float2* b, float2* c, long inner, long total)
{
    const long rows = total / inner, outer = rows / 512;
    CUtensorMap ms = make_map(enc, a, inner, rows, W, 256);
    CUtensorMap ms2 = make_map(enc, b, inner, rows, W, 256);
    CUtensorMap md0 = make_map(enc, MODE == 0 ? b : c, inner, rows, W, 256);
    CUtensorMap md1 = make_map(enc, c, inner, rows, W, 256);
    const int NIN = MODE == 0 ? 1 : 2;
    const size_t smem = (size_t)S * NIN * 512 * W * 8;
    auto k = k_tma<W, S, MODE>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        smem > 227 * 1024) {
        printf("W=%d S=%d mode=%d: smem %zu too large\n", W, S, MODE, smem);
        return;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i)
        k<<<148, 128, smem>>>(ms, ms2, md0, md1, inner, outer);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i)
        k<<<148, 128, smem>>>(ms, ms2, md0, md1, inner, outer);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t err = cudaGetLastError();
    float ms_;
    cudaEventElapsedTime(&ms_, e0, e1);
    ms_ /= reps;
    printf("TMA %s W=%2d (%3d B rows) S=%d inner=%7ld  %.3f ms  %.0f GB/s  %s\n", MODE == 0 ? "K1 1r2w" : "K3 2r1w", W,
           W * 8, S, inner, ms_, 3.0 * total * 8 / (ms_ * 1e-3) / 1e9, cudaGetErrorString(err));
}

int main()
{
    const long total = 512L * 512 * 512;
    float2 *a, *b, *c;
    cudaMalloc(&a, total * 8);
    cudaMalloc(&b, total * 8);
    cudaMalloc(&c, total * 8);
    cudaMemset(a, 0, total * 8);
    cudaMemset(b, 0, total * 8);
    EncodeFn enc = get_encode();
    if (!enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    for (long inner : {262144L, 512L}) {
        run<16, 2, 0>(enc, a, b, c, inner, total);
        run<16, 3, 0>(enc, a, b, c, inner, total);
        run<32, 1, 0>(enc, a, b, c, inner, total);
        run<8, 4, 0>(enc, a, b, c, inner, total);
        run<8, 6, 0>(enc, a, b, c, inner, total);
        run<16, 1, 1>(enc, a, b, c, inner, total);
        run<8, 3, 1>(enc, a, b, c, inner, total);
    }
    // contiguous reference: plain copy via TMA with wide rows
    return 0;
}
