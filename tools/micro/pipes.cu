// Microbenchmark (not product code): per-SM throughput of the data-movement
// instructions a leaf-pass redesign would trade against each other —
// shared-memory LDS.64 (conflict-free), warp shuffle (SHFL.32), and tensor
// memory reads (tcgen05.ld 32x32b.x16) — at a given number of warps per SM.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ITERS = 4096;

__global__ void k_lds(float* out, int warps)
{
    extern __shared__ float2 sm[];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x)
        sm[i] = make_float2(i, -i);
    __syncthreads();
    float2 acc = make_float2(0, 0);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
#pragma unroll 8
    for (int it = 0; it < ITERS; ++it) {
        const float2 v = sm[(w * 32 + lane + it * 64) & 4095];
        acc.x += v.x;
        acc.y += v.y;
    }
    if (acc.x == 1.2345f)
        out[threadIdx.x] = acc.y;
}

__global__ void k_shfl(float* out, int warps)
{
    float a = threadIdx.x, b = -a, c = a * 0.5f, d = a * 2.f;
#pragma unroll 8
    for (int it = 0; it < ITERS; ++it) {
        a = __shfl_xor_sync(0xffffffffu, a, 1);
        b = __shfl_xor_sync(0xffffffffu, b, 2);
        c = __shfl_xor_sync(0xffffffffu, c, 4);
        d = __shfl_xor_sync(0xffffffffu, d, 8);
    }
    if (a + b + c + d == 1.2345f)
        out[threadIdx.x] = a;
}

__global__ void k_ldtm(float* out, int warps)
{
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)(32 * (warp % 4)) << 16) + 16 * ((warp / 4) % 8);
    uint32_t s = 0;
#pragma unroll 4
    for (int it = 0; it < ITERS / 4; ++it) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15])
            : "r"(base));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i)
            s += r[i];
    }
    if (s == 12345u)
        out[threadIdx.x] = s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <class K>
static void run(const char* name, K kern, int warps, size_t smem, double bytes_per_iter_per_warp)
{
    float* out;
    cudaMalloc(&out, 4096 * sizeof(float));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<148, warps * 32, smem>>>(out, warps);
    cudaEventRecord(e0);
    kern<<<148, warps * 32, smem>>>(out, warps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cycles = ms * 1e-3 * 1.965e9;
    const double per_sm = bytes_per_iter_per_warp * ITERS * warps / cycles;
    printf("%-28s warps/SM %2d  %.3f ms  %.1f B/clk/SM  (%s)\n", name, warps, ms, per_sm,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main()
{
    for (int w : {8, 16, 32}) {
        run("LDS.64 conflict-free", k_lds, w, 4096 * 8, 32 * 8);
        run("SHFL.32 (4 independent)", k_shfl, w, 0, 4 * 32 * 4);
        run("tcgen05.ld 32x32b.x16", k_ldtm, w, 0, 32 * 16 * 4 / 4.0);
    }
    return 0;
}
