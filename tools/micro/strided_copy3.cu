// Microbenchmark (not product code): the K1 access pattern (one 512-row
// strided tile in, two tiles out, optional re-read of the input between the
// two stores) with the K1 thread geometry, no arithmetic: the memory ceiling
// the fused forward-split pass can reach per tile width / CTAs per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int TPR, bool RELOAD>
__global__ void k1_pattern(const float2* __restrict__ src, float2* __restrict__ d0,
                           float2* __restrict__ d1, long inner, long outer)
{
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const long cols = inner / W, ntiles = outer * cols;
    constexpr int R = 512 / TPR;
    for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long o = tile / cols, i0 = (tile % cols) * W;
        const long base = o * 512 * inner + i0 + w;
        float2 v[R];
        const long rs = (long)TPR * inner;
        const float2* ps = src + base + (long)t * inner;
        float2* p0 = d0 + base + (long)t * inner;
        float2* p1 = d1 + base + (long)t * inner;
#pragma unroll
        for (int m = 0; m < R; ++m)
            v[m] = ps[m * rs];
#pragma unroll
        for (int m = 0; m < R; ++m)
            p1[m * rs] = make_float2(v[m].y, v[m].x);
        if (RELOAD) {
#pragma unroll
            for (int m = 0; m < R; ++m)
                v[m] = ps[m * rs];
        }
#pragma unroll
        for (int m = 0; m < R; ++m)
            p0[m * rs] = v[m];
    }
}

template <int W, int TPR, bool RELOAD>
void run(const char* name, float2* a, float2* b, float2* c, long inner, long total, int cps)
{
    const long outer = total / (512 * inner);
    auto k = k1_pattern<W, TPR, RELOAD>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, W * TPR, 0);
    if (cps && cps < per_sm)
        per_sm = cps;
    const int grid = 148 * per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i)
        k<<<grid, W * TPR>>>(a, b, c, inner, outer);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i)
        k<<<grid, W * TPR>>>(a, b, c, inner, outer);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-34s inner=%7ld cta/sm=%d  %.3f ms  %.0f GB/s (3 vectors)\n", name, inner, per_sm, ms,
           3.0 * total * 8 / (ms * 1e-3) / 1e9);
}

int main()
{
    const long total = 512L * 512 * 512;
    float2 *a, *b, *c;
    cudaMalloc(&a, total * 8);
    cudaMalloc(&b, total * 8);
    cudaMalloc(&c, total * 8);
    cudaMemset(a, 0, total * 8);
    for (long inner : {262144L, 512L}) {
        run<16, 16, true>("W16 R32 reload 2cta/sm (K1 now)", a, b, c, inner, total, 2);
        run<16, 16, false>("W16 R32 noreload 2cta/sm", a, b, c, inner, total, 2);
        run<16, 16, true>("W16 R32 reload 4cta/sm", a, b, c, inner, total, 4);
        run<32, 16, true>("W32 R32 reload 1cta/sm", a, b, c, inner, total, 1);
        run<32, 16, true>("W32 R32 reload 2cta/sm", a, b, c, inner, total, 2);
        run<32, 16, false>("W32 R32 noreload 2cta/sm", a, b, c, inner, total, 2);
        run<32, 32, true>("W32 R16 reload 2cta/sm", a, b, c, inner, total, 2);
    }
    return 0;
}
