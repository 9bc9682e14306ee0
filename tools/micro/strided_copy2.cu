// Microbenchmark (not product code): which tile geometries/orders recover
// HBM bandwidth for 512-row strided tiles (K1/K3 access pattern).
#include <cstdio>
#include <cuda_runtime.h>

// BLK consecutive column tiles per CTA visit (blocked assignment)
template <int W, int TPR, int BLK>
__global__ void copy_tiles(const float2* __restrict__ src, float2* __restrict__ d0,
                           float2* __restrict__ d1, long inner, long outer)
{
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const long cols = inner / W, ntiles = outer * cols;
    constexpr int R = 512 / TPR;
    for (long blk = blockIdx.x; blk * BLK < ntiles; blk += gridDim.x)
        for (int b = 0; b < BLK; ++b) {
            const long tile = blk * BLK + b;
            if (tile >= ntiles) break;
            const long o = tile / cols, i0 = (tile % cols) * W;
            const long base = o * 512 * inner + i0 + w;
            float2 v[R];
#pragma unroll
            for (int m = 0; m < R; ++m)
                v[m] = src[base + (long)(t + m * TPR) * inner];
#pragma unroll
            for (int m = 0; m < R; ++m) {
                d0[base + (long)(t + m * TPR) * inner] = v[m];
                d1[base + (long)(t + m * TPR) * inner] = make_float2(v[m].y, v[m].x);
            }
        }
}

template <int W, int TPR, int BLK>
void run(const char* name, float2* a, float2* b, float2* c, long inner, long total, int cps = 0)
{
    const long outer = total / (512 * inner);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, copy_tiles<W, TPR, BLK>, W * TPR, 0);
    if (cps) per_sm = cps < per_sm ? cps : per_sm;
    const int grid = 148 * per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i)
        copy_tiles<W, TPR, BLK><<<grid, W * TPR>>>(a, b, c, inner, outer);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i)
        copy_tiles<W, TPR, BLK><<<grid, W * TPR>>>(a, b, c, inner, outer);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-26s inner=%7ld grid=%5d  %.3f ms  %.0f GB/s\n", name, inner, grid, ms,
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
    for (long inner : {262144L, 32768L, 4096L, 512L}) {
        run<8, 64, 1>("W8  R8  blk1", a, b, c, inner, total);
        run<8, 64, 4>("W8  R8  blk4", a, b, c, inner, total);
        run<8, 64, 16>("W8  R8  blk16", a, b, c, inner, total);
        run<8, 64, 1>("W8  R8  blk1 1cta/sm", a, b, c, inner, total, 1);
        run<16, 64, 1>("W16 R8  blk1", a, b, c, inner, total);
        run<16, 64, 4>("W16 R8  blk4", a, b, c, inner, total);
        run<32, 32, 1>("W32 R16 blk1", a, b, c, inner, total);
        run<32, 16, 1>("W32 R32 blk1 1cta/sm", a, b, c, inner, total, 1);
    }
    return 0;
}
