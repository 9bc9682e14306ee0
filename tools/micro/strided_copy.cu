// Microbenchmark (not product code): HBM throughput of K1's access pattern
// without any FFT work. Tile = 512 rows x W complex64 columns at row stride
// `inner`; each tile is read once and written to two outputs (K1's 1R/2W).
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int TPR>  // TPR: threads per column
__global__ void copy_tiles(const float2* __restrict__ src, float2* __restrict__ d0,
                           float2* __restrict__ d1, long inner, long outer)
{
    const int w = threadIdx.x % W, t = threadIdx.x / W;
    const long cols = inner / W, ntiles = outer * cols;
    constexpr int R = 512 / TPR;
    for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
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

template <int W, int TPR>
void run(const char* name, float2* a, float2* b, float2* c, long inner, long total)
{
    const long outer = total / (512 * inner);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, copy_tiles<W, TPR>, W * TPR, 0);
    const int grid = 148 * per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i)
        copy_tiles<W, TPR><<<grid, W * TPR>>>(a, b, c, inner, outer);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i)
        copy_tiles<W, TPR><<<grid, W * TPR>>>(a, b, c, inner, outer);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s inner=%8ld W=%2d TPR=%3d grid=%5d  %.3f ms  %.0f GB/s\n", name, inner, W, TPR,
           grid, ms, 3.0 * total * 8 / (ms * 1e-3) / 1e9);
}

int main()
{
    const long total = 512L * 512 * 512;  // one component of C3
    float2 *a, *b, *c;
    cudaMalloc(&a, total * 8);
    cudaMalloc(&b, total * 8);
    cudaMalloc(&c, total * 8);
    cudaMemset(a, 0, total * 8);
    for (long inner : {512L * 512, 512L}) {
        run<8, 64>("W8 TPR64 (R8)", a, b, c, inner, total);
        run<16, 64>("W16 TPR64 (R8)", a, b, c, inner, total);
        run<16, 32>("W16 TPR32 (R16)", a, b, c, inner, total);
        run<32, 32>("W32 TPR32 (R16)", a, b, c, inner, total);
        run<32, 16>("W32 TPR16 (R32)", a, b, c, inner, total);
        run<8, 32>("W8 TPR32 (R16)", a, b, c, inner, total);
    }
    // plain streaming copy 1R2W for reference
    printf("done\n");
    return 0;
}
