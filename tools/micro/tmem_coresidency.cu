// Microbenchmark (not product code): how many tcgen05 (TMEM-allocating) CTAs the
// B200 co-schedules per SM for a given column count, measured from %smid and
// %globaltimer intervals (the occupancy API reports 1 for any tcgen05 kernel).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <int COLS>
__global__ void __launch_bounds__(384, 1) k_tmem(unsigned long long* rec)
{
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "n"(COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint64_t t0 = gtime();
    while (gtime() - t0 < 200000) {}
    uint64_t t1 = gtime();
    uint32_t smid; asm("mov.u32 %0, %smid;" : "=r"(smid));
    if (threadIdx.x == 0) { rec[3 * blockIdx.x] = smid; rec[3 * blockIdx.x + 1] = t0; rec[3 * blockIdx.x + 2] = t1; }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(COLS));
}
template <int COLS>
void run(int grid)
{
    unsigned long long* d; cudaMalloc(&d, 3 * grid * 8);
    k_tmem<COLS><<<grid, 384>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(3 * grid);
    cudaMemcpy(h.data(), d, 3 * grid * 8, cudaMemcpyDeviceToHost);
    uint64_t tmin = ~0ull, tmax = 0;
    for (int i = 0; i < grid; ++i) { tmin = std::min<uint64_t>(tmin, h[3*i+1]); tmax = std::max<uint64_t>(tmax, h[3*i+2]); }
    // max concurrent CTAs on any SM
    int maxc = 0;
    for (int i = 0; i < grid; ++i) {
        int c = 0;
        for (int j = 0; j < grid; ++j)
            if (h[3*j] == h[3*i] && h[3*j+1] <= h[3*i+1] && h[3*i+1] < h[3*j+2]) ++c;
        maxc = std::max(maxc, c);
    }
    printf("cols %d grid %d: %s, span %.0f us (one CTA = 200 us), max co-resident CTAs per SM %d\n", COLS, grid,
           cudaGetErrorString(e), (tmax - tmin) / 1e3, maxc);
    cudaFree(d);
}
int main()
{
    run<256>(148); run<256>(296); run<128>(444); run<512>(296);
    return 0;
}
