// Tensor memory as thread-private storage (sm_100a tcgen05, 32x32b shape):
// warp w of a CTA reaches TMEM lanes 32*(w%4) .. +31, thread i its own lane;
// warps sharing a lane quadrant use disjoint column ranges. Used to park a
// thread's values across a phase that needs the registers (no shared-memory
// bandwidth spent, unlike a shared-memory stash).
#pragma once

#include <stdint.h>

#include <algorithm>

#include "tsk_common.cuh"

namespace tsk {

// 32-bit words of a complex value, by member access (a reinterpret_cast of a
// register array's address would force the array into local memory)
template <typename T2>
struct Words;
template <>
struct Words<float2> {
    static constexpr int W = 2;
    __device__ __forceinline__ static uint32_t get(const float2& v, int j)
    {
        return __float_as_uint(j == 0 ? v.x : v.y);
    }
    __device__ __forceinline__ static float2 make(const uint32_t* r)
    {
        return make_float2(__uint_as_float(r[0]), __uint_as_float(r[1]));
    }
};
template <>
struct Words<double2> {
    static constexpr int W = 4;
    __device__ __forceinline__ static uint32_t get(const double2& v, int j)
    {
        const double d = j < 2 ? v.x : v.y;
        return (uint32_t)((j & 1) ? __double2hiint(d) : __double2loint(d));
    }
    __device__ __forceinline__ static double2 make(const uint32_t* r)
    {
        return make_double2(__hiloint2double((int)r[1], (int)r[0]),
                            __hiloint2double((int)r[3], (int)r[2]));
    }
};


__device__ __forceinline__ uint32_t tmem_alloc(uint32_t* slot, int cols)
{
    // one warp allocates; the base address lands in shared memory
    if (threadIdx.x < 32) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa),
                     "r"(cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    return *slot;
}

__device__ __forceinline__ void tmem_free(uint32_t base, int cols)
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols)
                     : "memory");
}

// Store / load 32 consecutive 32-bit columns of this thread's lane.
__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31, %32};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Park / restore R complex values (2 or 4 words each) in this thread's lane.
// WAIT = false leaves the stores in flight: the caller issues tmem_wait_st()
// (or any later tcgen05.wait::st) before the values are read back.
template <typename T, int R, bool WAIT = true>
__device__ __forceinline__ void tmem_park(uint32_t lane_base, const typename cx<T>::t (&v)[R])
{
    constexpr int WORDS = R * (int)sizeof(typename cx<T>::t) / 4;
    static_assert(WORDS % 32 == 0, "park granularity is 32 words");
#pragma unroll
    for (int c = 0; c < WORDS / 32; ++c) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
            r[i] = Words<typename cx<T>::t>::get(v[(c * 32 + i) / Words<typename cx<T>::t>::W],
                                                 (c * 32 + i) % Words<typename cx<T>::t>::W);
        tmem_st32(lane_base + c * 32, r);
    }
    if constexpr (WAIT)
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <typename T, int R>
__device__ __forceinline__ void tmem_restore(uint32_t lane_base, typename cx<T>::t (&v)[R])
{
    constexpr int WORDS = R * (int)sizeof(typename cx<T>::t) / 4;
#pragma unroll
    for (int c = 0; c < WORDS / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(lane_base + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; i += Words<typename cx<T>::t>::W)
            v[(c * 32 + i) / Words<typename cx<T>::t>::W] = Words<typename cx<T>::t>::make(r + i);
    }
}


__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(addr)
        : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(addr)
                 : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Park / restore 8 complex values (16 or 32 words) at column offset col.
template <typename T2>
__device__ __forceinline__ void tmem_put8(uint32_t lane_base, int col, const T2 (&v)[8])
{
    constexpr int WORDS = 8 * (int)sizeof(T2) / 4;
#pragma unroll
    for (int c = 0; c < WORDS / 16; ++c) {
        uint32_t r[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            r[i] = Words<T2>::get(v[(c * 16 + i) / Words<T2>::W], (c * 16 + i) % Words<T2>::W);
        tmem_st16(lane_base + col + c * 16, r);
    }
}

template <typename T2>
__device__ __forceinline__ void tmem_get8(uint32_t lane_base, int col, T2 (&v)[8])
{
    constexpr int WORDS = 8 * (int)sizeof(T2) / 4;
#pragma unroll
    for (int c = 0; c < WORDS / 16; ++c) {
        uint32_t r[16];
        tmem_ld16(lane_base + col + c * 16, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += Words<T2>::W)
            v[(c * 16 + i) / Words<T2>::W] = Words<T2>::make(r + i);
    }
}

constexpr int tmem_cols_pow2(int n)
{
    return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}

}  // namespace tsk

#ifdef __CUDACC__
namespace tsk {
// CTAs per SM for a kernel that allocates tcols TMEM columns per CTA. The
// occupancy API reports one CTA per SM for every tcgen05 kernel; measured on
// B200 (tools/micro/tmem_coresidency.cu) the hardware co-schedules CTAs whose
// allocations sum to <= 512 columns, so the limit is computed from registers,
// shared memory, threads and TMEM columns directly.
template <class K>
static int tmem_occupancy(K kern, int nt, size_t dsmem, int tcols)
{
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess)
        return 1;
    int dev = 0, regs_sm = 65536, smem_sm = 233472, thr_sm = 2048, resv = 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    const int warps = (nt + 31) / 32;
    const int rpw = ((fa.numRegs * 32 + 255) / 256) * 256;  // registers per warp, allocation unit 256
    int n = regs_sm / (rpw * warps);
    n = std::min(n, smem_sm / (int)(dsmem + fa.sharedSizeBytes + resv));
    n = std::min(n, thr_sm / (warps * 32));
    if (tcols > 0)
        n = std::min(n, 512 / tcols);
    return n > 0 ? n : 1;
}
}  // namespace tsk
#endif
