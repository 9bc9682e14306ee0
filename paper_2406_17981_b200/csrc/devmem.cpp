// CUDA error mapping, device guard and the device-memory meter of libtoesplit.
// The meter is the B200 counterpart of the reference's AllocationMeter (ref
// proj/src/core/tensor.cpp:49-66: atomic live counter + CAS-maintained peak),
// kept per device in bytes and by kind (spectra / tables / workspace /
// staging) for every device buffer the library allocates.
#include <cuda_runtime.h>

#include <algorithm>

#include "engine.hpp"

namespace tsb {

void cuda_check(cudaError_t e, const char* what)
{
    if (e == cudaSuccess)
        return;
    cudaGetLastError();  // clear non-sticky errors
    const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation)
        fail(TS_ERR_RESOURCE, "device out of memory (" + msg + ")");
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorInvalidDevice)
        fail(TS_ERR_RESOURCE, "no usable CUDA device (" + msg + ")");
    fail(TS_ERR_INTERNAL, msg);
}

int32_t device_count()
{
    static const int n = [] {
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        return c;
    }();
    return n;
}

DeviceGuard::DeviceGuard(int dev)
{
    if (device_count() == 0)
        fail(TS_ERR_RESOURCE, "no CUDA device: the split engine runs on the GPU only");
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    if (dev >= 0 && dev != prev)
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    else
        prev = -1;  // nothing to restore
}

DeviceGuard::~DeviceGuard()
{
    if (prev >= 0)
        cudaSetDevice(prev);
}

// ---------------------------------------------------------------- meter

namespace {

constexpr int kMaxDev = 64;

struct Meter {
    std::atomic<uint64_t> live{0}, peak{0};
    std::atomic<uint64_t> kind[MEM_KINDS] = {};
};

Meter& meter(int dev)
{
    static Meter* m = new Meter[kMaxDev];  // process lifetime
    return m[std::clamp(dev, 0, kMaxDev - 1)];
}

}  // namespace

void meter_add(int dev, MemKind k, uint64_t bytes)
{
    Meter& mt = meter(dev);
    mt.kind[k].fetch_add(bytes, std::memory_order_relaxed);
    const uint64_t now = mt.live.fetch_add(bytes, std::memory_order_relaxed) + bytes;
    uint64_t prev = mt.peak.load(std::memory_order_relaxed);
    while (prev < now && !mt.peak.compare_exchange_weak(prev, now, std::memory_order_relaxed)) {
    }
}

void meter_sub(int dev, MemKind k, uint64_t bytes)
{
    Meter& mt = meter(dev);
    mt.kind[k].fetch_sub(bytes, std::memory_order_relaxed);
    mt.live.fetch_sub(bytes, std::memory_order_relaxed);
}

void meter_stats(int dev, ts_memory_stats* out)
{
    Meter& mt = meter(dev);
    ts_memory_stats r{};
    r.live_bytes = mt.live.load();
    r.peak_bytes = mt.peak.load();
    r.spectra_bytes = mt.kind[MEM_SPECTRA].load();
    r.table_bytes = mt.kind[MEM_TABLES].load();
    r.workspace_bytes = mt.kind[MEM_WORK].load();
    r.staging_bytes = mt.kind[MEM_STAGING].load();
    *out = r;
}

void meter_reset_peak(int dev)
{
    Meter& mt = meter(dev);
    mt.peak.store(mt.live.load());
}

// ---------------------------------------------------------------- DevBuf

DevBuf::DevBuf(size_t n, MemKind k) : bytes(n), kind(k)
{
    if (!n)
        return;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaMalloc(&p, n), "cudaMalloc");
    meter_add(dev, kind, bytes);
}

void DevBuf::reset()
{
    if (p) {
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != dev)
            cudaSetDevice(dev);
        cudaFree(p);
        if (cur != dev && cur >= 0)
            cudaSetDevice(cur);
        meter_sub(dev, kind, bytes);
    }
    p = nullptr;
    bytes = 0;
}

}  // namespace tsb
