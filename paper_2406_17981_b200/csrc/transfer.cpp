// ts_operator_apply with the reference ABI's host buffers (interleaved
// complex128 doubles, ref proj/src/capi/capi.cpp:97-115 marshalling +
// capi.cpp:259-285 apply). Caller memory is pageable, so every byte passes
// through pinned staging: T worker threads each own two pinned chunk slots
// and a copy stream; a worker converts chunk i of v to the operator precision
// straight into a pinned slot (complex64 operators halve the PCIe bytes:
// the c128 -> c64 rounding happens in the pass that pageable memory needs
// anyway) while the DMA of its previous chunk is in flight. The way back
// mirrors it: the D2H of chunk i overlaps the conversion of chunk i-T into
// the caller's y. The MVM itself runs on the operator's internal stream with
// its cached workspace (sched.cpp); apply_ns is its device time, excluding
// marshalling, as the reference's apply_ns excludes capi.cpp's sweeps
// (ref engine_split.cpp:119-131).
#include <cuda_runtime.h>

#include <immintrin.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "multi.hpp"

namespace tsb {

namespace {

constexpr size_t kChunkBytes = size_t(8) << 20;  // pinned bytes per slot

struct PinnedPool {
    std::mutex mu;
    std::vector<void*> free_;
    void* get()
    {
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!free_.empty()) {
                void* p = free_.back();
                free_.pop_back();
                return p;
            }
        }
        void* p = nullptr;
        cuda_check(cudaHostAlloc(&p, kChunkBytes, cudaHostAllocPortable), "cudaHostAlloc");
        return p;
    }
    void put(void* p)
    {
        std::lock_guard<std::mutex> lk(mu);
        free_.push_back(p);
    }
};

PinnedPool& pinned_pool()
{
    static PinnedPool* pool = new PinnedPool;  // process lifetime
    return *pool;
}

int transfer_threads(int64_t nchunks)
{
    static const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    // TSK_TRANSFER_THREADS overrides the worker count (A/B; default: host threads, at most 16)
    static const int cap = [] {
        const char* e = getenv("TSK_TRANSFER_THREADS");
        const int v = e ? atoi(e) : 0;
        return v > 0 ? std::min(v, 64) : 16;
    }();
    return static_cast<int>(std::clamp<int64_t>(std::min<int64_t>(nchunks, std::max(hw, cap > 16 ? cap : 0)), 1, cap));
}

// interleaved complex128 <-> operator precision, elements [0, n). The AVX2
// paths convert 4 reals per instruction and write with non-temporal stores
// (no read-for-ownership of the destination: the host passes are bound by
// host memory bandwidth, not arithmetic).
__attribute__((target("avx2"))) void c128_to_c64_avx2(const double* src, float* dst, int64_t nreal)
{
    int64_t i = 0;
    const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    for (; i + 4 <= nreal; i += 4) {
        const __m128 f = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i));
        if (aligned)
            _mm_stream_ps(dst + i, f);
        else
            _mm_storeu_ps(dst + i, f);
    }
    for (; i < nreal; ++i)
        dst[i] = static_cast<float>(src[i]);
    _mm_sfence();
}

__attribute__((target("avx2"))) void c64_to_c128_avx2(const float* src, double* dst, int64_t nreal)
{
    int64_t i = 0;
    // peel to a 32-byte aligned destination for the streaming stores
    for (; i < nreal && (reinterpret_cast<uintptr_t>(dst + i) & 31) != 0; ++i)
        dst[i] = static_cast<double>(src[i]);
    for (; i + 4 <= nreal; i += 4)
        _mm256_stream_pd(dst + i, _mm256_cvtps_pd(_mm_loadu_ps(src + i)));
    for (; i < nreal; ++i)
        dst[i] = static_cast<double>(src[i]);
    _mm_sfence();
}

bool have_avx2()
{
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

void to_device_prec(const double* src, void* dst, bool c64, int64_t n)
{
    if (!c64) {
        std::memcpy(dst, src, static_cast<size_t>(n) * 16);
        return;
    }
    float* d = static_cast<float*>(dst);
    if (have_avx2()) {
        c128_to_c64_avx2(src, d, 2 * n);
        return;
    }
    for (int64_t i = 0; i < 2 * n; ++i)
        d[i] = static_cast<float>(src[i]);
}

void from_device_prec(const void* src, double* dst, bool c64, int64_t n)
{
    if (!c64) {
        std::memcpy(dst, src, static_cast<size_t>(n) * 16);
        return;
    }
    const float* s = static_cast<const float*>(src);
    if (have_avx2()) {
        c64_to_c128_avx2(s, dst, 2 * n);
        return;
    }
    for (int64_t i = 0; i < 2 * n; ++i)
        dst[i] = static_cast<double>(s[i]);
}

// dir 0: host v -> device x; dir 1: device y -> host y. count complex
// elements; es = device element bytes. Blocks until done.
void host_transfer(int dir, int device, double* host, void* dev, size_t es, int64_t count)
{
    const bool c64 = es == 8;
    const int64_t per = static_cast<int64_t>(kChunkBytes / es);  // elements per chunk
    const int64_t nchunks = (count + per - 1) / per;
    const int T = transfer_threads(nchunks);
    std::vector<std::string> err(T);
    auto worker = [&](int k) {
        cudaStream_t s = nullptr;
        void* pin[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        try {
            cuda_check(cudaSetDevice(device), "device");
            cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
            for (int b = 0; b < 2; ++b) {
                pin[b] = pinned_pool().get();
                cuda_check(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "event");
            }
            int64_t prev = -1;
            int pslot = 0, j = 0;
            for (int64_t i = k; i < nchunks; i += T, ++j) {
                const int slot = j & 1;
                const int64_t off = i * per;
                const int64_t n = std::min<int64_t>(per, count - off);
                const size_t db = static_cast<size_t>(n) * es;
                char* dp = static_cast<char*>(dev) + static_cast<size_t>(off) * es;
                if (dir == 0) {
                    if (j >= 2)
                        cuda_check(cudaEventSynchronize(ev[slot]), "event");
                    to_device_prec(host + 2 * off, pin[slot], c64, n);
                    cuda_check(cudaMemcpyAsync(dp, pin[slot], db, cudaMemcpyHostToDevice, s), "H2D");
                    cuda_check(cudaEventRecord(ev[slot], s), "event");
                } else {
                    cuda_check(cudaMemcpyAsync(pin[slot], dp, db, cudaMemcpyDeviceToHost, s), "D2H");
                    cuda_check(cudaEventRecord(ev[slot], s), "event");
                    if (prev >= 0) {  // convert the previous chunk while this one is in flight
                        cuda_check(cudaEventSynchronize(ev[pslot]), "event");
                        const int64_t po = prev * per;
                        from_device_prec(pin[pslot], host + 2 * po, c64, std::min<int64_t>(per, count - po));
                    }
                    prev = i;
                    pslot = slot;
                }
            }
            if (dir == 1 && prev >= 0) {
                cuda_check(cudaEventSynchronize(ev[pslot]), "event");
                const int64_t po = prev * per;
                from_device_prec(pin[pslot], host + 2 * po, c64, std::min<int64_t>(per, count - po));
            }
            cuda_check(cudaStreamSynchronize(s), "transfer sync");
        } catch (const std::exception& e) {
            err[k] = e.what();
        }
        if (s)
            cudaStreamSynchronize(s);
        for (int b = 0; b < 2; ++b) {
            if (pin[b])
                pinned_pool().put(pin[b]);
            if (ev[b])
                cudaEventDestroy(ev[b]);
        }
        if (s)
            cudaStreamDestroy(s);
    };
    if (T == 1) {
        worker(0);
    } else {
        std::vector<std::thread> th;
        for (int k = 0; k < T; ++k)
            th.emplace_back(worker, k);
        for (auto& t : th)
            t.join();
    }
    for (auto& e : err)
        if (!e.empty())
            fail(TS_ERR_RESOURCE, "host transfer: " + e);
}

}  // namespace

void apply_host(const DeviceOperator& op, const double* v, double* y, const ts_policy* policy,
                ts_metrics* metrics)
{
    if (!v || !y)
        fail(TS_ERR_INVALID_ARGUMENT, "null argument");
    if (policy && policy->task_budget < 1 && !op.is_embed)
        fail(TS_ERR_INVALID_ARGUMENT, "task budget must be >= 1");
    // (the policy selects host threads in the reference, ref engine_split.cpp:77-83;
    // every policy runs the same device schedule here, so results are
    // bit-identical across policies as the reference requires)
    DeviceGuard guard(op.device);
    CtxLease lease(op, nullptr, true, op.multi ? 0 : 1);
    ApplyCtx* c = lease.c;
    const size_t vb = op.vec_bytes();
    if (c->hx.bytes < vb) {
        c->hx.reset();
        c->hx = DevBuf(vb, MEM_STAGING);
    }
    if (c->hy.bytes < vb) {
        c->hy.reset();
        c->hy = DevBuf(vb, MEM_STAGING);
    }
    const int64_t count = op.s * op.m;
    // TSK_DEBUG_TRANSFER=1: host wall clock of the three phases to stderr
    static const bool dbg = [] {
        const char* e = getenv("TSK_DEBUG_TRANSFER");
        return e && e[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    host_transfer(0, op.device, const_cast<double*>(v), c->hx.p, op.es(), count);
    const auto t1 = clk::now();
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard()
        {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } eg{e0, e1};
    int64_t peak = 2;
    cuda_check(cudaEventRecord(e0, c->st), "event");
    if (op.multi)
        multi_apply_device(op, c->hx.p, c->hy.p, 1, c->st, nullptr);
    else if (op.is_embed)
        apply_embed(op, c->hx.p, c->hy.p, c->st, c->work.p);
    else
        peak = enqueue_apply(op, c, c->hx.p, c->hy.p, 1);
    cuda_check(cudaEventRecord(e1, c->st), "event");
    cuda_check(cudaStreamSynchronize(c->st), "apply sync");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    const auto t2 = clk::now();
    host_transfer(1, op.device, y, c->hy.p, op.es(), count);
    if (dbg) {
        const auto ms_of = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        fprintf(stderr, "ts_operator_apply: host->device %.1f ms, MVM %.1f ms, device->host %.1f ms (%.2f GB each way)\n",
                ms_of(t0, t1), ms_of(t1, t2), ms_of(t2, clk::now()),
                static_cast<double>(count) * static_cast<double>(op.es()) / 1e9);
    }
    if (metrics) {
        if (op.is_embed)
            embed_counters(op, metrics);
        else
            fill_counters(op, metrics, peak);
        metrics->apply_ns = static_cast<uint64_t>(static_cast<double>(ms) * 1e6);
    }
}

}  // namespace tsb
