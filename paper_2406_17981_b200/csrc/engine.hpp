// Internals shared by the device-engine translation units of libtoesplit:
// CUDA error mapping, the device-memory meter (the B200 counterpart of the
// reference's AllocationMeter, ref proj/src/core/tensor.hpp:21-33 /
// tensor.cpp:49-66, counting device bytes instead of host elements), device
// buffers, per-length twiddle tables, and the device operator with its
// per-stream apply contexts (cached workspace + CUDA graphs).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host.hpp"
#include "tsk_launch.h"

namespace tsb {

// ---------------------------------------------------------------- errors

void cuda_check(cudaError_t e, const char* what);
inline void launch_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

// Restores the caller's current device on scope exit; fails with
// TS_ERR_RESOURCE when no CUDA device exists (no CPU fallback).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// ---------------------------------------------------------------- meter

enum MemKind { MEM_SPECTRA = 0, MEM_TABLES = 1, MEM_WORK = 2, MEM_STAGING = 3, MEM_KINDS = 4 };

// Library-owned device bytes per device: live, high-water mark, live by kind.
void meter_add(int dev, MemKind k, uint64_t bytes);
void meter_sub(int dev, MemKind k, uint64_t bytes);
void meter_stats(int dev, ts_memory_stats* out);
void meter_reset_peak(int dev);

// cudaMalloc'd device buffer, metered under `kind` on the current device.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = -1;
    MemKind kind = MEM_WORK;
    DevBuf() = default;
    DevBuf(size_t n, MemKind k);
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { swap(o); }
    DevBuf& operator=(DevBuf&& o) noexcept
    {
        swap(o);
        return *this;
    }
    ~DevBuf() { reset(); }
    void reset();
    void swap(DevBuf& o) noexcept
    {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        std::swap(dev, o.dev);
        std::swap(kind, o.kind);
    }
};

// ---------------------------------------------------------------- tables

// ref kernel.cpp:17-21
inline int64_t stored_len_host(int64_t n, int odd) { return odd ? (n + 1) / 2 : n / 2 + 1; }

// Per-length device tables: roots exp(-2 pi i k/n) and phases exp(-i pi k/n),
// computed in double (octant-reduced) and rounded once for complex64.
struct AxisTables {
    int64_t n = 0;
    DevBuf roots, phase;
    std::vector<int32_t> rad;
};
std::shared_ptr<AxisTables> make_tables(int64_t n, int prec);

// ---------------------------------------------------------------- operator

struct DeviceOperator;

// One apply context per (operator, stream): the depth-first schedule's child
// buffers for up to `work_rhs` right-hand sides, kept across calls (no
// per-call allocation), and CUDA graphs of the launch sequence for small
// operators keyed by (x, y, nrhs). Contexts are used by one host thread at a
// time (`busy`); the stream orders the device work of successive calls.
struct ApplyCtx {
    int dev = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;  // internal stream of the host-buffer ABI path
    bool busy = false;
    uint64_t lru = 0;
    DevBuf work;
    int64_t work_rhs = 0;
    DevBuf hx, hy;  // device x / y of the host-buffer path
    struct Graph {
        const void* x = nullptr;
        void* y = nullptr;
        int64_t nrhs = 0;
        cudaGraphExec_t exec = nullptr;
        int64_t peak_children = 0;
        uint64_t lru = 0;
    } graph[2];
    uint64_t graph_tick = 0;
    uint64_t graph_replays = 0;
    ~ApplyCtx();
};

struct DeviceOperator {
    int device = 0;
    Shape levels;
    int d = 0;
    int64_t s = 0;
    int m = 1, n_unique = 1;
    std::vector<int> comp_map;
    std::vector<uint32_t> skew_mask;  // per unique component
    std::vector<int> axis_sign;       // per unique component x axis
    int prec = 0;                     // 0 c128, 1 c64
    bool compressed = false;
    int part = 0, nparts = 1, q = 0;
    int tskf_symmetry = 0;  // symmetry byte for version-1 files, 255 = mixed
    DevBuf spectra;
    uint64_t spectra_elems = 0;  // complex elements stored on this device
    std::vector<int64_t> branch_base, block_elems;
    std::vector<std::shared_ptr<AxisTables>> tab;  // per axis
    uint64_t precompute_ns = 0;
    // full-embedding baseline operator
    bool is_embed = false;
    bool embed_corner = false, embed_skew = false;
    DevBuf symbol;
    std::vector<std::shared_ptr<AxisTables>> tab2;  // per axis, length 2n
    // several GPUs (multi.cpp): parts, communicators, streams
    std::shared_ptr<struct MultiGpu> multi;
    // apply contexts
    mutable std::mutex ctx_mu;
    mutable std::vector<std::unique_ptr<ApplyCtx>> ctxs;
    mutable uint64_t tick = 0;

    size_t es() const { return prec ? 8 : 16; }
    size_t vec_bytes() const { return static_cast<size_t>(s) * m * es(); }
    bool owns(uint32_t b) const
    {
        return (b & static_cast<uint32_t>(nparts - 1)) == static_cast<uint32_t>(part);
    }
    uint64_t table_bytes() const;
    uint64_t cached_bytes() const;
};

void fill_tables(DeviceOperator& op, const Shape& lens, std::vector<std::shared_ptr<AxisTables>>& out);
tsk_axis axis_desc(const Shape& shape, const std::vector<std::shared_ptr<AxisTables>>& tabs, int axis,
                   int ncomp, int64_t cstride, int prec);

// Borrow / return an apply context for `stream` (nullptr with own = true: an
// internal stream). Workspace is (re)sized for nrhs right-hand sides.
ApplyCtx* acquire_ctx(const DeviceOperator& op, cudaStream_t stream, bool own, int64_t nrhs);
void release_ctx(const DeviceOperator& op, ApplyCtx* c);
struct CtxLease {
    const DeviceOperator& op;
    ApplyCtx* c;
    CtxLease(const DeviceOperator& o, cudaStream_t st, bool own, int64_t nrhs)
        : op(o), c(acquire_ctx(o, st, own, nrhs))
    {
    }
    ~CtxLease() { release_ctx(op, c); }
    CtxLease(const CtxLease&) = delete;
    CtxLease& operator=(const CtxLease&) = delete;
};

// Enqueue one (batched) MVM on ctx->st; returns the peak number of vector
// buffers (x, y and child buffers, in units of nrhs*m*s elements) that the
// schedule holds at once — the measured counterpart of the reference's
// peak_live_elems / (m s).
int64_t enqueue_apply(const DeviceOperator& op, ApplyCtx* ctx, const void* x, void* y, int64_t nrhs,
                      std::vector<ts_launch_record>* rec = nullptr);
// As enqueue_apply (no graph), with the root-level inverse pass split per
// component vector and hook(c) called after component c is enqueued.
int64_t enqueue_apply_hooked(const DeviceOperator& op, ApplyCtx* ctx, const void* x, void* y,
                             int64_t nrhs, const std::function<void(int64_t)>& hook);
// work: m (2n)^d elements of the operator precision (the apply context's)
void apply_embed(const DeviceOperator& op, const void* x, void* y, cudaStream_t st, void* work);
void embed_counters(const DeviceOperator& op, ts_metrics* m);
void fill_counters(const DeviceOperator& op, ts_metrics* m, int64_t peak_vectors);
uint64_t count_launches(int d, int q);

}  // namespace tsb
