// The depth-first branch scheduler (the reference's `branch` recursion, ref
// proj/src/core/engine_split.cpp:61-135, as a launch sequence of the fused
// K1 / K2 / K3 passes) and the device-buffer apply paths of libtoesplit:
// single and multi-RHS applies, per-launch profiling, per-stream apply
// contexts that keep the child buffers across calls and replay small
// operators' launch sequences as CUDA graphs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <functional>

#include "engine.hpp"
#include "multi.hpp"

namespace tsb {

// ---------------------------------------------------------------- contexts

ApplyCtx::~ApplyCtx()
{
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != dev)
        cudaSetDevice(dev);
    for (auto& g : graph)
        if (g.exec)
            cudaGraphExecDestroy(g.exec);
    if (own_stream && st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    work.reset();
    hx.reset();
    hy.reset();
    if (cur != dev && cur >= 0)
        cudaSetDevice(cur);
}

uint64_t DeviceOperator::cached_bytes() const
{
    std::lock_guard<std::mutex> lk(ctx_mu);
    uint64_t b = 0;
    for (const auto& c : ctxs)
        b += c->work.bytes + c->hx.bytes + c->hy.bytes;
    return b;
}

static size_t work_bytes(const DeviceOperator& op, int64_t nrhs)
{
    if (op.is_embed)  // the (2n)^d padded copies of the m components
        return static_cast<size_t>(op.s) * op.m * op.es() << op.d;
    const int nchild = std::max(0, op.d - 1 - op.q);
    return op.vec_bytes() * static_cast<size_t>(nrhs) * static_cast<size_t>(nchild);
}

// Contexts kept per operator: at most kMaxCtx, and at most two holding a
// workspace of 1 GB or more (C3: 6.4 GB each); the least recently used idle
// context is evicted (cudaFree waits for its stream's work).
static constexpr size_t kMaxCtx = 8;

ApplyCtx* acquire_ctx(const DeviceOperator& op, cudaStream_t stream, bool own, int64_t nrhs)
{
    const size_t need = op.multi || nrhs < 1 ? 0 : work_bytes(op, op.is_embed ? 1 : nrhs);
    std::unique_ptr<ApplyCtx> fresh;
    ApplyCtx* c = nullptr;
    {
        std::lock_guard<std::mutex> lk(op.ctx_mu);
        for (auto& p : op.ctxs)
            if (!p->busy && p->own_stream == own && (own || p->st == stream)) {
                c = p.get();
                break;
            }
        if (c) {
            c->busy = true;
            c->lru = ++op.tick;
        }
    }
    if (!c) {
        fresh = std::make_unique<ApplyCtx>();
        c = fresh.get();
        c->dev = op.device;
        c->busy = true;
        if (own) {
            cuda_check(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "stream");
            c->own_stream = true;
        } else {
            c->st = stream;
        }
    }
    if (c->work.bytes < need) {
        try {
            c->work.reset();
            c->work = DevBuf(need, MEM_WORK);
            c->work_rhs = nrhs;
            for (auto& g : c->graph)  // captured against the old buffer
                if (g.exec) {
                    cudaGraphExecDestroy(g.exec);
                    g = ApplyCtx::Graph{};
                }
        } catch (...) {
            if (!fresh) {
                std::lock_guard<std::mutex> lk(op.ctx_mu);
                c->busy = false;
            }
            throw;
        }
    }
    if (fresh) {
        std::lock_guard<std::mutex> lk(op.ctx_mu);
        c->lru = ++op.tick;
        op.ctxs.push_back(std::move(fresh));
        // evict idle contexts beyond the bounds (LRU first)
        for (;;) {
            size_t big = 0;
            for (auto& p : op.ctxs)
                big += p->work.bytes >= (size_t(1) << 30);
            if (op.ctxs.size() <= kMaxCtx && big <= 2)
                break;
            ApplyCtx* victim = nullptr;
            for (auto& p : op.ctxs)
                if (!p->busy && (!victim || p->lru < victim->lru))
                    victim = p.get();
            if (!victim)
                break;
            op.ctxs.erase(std::find_if(op.ctxs.begin(), op.ctxs.end(),
                                       [victim](auto& p) { return p.get() == victim; }));
        }
    }
    return c;
}

void release_ctx(const DeviceOperator& op, ApplyCtx* c)
{
    if (!c)
        return;
    std::lock_guard<std::mutex> lk(op.ctx_mu);
    c->busy = false;
}

// ---------------------------------------------------------------- scheduler

namespace {

struct Sched {
    const DeviceOperator& op;
    cudaStream_t st;
    int64_t nrhs = 1;
    std::vector<void*> buf;  // child buffer per depth (index q+1..d-1)
    int launches = 0;
    int64_t live = 2, peak = 2;  // vectors held: x, y, children
    // profiling: an event pair around every launch when rec != nullptr
    std::vector<ts_launch_record>* rec = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* ev = nullptr;
    // multi-GPU: the root-level inverse pass is split per component vector
    // and root_hook(c) runs after component c is enqueued
    std::function<void(int64_t)> root_hook;

    uint64_t unit() const { return static_cast<uint64_t>(op.vec_bytes()) * static_cast<uint64_t>(nrhs); }

    void before()
    {
        if (!rec)
            return;
        cudaEvent_t a, b;
        cuda_check(cudaEventCreate(&a), "event");
        cuda_check(cudaEventCreate(&b), "event");
        cuda_check(cudaEventRecord(a, st), "event");
        ev->emplace_back(a, b);
    }
    void after(int kind, int axis, int single, uint64_t bytes)
    {
        ++launches;
        if (!rec)
            return;
        cuda_check(cudaEventRecord(ev->back().second, st), "event");
        ts_launch_record r{};
        r.kind = kind;
        r.axis = axis;
        r.single_child = single;
        r.alg_bytes = bytes;
        rec->push_back(r);
    }

    // K1 / K3 treat the nrhs * m component tensors (s elements apart) as one batch
    tsk_axis ax(int axis) const
    {
        return axis_desc(op.levels, op.tab, axis, static_cast<int>(op.m * nrhs), op.s, op.prec);
    }

    void leaf(uint32_t b, const void* in, void* out, int use_even, int use_odd)
    {
        const int a = op.d - 1;
        tsk_axis x = axis_desc(op.levels, op.tab, a, op.m, op.s, op.prec);
        x.nrhs = nrhs;
        x.rstride = op.s * op.m;
        x.src0 = in;
        x.dst0 = out;
        x.use_even = use_even;
        x.use_odd = use_odd;
        x.scale = 0.5 / static_cast<double>(op.levels[a]);
        tsk_spectra sp{};
        sp.data = op.spectra.p;
        const uint32_t be = b, bo = b | (1u << a);
        sp.branch_base[0] = op.branch_base[be];
        sp.branch_base[1] = op.branch_base[bo];
        sp.block_elems[0] = op.block_elems[be];
        sp.block_elems[1] = op.block_elems[bo];
        sp.branch_bits[0] = be;
        sp.branch_bits[1] = bo;
        sp.compressed = op.compressed ? 1 : 0;
        sp.d = op.d;
        sp.m = op.m;
        sp.n_unique = op.n_unique;
        for (int i = 0; i < op.d; ++i)
            sp.levels[i] = op.levels[i];
        for (int u = 0; u < op.n_unique; ++u)
            sp.skew_mask[u] = op.skew_mask[u];
        for (int i = 0; i < op.m * op.m; ++i)
            sp.comp_map[i] = static_cast<int8_t>(op.comp_map[i]);
        before();
        launch_check(tsk_leaf_pair(&x, &sp, st), "leaf pair");
        // spectra are read once per launch whatever nrhs (SURVEY.md §8(d) K_bytes)
        const uint64_t spec = static_cast<uint64_t>(op.n_unique) * op.es() *
                              ((use_even ? op.block_elems[be] : 0) + (use_odd ? op.block_elems[bo] : 0));
        after(2, a, !(use_even && use_odd), 2 * unit() + spec);
    }

    void inverse(int delta, tsk_axis iv, int single, uint64_t bytes)
    {
        if (delta == 0 && root_hook) {
            const int64_t nc = op.m * nrhs;
            const size_t cb = static_cast<size_t>(op.s) * op.es();
            for (int64_t c = 0; c < nc; ++c) {
                tsk_axis one = iv;
                one.ncomp = 1;
                one.src0 = static_cast<const char*>(iv.src0) + c * cb;
                one.src1 = static_cast<const char*>(iv.src1) + c * cb;
                one.dst0 = static_cast<char*>(iv.dst0) + c * cb;
                before();
                launch_check(tsk_inv_merge(&one, st), single ? "inv merge'" : "inv merge");
                after(3, delta, single, bytes / static_cast<uint64_t>(nc));
                root_hook(c);
            }
            return;
        }
        before();
        launch_check(tsk_inv_merge(&iv, st), single ? "inv merge'" : "inv merge");
        after(3, delta, single, bytes);
    }

    // Node at depth delta holds data transformed along axes < delta.
    void solve(int delta, uint32_t b, const void* in, void* out)
    {
        const int d = op.d;
        if (delta == d - 1) {
            if (delta < op.q) {
                const int odd = (op.part >> delta) & 1;
                leaf(b, in, out, !odd, odd);
            } else {
                leaf(b, in, out, 1, 1);
            }
            if (delta == 0 && root_hook)  // d = 1: the leaf pass is the root level
                for (int64_t c = 0; c < op.m * nrhs; ++c)
                    root_hook(c);
            return;
        }
        if (delta < op.q) {
            // single-child path level (K1' / K3')
            const int odd = (op.part >> delta) & 1;
            tsk_axis f = ax(delta);
            f.src0 = in;
            f.dst0 = out;
            f.dst1 = out;
            f.use_even = !odd;
            f.use_odd = odd;
            before();
            launch_check(tsk_fwd_split(&f, st), "fwd split'");
            after(1, delta, 1, 2 * unit());
            solve(delta + 1, odd ? b | (1u << delta) : b, out, out);
            tsk_axis iv = ax(delta);
            iv.src0 = out;
            iv.src1 = out;
            iv.dst0 = out;
            iv.use_even = !odd;
            iv.use_odd = odd;
            iv.scale = 0.5 / static_cast<double>(op.levels[delta]);
            inverse(delta, iv, 1, 2 * unit());
            return;
        }
        void* child = buf[delta + 1];
        tsk_axis f = ax(delta);
        f.src0 = in;
        f.dst0 = out;
        f.dst1 = child;
        peak = std::max(peak, ++live);
        before();
        launch_check(tsk_fwd_split(&f, st), "fwd split");
        after(1, delta, 0, 3 * unit());
        solve(delta + 1, b, out, out);
        solve(delta + 1, b | (1u << delta), child, child);
        tsk_axis iv = ax(delta);
        iv.src0 = out;
        iv.src1 = child;
        iv.dst0 = out;
        iv.scale = 0.5 / static_cast<double>(op.levels[delta]);
        inverse(delta, iv, 0, 3 * unit());
        --live;
    }
};

bool env_flag(const char* name)
{
    const char* e = getenv(name);
    return e && e[0] == '1';
}

// Graph replay pays off where launch latency is a visible share of the MVM;
// long axes (global-memory passes with their own stream-ordered scratch) are
// launched directly.
bool graph_eligible(const DeviceOperator& op, int64_t nrhs)
{
    static const bool off = env_flag("TSK_NO_GRAPH");
    if (off || op.is_embed)
        return false;
    if (op.vec_bytes() * static_cast<size_t>(nrhs) > (size_t(64) << 20))
        return false;
    for (auto n : op.levels)
        if (n > 4096)
            return false;
    return true;
}

int64_t run_sched(const DeviceOperator& op, cudaStream_t st, void* work, const void* x, void* y,
                  int64_t nrhs, std::vector<ts_launch_record>* rec,
                  std::function<void(int64_t)> hook = {})
{
    const size_t vbytes = op.vec_bytes() * static_cast<size_t>(nrhs);
    const int nchild = std::max(0, op.d - 1 - op.q);
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    Sched sc{op, st, nrhs, std::vector<void*>(op.d + 1, nullptr)};
    sc.rec = rec;
    sc.ev = &ev;
    sc.root_hook = std::move(hook);
    for (int i = 0; i < nchild; ++i)
        sc.buf[op.q + 1 + i] = static_cast<char*>(work) + vbytes * i;
    sc.solve(0, 0, x, y);
    if (rec) {
        cuda_check(cudaStreamSynchronize(st), "profile sync");
        for (size_t i = 0; i < ev.size(); ++i) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, ev[i].first, ev[i].second), "elapsed");
            (*rec)[i].ms = ms;
            cudaEventDestroy(ev[i].first);
            cudaEventDestroy(ev[i].second);
        }
    }
    return sc.peak;
}

}  // namespace

int64_t enqueue_apply(const DeviceOperator& op, ApplyCtx* ctx, const void* x, void* y, int64_t nrhs,
                      std::vector<ts_launch_record>* rec)
{
    if (rec || !graph_eligible(op, nrhs))
        return run_sched(op, ctx->st, ctx->work.p, x, y, nrhs, rec);
    // graph replay keyed by (x, y, nrhs); the first sight of a key runs
    // directly (kernel attributes and occupancy caches are set up outside a
    // capture), the second captures, later ones replay
    ApplyCtx::Graph* hit = nullptr;
    for (auto& g : ctx->graph)
        if (g.x == x && g.y == y && g.nrhs == nrhs)
            hit = &g;
    if (hit && hit->exec) {
        hit->lru = ++ctx->graph_tick;
        ++ctx->graph_replays;
        cuda_check(cudaGraphLaunch(hit->exec, ctx->st), "cudaGraphLaunch");
        return hit->peak_children;
    }
    if (!hit) {
        ApplyCtx::Graph* slot = &ctx->graph[0];
        for (auto& g : ctx->graph)
            if (g.lru < slot->lru)
                slot = &g;
        if (slot->exec)
            cudaGraphExecDestroy(slot->exec);
        *slot = ApplyCtx::Graph{x, y, nrhs, nullptr, 0, ++ctx->graph_tick};
        return run_sched(op, ctx->st, ctx->work.p, x, y, nrhs, nullptr);
    }
    cudaStream_t cap;
    cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{cap};
    cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed), "capture");
    int64_t peak = 0;
    try {
        peak = run_sched(op, cap, ctx->work.p, x, y, nrhs, nullptr);
    } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(cap, &g);
        if (g)
            cudaGraphDestroy(g);
        throw;
    }
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamEndCapture(cap, &g), "end capture");
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    cuda_check(e, "cudaGraphInstantiate");
    hit->exec = exec;
    hit->peak_children = peak;
    hit->lru = ++ctx->graph_tick;
    ++ctx->graph_replays;
    cuda_check(cudaGraphLaunch(exec, ctx->st), "cudaGraphLaunch");
    return peak;
}

int64_t enqueue_apply_hooked(const DeviceOperator& op, ApplyCtx* ctx, const void* x, void* y,
                             int64_t nrhs, const std::function<void(int64_t)>& hook)
{
    return run_sched(op, ctx->st, ctx->work.p, x, y, nrhs, nullptr, hook);
}

uint64_t count_launches(int d, int q)
{
    // q single-child path levels (K1' + K3' each); below them a subtree of
    // mlev levels: 2^(mlev-1) - 1 K1 and K3 each plus 2^(mlev-1) leaf pairs.
    const int mlev = d - q;
    if (mlev == 0)
        return static_cast<uint64_t>(2 * (q - 1) + 1);
    return static_cast<uint64_t>(2 * q) + 3 * (uint64_t(1) << (mlev - 1)) - 2;
}

void fill_counters(const DeviceOperator& op, ts_metrics* m, int64_t peak_vectors)
{
    if (!m)
        return;
    // logical counts of the reference recursion (ref engine_split.cpp:69,74,
    // 90,93,98) restricted to the owned subtree, per vector component.
    const int d = op.d, q = op.q;
    const uint64_t s = static_cast<uint64_t>(op.s), mm = static_cast<uint64_t>(op.m);
    const uint64_t leaves = uint64_t(1) << (d - q);
    uint64_t ffts = 0, internal = 0;
    for (int depth = 1; depth <= d; ++depth)  // nodes at depth with an FFT on entry
        ffts += depth <= q ? 1 : (uint64_t(1) << (depth - q));
    for (int depth = 0; depth < d; ++depth)
        internal += depth < q ? 1 : (uint64_t(1) << (depth - q));
    m->fft_forward = ffts * mm;
    m->fft_inverse = ffts * mm;
    m->diag_mults = leaves * s * mm * mm;
    m->phase_mults = 2 * internal * s * mm;
    // measured: vectors the schedule held at once (x, y, children) — the
    // reference's lazy peak (d+1) s counts y = clone(v) and d children
    m->peak_live_elems = peak_vectors * static_cast<int64_t>(s * mm);
    m->kernel_elems = op.spectra_elems;
    m->precompute_ns = op.precompute_ns;
    m->apply_ns = 0;
}

// ---------------------------------------------------------------- device API

static void check_vectors(const DeviceOperator& op, const void* x, const void* y, int64_t nrhs)
{
    if (!x || !y)
        fail(TS_ERR_INVALID_ARGUMENT, "null argument");
    if (nrhs < 1)
        fail(TS_ERR_INVALID_ARGUMENT, "nrhs must be >= 1");
    // the fast passes move 16-byte vectors and bulk-copy rows (cp.async.bulk / TMA):
    // a base pointer off that alignment would fault inside a kernel
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must be 16-byte aligned device pointers");
    const size_t vb = op.vec_bytes() * static_cast<size_t>(nrhs);
    const char* xb = static_cast<const char*>(x);
    const char* yb = static_cast<const char*>(y);
    if (xb < yb + vb && yb < xb + vb)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must not alias");
}

std::vector<ts_launch_record> profile_device(const DeviceOperator& op, const void* x, void* y,
                                             void* stream)
{
    check_vectors(op, x, y, 1);
    if (op.is_embed || op.multi)
        fail(TS_ERR_INVALID_ARGUMENT, "profiling covers single-GPU split operators");
    DeviceGuard guard(op.device);
    std::vector<ts_launch_record> rec;
    CtxLease lease(op, static_cast<cudaStream_t>(stream), false, 1);
    enqueue_apply(op, lease.c, x, y, 1, &rec);
    return rec;
}

void apply_device(const DeviceOperator& op, const void* x, void* y, void* stream, ts_metrics* metrics)
{
    apply_batch_device(op, x, y, 1, stream, metrics);
}

void apply_batch_device(const DeviceOperator& op, const void* x, void* y, int64_t nrhs, void* stream,
                        ts_metrics* metrics)
{
    check_vectors(op, x, y, nrhs);
    if (op.multi) {
        multi_apply_device(op, x, y, nrhs, static_cast<cudaStream_t>(stream), metrics);
        return;
    }
    DeviceGuard guard(op.device);
    int64_t peak = 2;
    if (op.is_embed) {
        CtxLease lease(op, static_cast<cudaStream_t>(stream), false, 1);
        for (int64_t r = 0; r < nrhs; ++r)
            apply_embed(op, static_cast<const char*>(x) + op.vec_bytes() * r,
                        static_cast<char*>(y) + op.vec_bytes() * r, lease.c->st, lease.c->work.p);
    } else {
        CtxLease lease(op, static_cast<cudaStream_t>(stream), false, nrhs);
        peak = enqueue_apply(op, lease.c, x, y, nrhs);
    }
    cuda_check(cudaGetLastError(), "apply");
    if (metrics) {
        if (op.is_embed) {
            embed_counters(op, metrics);
        } else {
            fill_counters(op, metrics, peak);
            const uint64_t k = static_cast<uint64_t>(nrhs);
            metrics->fft_forward *= k;
            metrics->fft_inverse *= k;
            metrics->diag_mults *= k;
            metrics->phase_mults *= k;
            metrics->peak_live_elems *= static_cast<int64_t>(nrhs);
        }
    }
}

void embed_counters(const DeviceOperator& op, ts_metrics* metrics)
{
    // ref engine_embed.cpp:113-168 per component; the m x m block multiply
    // makes m^2 products per embedded frequency
    const uint64_t s = static_cast<uint64_t>(op.s), mm = static_cast<uint64_t>(op.m);
    metrics->fft_forward = static_cast<uint64_t>(op.d) * mm;
    metrics->fft_inverse = static_cast<uint64_t>(op.d) * mm;
    metrics->diag_mults = (uint64_t(1) << op.d) * s * mm * mm;
    metrics->phase_mults = 0;
    metrics->peak_live_elems = static_cast<int64_t>(((uint64_t(1) << op.d) + 2) * s * mm);
    metrics->kernel_elems = op.spectra_elems;
    metrics->precompute_ns = op.precompute_ns;
    metrics->apply_ns = 0;
}

void operator_info(const DeviceOperator& op, ts_operator_info* out)
{
    ts_operator_info r{};
    r.d = op.d;
    r.m = op.m;
    r.n_unique = op.n_unique;
    r.precision = op.prec;
    r.storage = op.compressed || op.embed_corner ? TS_STORAGE_COMPRESSED : TS_STORAGE_FULL;
    r.is_embed = op.is_embed ? 1 : 0;
    r.device = op.device;
    r.part = op.part;
    r.nparts = op.nparts;
    r.elem_bytes = op.es();
    r.spectra_bytes = op.spectra_elems * op.es();
    r.table_bytes = op.table_bytes();
    r.cached_bytes = op.cached_bytes();
    r.ndevices = 1;
    {
        std::lock_guard<std::mutex> lk(op.ctx_mu);
        for (const auto& c : op.ctxs)
            r.graph_replays += c->graph_replays;
    }
    if (op.is_embed) {
        r.workspace_bytes = work_bytes(op, 1);
        r.launches = 2 * op.d + 1 + 2 * op.m;
    } else {
        r.workspace_bytes = work_bytes(op, 1);
        r.launches = count_launches(op.d, op.q);
    }
    if (op.multi)
        multi_info(op, &r);
    *out = r;
}

}  // namespace tsb
