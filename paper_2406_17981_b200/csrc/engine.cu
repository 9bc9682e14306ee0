// Device engine of libtoesplit (B200): operator construction with on-device
// spectra precompute, the depth-first branch scheduler that drives the
// K1/K2/K3 kernels through the tsk_* launcher layer, the full-embedding
// baseline operator, and TSKF kernel files.
//
// Reference counterparts (relative to /root/reference/proj):
//   SplitOperator / build_spectra     src/core/engine_split.cpp:188-228
//   apply_split / branch recursion    src/core/engine_split.cpp:61-135
//   precompute_spectra (branchwise)   src/core/kernel.cpp:223-323
//   compress_spectra                  src/core/kernel.cpp:325-390
//   EmbedOperator                     src/core/engine_embed.cpp:61-168
//   TSKF save / load                  src/core/kernel.cpp:456-537
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "host.hpp"
#include "tsk_launch.h"

namespace tsb {

// ref kernel.cpp:17-21
static int64_t stored_len_host(int64_t n, int odd) { return odd ? (n + 1) / 2 : n / 2 + 1; }

// ---------------------------------------------------------------- errors

static void cuda_check(cudaError_t e, const char* what)
{
    if (e == cudaSuccess)
        return;
    cudaGetLastError();  // clear sticky-free errors
    const std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation)
        fail(TS_ERR_RESOURCE, "device out of memory (" + msg + ")");
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver || e == cudaErrorInvalidDevice)
        fail(TS_ERR_RESOURCE, "no usable CUDA device (" + msg + ")");
    fail(TS_ERR_INTERNAL, msg);
}

static void launch_check(int e, const char* what) { cuda_check(static_cast<cudaError_t>(e), what); }

int32_t device_count()
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (device_count() == 0)
            fail(TS_ERR_RESOURCE, "no CUDA device: the split engine runs on the GPU only");
        cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (dev >= 0 && dev != prev)
            cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard()
    {
        if (prev >= 0)
            cudaSetDevice(prev);
    }
};

struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes)
    {
        if (bytes)
            cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept
    {
        std::swap(p, o.p);
        return *this;
    }
    ~DevBuf()
    {
        if (p)
            cudaFree(p);
    }
};

// Keep freed stream-ordered memory in the device pool instead of returning it
// to the driver at every synchronization (the default threshold of 0 would
// remap the per-call workspace on each apply).
static void retain_pool()
{
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev)
        return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done_dev = dev;
}

// Stream-ordered scratch (cudaMallocAsync) released on scope exit.
struct AsyncBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    AsyncBuf(size_t bytes, cudaStream_t s) : st(s)
    {
        retain_pool();
        if (bytes)
            cuda_check(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
    }
    AsyncBuf(const AsyncBuf&) = delete;
    ~AsyncBuf()
    {
        if (p)
            cudaFreeAsync(p, st);
    }
};

// ---------------------------------------------------------------- tables

// exp(sign * 2 pi i k / n), octant-reduced so the table is ~1 ulp accurate
// (the c64 path rounds these double values; SURVEY.md §7 hard part 3).
static cplx unit_root(int64_t k, int64_t n, int sign)
{
    k %= n;
    if (k < 0)
        k += n;
    const int64_t a = 8 * k, o = a / n, r = a - o * n;
    double c, s;
    if ((o & 1) == 0) {
        const double th = (std::numbers::pi / 4.0) * (static_cast<double>(r) / n);
        c = std::cos(th);
        s = std::sin(th);
    } else {
        const double th = (std::numbers::pi / 4.0) * (static_cast<double>(n - r) / n);
        c = std::sin(th);
        s = std::cos(th);
    }
    double cr, sr;
    switch ((o / 2) & 3) {
    case 0: cr = c; sr = s; break;
    case 1: cr = -s; sr = c; break;
    case 2: cr = -c; sr = -s; break;
    default: cr = s; sr = -c; break;
    }
    return {cr, sign < 0 ? -sr : sr};
}

static std::vector<int32_t> radices(int64_t n)
{
    std::vector<int32_t> r;
    int64_t m = n;
    while (m % 8 == 0) {
        r.push_back(8);
        m /= 8;
    }
    while (m % 4 == 0) {
        r.push_back(4);
        m /= 4;
    }
    while (m % 2 == 0) {
        r.push_back(2);
        m /= 2;
    }
    for (int64_t f = 3; m > 1; f += 2) {
        while (m % f == 0) {
            r.push_back(static_cast<int32_t>(f));
            m /= f;
        }
        if (f * f > m && m > 1) {
            r.push_back(static_cast<int32_t>(m));
            m = 1;
        }
    }
    if (static_cast<int>(r.size()) > TSK_MAX_RADICES)
        fail(TS_ERR_SHAPE, "axis length has too many prime factors");
    return r;
}

// Per-length device tables: roots exp(-2 pi i k/n) and phases exp(-i pi k/n).
struct AxisTables {
    int64_t n = 0;
    DevBuf roots, phase;
    std::vector<int32_t> rad;
};

static std::shared_ptr<AxisTables> make_tables(int64_t n, int prec)
{
    if (n > (int64_t(1) << 24))
        fail(TS_ERR_SHAPE, "axis length too large for the device engine");
    auto t = std::make_shared<AxisTables>();
    t->n = n;
    t->rad = radices(n);
    const size_t es = prec ? 8 : 16;
    t->roots = DevBuf(n * es);
    t->phase = DevBuf(n * es);
    std::vector<double> hr(2 * n), hp(2 * n);
    for (int64_t k = 0; k < n; ++k) {
        const cplx w = unit_root(k, n, -1), p = unit_root(k, 2 * n, -1);
        hr[2 * k] = w.real();
        hr[2 * k + 1] = w.imag();
        hp[2 * k] = p.real();
        hp[2 * k + 1] = p.imag();
    }
    if (prec) {
        std::vector<float> fr(hr.begin(), hr.end()), fp(hp.begin(), hp.end());
        cuda_check(cudaMemcpy(t->roots.p, fr.data(), n * es, cudaMemcpyHostToDevice), "tables");
        cuda_check(cudaMemcpy(t->phase.p, fp.data(), n * es, cudaMemcpyHostToDevice), "tables");
    } else {
        cuda_check(cudaMemcpy(t->roots.p, hr.data(), n * es, cudaMemcpyHostToDevice), "tables");
        cuda_check(cudaMemcpy(t->phase.p, hp.data(), n * es, cudaMemcpyHostToDevice), "tables");
    }
    return t;
}

// ---------------------------------------------------------------- operator

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

    size_t es() const { return prec ? 8 : 16; }
    bool owns(uint32_t b) const { return (b & static_cast<uint32_t>(nparts - 1)) == static_cast<uint32_t>(part); }
};

const Shape& operator_levels(const DeviceOperator& op) { return op.levels; }
uint64_t operator_kernel_elems(const DeviceOperator& op) { return op.spectra_elems; }

static void fill_tables(DeviceOperator& op, const Shape& lens,
                        std::vector<std::shared_ptr<AxisTables>>& out)
{
    std::map<int64_t, std::shared_ptr<AxisTables>> cache;
    out.clear();
    for (auto n : lens) {
        auto it = cache.find(n);
        if (it == cache.end())
            it = cache.emplace(n, make_tables(n, op.prec)).first;
        out.push_back(it->second);
    }
}

static tsk_axis axis_desc(const DeviceOperator& op, const Shape& shape,
                          const std::vector<std::shared_ptr<AxisTables>>& tabs, int axis,
                          int ncomp, int64_t cstride, int prec)
{
    tsk_axis a{};
    int64_t inner = 1, outer = 1;
    for (size_t b = axis + 1; b < shape.size(); ++b)
        inner *= shape[b];
    for (int b = 0; b < axis; ++b)
        outer *= shape[b];
    a.outer = outer;
    a.inner = inner;
    a.n = shape[axis];
    a.ncomp = ncomp;
    a.prec = prec;
    a.cstride = cstride;
    a.roots = tabs[axis]->roots.p;
    a.phase = tabs[axis]->phase.p;
    a.use_even = 1;
    a.use_odd = 1;
    a.scale = 1.0;
    a.nrad = static_cast<int32_t>(tabs[axis]->rad.size());
    for (int i = 0; i < a.nrad; ++i)
        a.rad[i] = tabs[axis]->rad[i];
    (void)op;
    return a;
}

// ---------------------------------------------------------------- precompute

namespace {

struct Precompute {
    DeviceOperator& op;
    const BlockGenerator& g;
    cudaStream_t st;
    std::vector<std::shared_ptr<AxisTables>> tabs64;  // c128 tables for the block FFTs
    DevBuf check;                                     // 2 doubles
    int u = 0;
    cplx s0;

    // ref kernel.cpp:260-275 (branchwise_blocks), depth-first, skipping
    // subtrees this partition does not own.
    void recurse(const void* t, Shape shape, int axis, uint32_t bits)
    {
        const int d = op.d;
        if (axis == d) {
            finish_block(t, bits);
            return;
        }
        Shape half = shape;
        half[axis] /= 2;
        DevBuf buf(static_cast<size_t>(volume(half)) * 16);
        for (int odd = 0; odd < 2; ++odd) {
            const uint32_t nb = odd ? bits | (1u << axis) : bits;
            if (axis < op.q && ((static_cast<uint32_t>(op.part) >> axis) & 1u) != static_cast<uint32_t>(odd))
                continue;
            launch_check(tsk_fold_axis(d, shape.data(), axis, odd, t, buf.p, st), "fold");
            recurse(buf.p, half, axis + 1, nb);
        }
    }

    void finish_block(const void* blk_c, uint32_t bits)
    {
        void* blk = const_cast<void*>(blk_c);
        // forward DFT along every axis, in place, c128 (fft_all_axes_inplace)
        for (int a = 0; a < op.d; ++a) {
            tsk_axis ax = axis_desc(op, op.levels, tabs64, a, 1, 0, 0);
            ax.src0 = blk;
            ax.dst0 = blk;
            ax.use_odd = 0;
            launch_check(tsk_fwd_split(&ax, st), "block fft");
        }
        if (op.compressed) {
            launch_check(tsk_mirror_check(op.d, op.levels.data(), bits, op.skew_mask[u], blk,
                                          static_cast<double*>(check.p), st),
                         "mirror check");
            double h[2];
            cuda_check(cudaMemcpyAsync(h, check.p, sizeof h, cudaMemcpyDeviceToHost, st), "check");
            cuda_check(cudaStreamSynchronize(st), "sync");
            const double tol = 1e-9 * std::max(h[0], 1.0);
            if (!(h[1] <= tol))
                fail(TS_ERR_SYMMETRY, std::string("spectra are not mirror ") +
                                          (op.skew_mask[u] ? "antisymmetric" : "symmetric") +
                                          " (wrong mode or nonzero skew padding)");
        }
        char* dst = static_cast<char*>(op.spectra.p) +
                    (op.branch_base[bits] + static_cast<int64_t>(u) * op.block_elems[bits]) * op.es();
        launch_check(tsk_store_block(op.d, op.levels.data(), bits, op.compressed ? 1 : 0, blk, dst,
                                     op.prec, st),
                     "store block");
    }
};

}  // namespace

std::shared_ptr<DeviceOperator> create_split(const BlockGenerator& g, const ts_split_options& opt)
{
    const auto t0 = std::chrono::steady_clock::now();
    if (opt.precision != TS_PREC_C128 && opt.precision != TS_PREC_C64)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid precision value");
    if (opt.storage != TS_STORAGE_AUTO && opt.storage != TS_STORAGE_FULL &&
        opt.storage != TS_STORAGE_COMPRESSED)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid storage value");
    const int d = static_cast<int>(g.levels.size());
    int q = 0;
    while ((1 << q) < opt.nparts)
        ++q;
    if (opt.nparts < 1 || (1 << q) != opt.nparts || q > d || opt.part < 0 || opt.part >= opt.nparts)
        fail(TS_ERR_INVALID_ARGUMENT, "nparts must be a power of two <= 2^d and 0 <= part < nparts");

    // storage rule (ref engine_split.cpp:193-202), per-axis generalisation:
    // compressible iff every stored component has a sign on every axis, and
    // skew axes need zero padding for the mirror property.
    const cplx s0{opt.s0_re, opt.s0_im};
    bool all_signed = true, any_skew = false;
    for (int v : g.axis_sign) {
        all_signed = all_signed && v != 0;
        any_skew = any_skew || v < 0;
    }
    bool compress;
    if (opt.storage == TS_STORAGE_AUTO)
        compress = all_signed && (!any_skew || s0 == cplx{});
    else
        compress = opt.storage == TS_STORAGE_COMPRESSED;
    if (compress && !all_signed)
        fail(TS_ERR_SYMMETRY, "compression requires a symmetric or skew generator");

    DeviceGuard guard(opt.device);
    auto op = std::make_shared<DeviceOperator>();
    cuda_check(cudaGetDevice(&op->device), "cudaGetDevice");
    op->levels = g.levels;
    op->d = d;
    op->s = volume(g.levels);
    op->m = g.m;
    op->n_unique = g.n_unique;
    op->comp_map = g.comp_map;
    op->axis_sign = g.axis_sign;
    op->prec = opt.precision;
    op->compressed = compress;
    op->part = opt.part;
    op->nparts = opt.nparts;
    op->q = q;
    op->tskf_symmetry = g.scalar_symmetry >= 0 ? g.scalar_symmetry : 255;
    for (int u = 0; u < g.n_unique; ++u) {
        uint32_t mask = 0;
        for (int a = 0; a < d; ++a)
            if (g.axis_sign[u * d + a] < 0)
                mask |= 1u << a;
        op->skew_mask.push_back(mask);
    }

    const uint32_t nb = 1u << d;
    op->branch_base.assign(nb, 0);
    op->block_elems.assign(nb, 0);
    int64_t total = 0;
    for (uint32_t b = 0; b < nb; ++b) {
        int64_t e = 1;
        for (int a = 0; a < d; ++a)
            e *= compress ? stored_len_host(g.levels[a], (b >> a) & 1u) : g.levels[a];
        op->block_elems[b] = e;
        if (op->owns(b)) {
            op->branch_base[b] = total;
            total += e * g.n_unique;
        }
    }
    op->spectra_elems = static_cast<uint64_t>(total);
    op->spectra = DevBuf(static_cast<size_t>(total) * op->es());
    fill_tables(*op, op->levels, op->tab);

    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};

    Precompute pc{*op, g, st, {}, DevBuf(2 * sizeof(double)), 0, s0};
    {
        DeviceOperator tmp;
        tmp.prec = 0;
        fill_tables(tmp, op->levels, pc.tabs64);
    }
    Shape eshape(d);
    for (int a = 0; a < d; ++a)
        eshape[a] = 2 * g.levels[a];
    const int64_t evol = volume(eshape);
    DevBuf emb(static_cast<size_t>(evol) * 16);
    DevBuf lagbuf;
    for (int u = 0; u < g.n_unique; ++u) {
        pc.u = u;
        if (g.dyadic) {
            launch_check(tsk_embed_dyadic(d, g.levels.data(), g.dyadic_ij[u].first,
                                          g.dyadic_ij[u].second, g.k, g.self_term.real(),
                                          g.self_term.imag(), s0.real(), s0.imag(), emb.p, st),
                         "embed dyadic");
        } else {
            const auto& lags = g.lags[u];
            if (!lagbuf.p)
                lagbuf = DevBuf(lags.size() * 16);
            cuda_check(cudaMemcpyAsync(lagbuf.p, lags.data(), lags.size() * 16,
                                       cudaMemcpyHostToDevice, st),
                       "upload lags");
            launch_check(tsk_embed_generator(d, g.levels.data(), lagbuf.p, s0.real(), s0.imag(),
                                             emb.p, st),
                         "embed generator");
        }
        pc.recurse(emb.p, eshape, 0, 0);
    }
    cuda_check(cudaStreamSynchronize(st), "precompute sync");
    op->precompute_ns = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
            .count());
    return op;
}

// ---------------------------------------------------------------- scheduler

namespace {

struct Sched {
    const DeviceOperator& op;
    cudaStream_t st;
    std::vector<void*> buf;  // child buffer per depth (index 1..d-1)
    int launches = 0;
    // profiling: an event pair around every launch when rec != nullptr
    std::vector<ts_launch_record>* rec = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* ev = nullptr;

    uint64_t unit() const { return static_cast<uint64_t>(op.s) * op.m * op.es(); }

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

    tsk_axis ax(int axis) const
    {
        return axis_desc(op, op.levels, op.tab, axis, op.m, op.s, op.prec);
    }

    void leaf(uint32_t b, const void* in, void* out, int use_even, int use_odd)
    {
        const int a = op.d - 1;
        tsk_axis x = ax(a);
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
        const uint64_t spec = static_cast<uint64_t>(op.n_unique) * op.es() *
                              ((use_even ? op.block_elems[be] : 0) + (use_odd ? op.block_elems[bo] : 0));
        after(2, a, !(use_even && use_odd), 2 * unit() + spec);
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
            before();
            launch_check(tsk_inv_merge(&iv, st), "inv merge'");
            after(3, delta, 1, 2 * unit());
            return;
        }
        void* child = buf[delta + 1];
        tsk_axis f = ax(delta);
        f.src0 = in;
        f.dst0 = out;
        f.dst1 = child;
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
        before();
        launch_check(tsk_inv_merge(&iv, st), "inv merge");
        after(3, delta, 0, 3 * unit());
    }
};

uint64_t count_launches(int d, int q)
{
    // q single-child path levels (K1' + K3' each); below them a subtree of
    // mlev levels: 2^(mlev-1) - 1 K1 and K3 each plus 2^(mlev-1) leaf pairs.
    const int mlev = d - q;
    if (mlev == 0)
        return static_cast<uint64_t>(2 * (q - 1) + 1);
    return static_cast<uint64_t>(2 * q) + 3 * (uint64_t(1) << (mlev - 1)) - 2;
}

void fill_counters(const DeviceOperator& op, ts_metrics* m)
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
    m->peak_live_elems = static_cast<int64_t>((d + 1) * s * mm);
    m->kernel_elems = op.spectra_elems;
    m->precompute_ns = op.precompute_ns;
    m->apply_ns = 0;
}

}  // namespace

static void apply_embed(const DeviceOperator& op, const void* x, void* y, cudaStream_t st);

static void apply_stream(const DeviceOperator& op, const void* x, void* y, cudaStream_t st,
                         std::vector<ts_launch_record>* rec = nullptr)
{
    if (op.is_embed) {
        apply_embed(op, x, y, st);
        return;
    }
    const size_t vbytes = static_cast<size_t>(op.s) * op.m * op.es();
    const int nchild = std::max(0, op.d - 1 - op.q);
    AsyncBuf work(vbytes * nchild, st);
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    Sched sc{op, st, std::vector<void*>(op.d + 1, nullptr)};
    sc.rec = rec;
    sc.ev = &ev;
    for (int i = 0; i < nchild; ++i)
        sc.buf[op.q + 1 + i] = static_cast<char*>(work.p) + vbytes * i;
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
}

std::vector<ts_launch_record> profile_device(const DeviceOperator& op, const void* x, void* y,
                                             void* stream)
{
    if (!x || !y || x == y)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must be distinct device buffers");
    if (op.is_embed)
        fail(TS_ERR_INVALID_ARGUMENT, "profiling covers split operators");
    DeviceGuard guard(op.device);
    std::vector<ts_launch_record> rec;
    apply_stream(op, x, y, static_cast<cudaStream_t>(stream), &rec);
    return rec;
}

void apply_device(const DeviceOperator& op, const void* x, void* y, void* stream,
                  ts_metrics* metrics)
{
    if (!x || !y)
        fail(TS_ERR_INVALID_ARGUMENT, "null argument");
    if (x == y)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must not alias");
    DeviceGuard guard(op.device);
    apply_stream(op, x, y, static_cast<cudaStream_t>(stream));
    cuda_check(cudaGetLastError(), "apply");
    if (metrics)
        fill_counters(op, metrics);
}

void apply_batch_device(const DeviceOperator& op, const void* x, void* y, int64_t nrhs, void* stream,
                        ts_metrics* metrics)
{
    if (!x || !y)
        fail(TS_ERR_INVALID_ARGUMENT, "null argument");
    if (nrhs < 1)
        fail(TS_ERR_INVALID_ARGUMENT, "nrhs must be >= 1");
    const size_t vb = static_cast<size_t>(op.s) * op.m * op.es();
    const char* xb = static_cast<const char*>(x);
    char* yb = static_cast<char*>(y);
    if (xb < yb + vb * nrhs && yb < xb + vb * nrhs)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must not alias");
    DeviceGuard guard(op.device);
    for (int64_t r = 0; r < nrhs; ++r)
        apply_stream(op, xb + vb * r, yb + vb * r, static_cast<cudaStream_t>(stream));
    cuda_check(cudaGetLastError(), "apply batch");
    if (metrics) {
        fill_counters(op, metrics);
        const uint64_t k = static_cast<uint64_t>(nrhs);
        metrics->fft_forward *= k;
        metrics->fft_inverse *= k;
        metrics->diag_mults *= k;
        metrics->phase_mults *= k;
    }
}


// ---- host <-> device transfer of the reference ABI's interleaved complex128
// buffers. Caller memory is pageable, so a single cudaMemcpy runs at the
// driver's bounce-buffer rate; large transfers instead use T worker threads,
// each with its own stream and two pinned 16 MB slots: a worker copies chunk
// i into a pinned slot (host memcpy) while the DMA of its previous chunk is in
// flight, and complex64 operators convert on the device per chunk.
namespace {

constexpr size_t kChunkElems = size_t(1) << 20;  // complex elements (16 MB as complex128)

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
        cuda_check(cudaHostAlloc(&p, kChunkElems * 16, cudaHostAllocPortable), "cudaHostAlloc");
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

int transfer_threads()
{
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return static_cast<int>(std::clamp(hw / 2, 2u, 8u));
}

// dir 0: host complex128 v -> device x (complex64 when c64); dir 1: device y
// -> host complex128. Blocks until done; errors surface as TsError.
void host_transfer(int dir, int device, double* host, void* dev, bool c64, int64_t count)
{
    const int64_t nchunks = (count + static_cast<int64_t>(kChunkElems) - 1) / static_cast<int64_t>(kChunkElems);
    const int T = static_cast<int>(std::min<int64_t>(transfer_threads(), nchunks));
    std::vector<std::thread> th;
    std::vector<std::string> err(T);
    for (int k = 0; k < T; ++k) {
        th.emplace_back([&, k] {
            cudaStream_t s = nullptr;
            void* pin[2] = {nullptr, nullptr};
            void* stage[2] = {nullptr, nullptr};
            cudaEvent_t ev[2] = {nullptr, nullptr};
            try {
                cuda_check(cudaSetDevice(device), "device");
                cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
                for (int b = 0; b < 2; ++b) {
                    pin[b] = pinned_pool().get();
                    cuda_check(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "event");
                    if (c64)
                        cuda_check(cudaMallocAsync(&stage[b], kChunkElems * 16, s), "cudaMallocAsync");
                }
                int64_t prev = -1;
                int pslot = 0;
                int j = 0;
                for (int64_t i = k; i < nchunks; i += T, ++j) {
                    const int slot = j & 1;
                    const int64_t off = i * static_cast<int64_t>(kChunkElems);
                    const int64_t n = std::min<int64_t>(kChunkElems, count - off);
                    const size_t hb = static_cast<size_t>(n) * 16;
                    if (dir == 0) {
                        if (j >= 2)
                            cuda_check(cudaEventSynchronize(ev[slot]), "event");
                        std::memcpy(pin[slot], host + 2 * off, hb);
                        if (c64) {
                            cuda_check(cudaMemcpyAsync(stage[slot], pin[slot], hb, cudaMemcpyHostToDevice, s), "H2D");
                            launch_check(tsk_convert(stage[slot], 0, static_cast<char*>(dev) + off * 8, 1, n, s),
                                         "convert");
                        } else {
                            cuda_check(cudaMemcpyAsync(static_cast<char*>(dev) + off * 16, pin[slot], hb,
                                                       cudaMemcpyHostToDevice, s),
                                       "H2D");
                        }
                        cuda_check(cudaEventRecord(ev[slot], s), "event");
                    } else {
                        if (c64) {
                            launch_check(tsk_convert(static_cast<char*>(dev) + off * 8, 1, stage[slot], 0, n, s),
                                         "convert");
                            cuda_check(cudaMemcpyAsync(pin[slot], stage[slot], hb, cudaMemcpyDeviceToHost, s), "D2H");
                        } else {
                            cuda_check(cudaMemcpyAsync(pin[slot], static_cast<char*>(dev) + off * 16, hb,
                                                       cudaMemcpyDeviceToHost, s),
                                       "D2H");
                        }
                        cuda_check(cudaEventRecord(ev[slot], s), "event");
                        // drain the previous chunk while this one is in flight
                        if (prev >= 0) {
                            cuda_check(cudaEventSynchronize(ev[pslot]), "event");
                            const int64_t po = prev * static_cast<int64_t>(kChunkElems);
                            const int64_t pn = std::min<int64_t>(kChunkElems, count - po);
                            std::memcpy(host + 2 * po, pin[pslot], static_cast<size_t>(pn) * 16);
                        }
                        prev = i;
                        pslot = slot;
                    }
                }
                if (dir == 1 && prev >= 0) {
                    cuda_check(cudaEventSynchronize(ev[pslot]), "event");
                    const int64_t po = prev * static_cast<int64_t>(kChunkElems);
                    const int64_t pn = std::min<int64_t>(kChunkElems, count - po);
                    std::memcpy(host + 2 * po, pin[pslot], static_cast<size_t>(pn) * 16);
                }
                cuda_check(cudaStreamSynchronize(s), "transfer sync");
            } catch (const std::exception& e) {
                err[k] = e.what();
            }
            if (s)
                cudaStreamSynchronize(s);
            for (int b = 0; b < 2; ++b) {
                if (stage[b])
                    cudaFreeAsync(stage[b], s);
                if (pin[b])
                    pinned_pool().put(pin[b]);
                if (ev[b])
                    cudaEventDestroy(ev[b]);
            }
            if (s) {
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            }
        });
    }
    for (auto& t : th)
        t.join();
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
    DeviceGuard guard(op.device);
    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    const int64_t count = op.s * op.m;
    const size_t hbytes = static_cast<size_t>(count) * 16;
    const size_t vbytes = static_cast<size_t>(count) * op.es();
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    uint64_t ns = 0;
    if (hbytes >= (size_t(64) << 20)) {
        // large: chunked, multi-threaded pinned staging (no full-size complex128 copies on device)
        AsyncBuf xw(vbytes, st), yw(vbytes, st);
        cuda_check(cudaStreamSynchronize(st), "alloc sync");
        host_transfer(0, op.device, const_cast<double*>(v), xw.p, op.prec != 0, count);
        cuda_check(cudaEventRecord(e0, st), "event");
        apply_stream(op, xw.p, yw.p, st);
        cuda_check(cudaEventRecord(e1, st), "event");
        cuda_check(cudaStreamSynchronize(st), "apply sync");
        host_transfer(1, op.device, y, yw.p, op.prec != 0, count);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ns = static_cast<uint64_t>(static_cast<double>(ms) * 1e6);
    } else {
        AsyncBuf xs(hbytes, st), ys(hbytes, st);
        AsyncBuf xw(op.prec ? vbytes : 0, st), yw(op.prec ? vbytes : 0, st);
        void* xin = op.prec ? xw.p : xs.p;
        void* yout = op.prec ? yw.p : ys.p;
        cuda_check(cudaMemcpyAsync(xs.p, v, hbytes, cudaMemcpyHostToDevice, st), "H2D");
        if (op.prec)
            launch_check(tsk_convert(xs.p, 0, xw.p, 1, count, st), "convert");
        cuda_check(cudaEventRecord(e0, st), "event");
        apply_stream(op, xin, yout, st);
        cuda_check(cudaEventRecord(e1, st), "event");
        if (op.prec)
            launch_check(tsk_convert(yw.p, 1, ys.p, 0, count, st), "convert");
        cuda_check(cudaMemcpyAsync(y, ys.p, hbytes, cudaMemcpyDeviceToHost, st), "D2H");
        cuda_check(cudaStreamSynchronize(st), "apply sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        ns = static_cast<uint64_t>(static_cast<double>(ms) * 1e6);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cuda_check(cudaStreamSynchronize(st), "apply sync");
    if (metrics) {
        if (op.is_embed) {
            const uint64_t s = static_cast<uint64_t>(op.s);
            metrics->fft_forward = static_cast<uint64_t>(op.d);
            metrics->fft_inverse = static_cast<uint64_t>(op.d);
            metrics->diag_mults = (uint64_t(1) << op.d) * s;
            metrics->phase_mults = 0;
            metrics->peak_live_elems = static_cast<int64_t>(((uint64_t(1) << op.d) + 2) * s);
            metrics->kernel_elems = op.spectra_elems;
            metrics->precompute_ns = op.precompute_ns;
        } else {
            fill_counters(op, metrics);
        }
        metrics->apply_ns = ns;
    }
}

void operator_info(const DeviceOperator& op, ts_operator_info* out)
{
    ts_operator_info r{};
    r.d = op.d;
    r.m = op.m;
    r.n_unique = op.n_unique;
    r.precision = op.prec;
    r.storage = op.compressed ? TS_STORAGE_COMPRESSED : TS_STORAGE_FULL;
    r.is_embed = op.is_embed ? 1 : 0;
    r.device = op.device;
    r.part = op.part;
    r.nparts = op.nparts;
    r.elem_bytes = op.es();
    r.spectra_bytes = op.spectra_elems * op.es();
    if (op.is_embed) {
        r.workspace_bytes = (static_cast<uint64_t>(1) << op.d) * op.s * op.es();
        r.launches = 2 * op.d + 3;
    } else {
        r.workspace_bytes = static_cast<uint64_t>(std::max(0, op.d - 1 - op.q)) * op.s * op.m * op.es();
        r.launches = count_launches(op.d, op.q);
    }
    *out = r;
}

// ---------------------------------------------------------------- embed

std::shared_ptr<DeviceOperator> create_embed(const Generator& g, cplx s0, ts_storage storage)
{
    const auto t0 = std::chrono::steady_clock::now();
    if (storage != TS_STORAGE_AUTO && storage != TS_STORAGE_FULL && storage != TS_STORAGE_COMPRESSED)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid storage value");
    bool compress = storage == TS_STORAGE_AUTO
                        ? (g.symmetry == TS_SYM_SYMMETRIC || (g.symmetry == TS_SYM_SKEW && s0 == cplx{}))
                        : storage == TS_STORAGE_COMPRESSED;
    if (compress && g.symmetry == TS_SYM_GENERAL)
        fail(TS_ERR_SYMMETRY, "compression requires a symmetric or skew generator");
    DeviceGuard guard(-1);
    auto op = std::make_shared<DeviceOperator>();
    cuda_check(cudaGetDevice(&op->device), "cudaGetDevice");
    op->is_embed = true;
    op->levels = g.levels;
    op->d = static_cast<int>(g.levels.size());
    op->s = volume(g.levels);
    op->prec = 0;
    op->embed_corner = compress;
    op->embed_skew = g.symmetry == TS_SYM_SKEW;
    Shape eshape(op->d);
    for (int a = 0; a < op->d; ++a)
        eshape[a] = 2 * g.levels[a];
    fill_tables(*op, eshape, op->tab2);
    const int64_t evol = volume(eshape);
    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevBuf spec(static_cast<size_t>(evol) * 16);
    {
        DevBuf lags(g.lags.size() * 16);
        cuda_check(cudaMemcpyAsync(lags.p, g.lags.data(), g.lags.size() * 16,
                                   cudaMemcpyHostToDevice, st),
                   "upload");
        launch_check(tsk_embed_generator(op->d, g.levels.data(), lags.p, s0.real(), s0.imag(),
                                         spec.p, st),
                     "embed");
        for (int a = 0; a < op->d; ++a) {
            tsk_axis x = axis_desc(*op, eshape, op->tab2, a, 1, 0, 0);
            x.src0 = spec.p;
            x.dst0 = spec.p;
            x.use_odd = 0;
            launch_check(tsk_fwd_split(&x, st), "symbol fft");
        }
        cuda_check(cudaStreamSynchronize(st), "sync");
    }
    if (compress) {
        DevBuf chk(2 * sizeof(double));
        const uint32_t mask = op->embed_skew ? ~0u : 0u;
        launch_check(tsk_mirror_check(op->d, eshape.data(), 0, mask, spec.p,
                                      static_cast<double*>(chk.p), st),
                     "mirror check");
        double h[2];
        cuda_check(cudaMemcpyAsync(h, chk.p, sizeof h, cudaMemcpyDeviceToHost, st), "check");
        cuda_check(cudaStreamSynchronize(st), "sync");
        if (!(h[1] <= 1e-9 * std::max(h[0], 1.0)))
            fail(TS_ERR_SYMMETRY, std::string("embedded spectrum is not mirror ") +
                                      (op->embed_skew ? "antisymmetric" : "symmetric"));
        int64_t corner = 1;
        for (auto n : g.levels)
            corner *= n + 1;
        op->symbol = DevBuf(static_cast<size_t>(corner) * 16);
        launch_check(tsk_store_block(op->d, eshape.data(), 0, 1, spec.p, op->symbol.p, 0, st),
                     "corner");
        cuda_check(cudaStreamSynchronize(st), "sync");
        op->spectra_elems = static_cast<uint64_t>(corner);
    } else {
        op->symbol = std::move(spec);
        op->spectra_elems = static_cast<uint64_t>(evol);
    }
    op->precompute_ns = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
            .count());
    return op;
}

// pad -> d forward passes -> symbol multiply -> d inverse passes -> project
// (ref engine_embed.cpp:113-168)
static void apply_embed(const DeviceOperator& op, const void* x, void* y, cudaStream_t st)
{
    Shape eshape(op.d);
    for (int a = 0; a < op.d; ++a)
        eshape[a] = 2 * op.levels[a];
    AsyncBuf work(static_cast<size_t>(volume(eshape)) * op.es(), st);
    launch_check(tsk_embed_corner(op.d, op.levels.data(), op.prec, x, work.p, 0, st), "pad");
    for (int a = 0; a < op.d; ++a) {
        tsk_axis f = axis_desc(op, eshape, op.tab2, a, 1, 0, op.prec);
        f.src0 = work.p;
        f.dst0 = work.p;
        f.use_odd = 0;
        launch_check(tsk_fwd_split(&f, st), "embed fwd");
    }
    launch_check(tsk_symbol_multiply(op.d, op.levels.data(), op.prec, work.p, op.symbol.p,
                                     op.embed_corner ? 1 : 0, op.embed_skew ? 1 : 0, st),
                 "symbol");
    for (int a = 0; a < op.d; ++a) {
        tsk_axis iv = axis_desc(op, eshape, op.tab2, a, 1, 0, op.prec);
        iv.src0 = work.p;
        iv.dst0 = work.p;
        iv.use_odd = 0;
        iv.scale = 1.0 / static_cast<double>(eshape[a]);
        launch_check(tsk_inv_merge(&iv, st), "embed inv");
    }
    launch_check(tsk_embed_corner(op.d, op.levels.data(), op.prec, work.p, y, 1, st), "project");
}

// ---------------------------------------------------------------- TSKF

namespace {

constexpr char kMagic[4] = {'T', 'S', 'K', 'F'};

void put_u32(std::ofstream& o, uint32_t v)
{
    unsigned char b[4];
    for (int i = 0; i < 4; ++i)
        b[i] = static_cast<unsigned char>(v >> (8 * i));
    o.write(reinterpret_cast<char*>(b), 4);
}

void put_i64(std::ofstream& o, int64_t v)
{
    unsigned char b[8];
    const auto u = static_cast<uint64_t>(v);
    for (int i = 0; i < 8; ++i)
        b[i] = static_cast<unsigned char>(u >> (8 * i));
    o.write(reinterpret_cast<char*>(b), 8);
}

uint32_t get_u32(std::ifstream& in)
{
    unsigned char b[4];
    if (!in.read(reinterpret_cast<char*>(b), 4))
        fail(TS_ERR_IO, "kernel file truncated");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i)
        v |= static_cast<uint32_t>(b[i]) << (8 * i);
    return v;
}

int64_t get_i64(std::ifstream& in)
{
    unsigned char b[8];
    if (!in.read(reinterpret_cast<char*>(b), 8))
        fail(TS_ERR_IO, "kernel file truncated");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i)
        v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return static_cast<int64_t>(v);
}

bool little_endian() { return std::endian::native == std::endian::little; }

}  // namespace

// Version 1 (ref proj/README.md:158-170, kernel.cpp:456-485) for scalar c128
// whole-tree operators; version 2 adds precision, block map, per-component
// skew masks and the partition:
//   ... u8 symmetry (255 = per-axis) | u8 storage | u16 reserved
//   | u32 m | u32 n_unique | u32 precision | u32 part | u32 nparts
//   | m*m x u8 comp_map | n_unique x u32 skew_mask
//   then per owned branch (ascending id), per unique component:
//   i64 count | count x (re, im) in the operator precision (f64 or f32).
void save_kernel(const DeviceOperator& op, const std::string& path)
{
    if (op.is_embed)
        fail(TS_ERR_INVALID_ARGUMENT, "kernel files hold split parity spectra only");
    if (!little_endian())
        fail(TS_ERR_IO, "TSKF writer requires a little-endian host");
    DeviceGuard guard(op.device);
    std::vector<char> host(op.spectra_elems * op.es());
    cuda_check(cudaMemcpy(host.data(), op.spectra.p, host.size(), cudaMemcpyDeviceToHost),
               "D2H spectra");
    std::ofstream out(path, std::ios::binary);
    if (!out)
        fail(TS_ERR_IO, "cannot write kernel file: " + path);
    const bool v1 = op.m == 1 && op.prec == 0 && op.nparts == 1 && op.tskf_symmetry != 255;
    out.write(kMagic, 4);
    put_u32(out, v1 ? 1 : 2);
    put_u32(out, static_cast<uint32_t>(op.d));
    for (auto n : op.levels)
        put_i64(out, n);
    const unsigned char hdr[4] = {static_cast<unsigned char>(v1 ? op.tskf_symmetry : 255),
                                  static_cast<unsigned char>(op.compressed ? 1 : 0), 0, 0};
    out.write(reinterpret_cast<const char*>(hdr), 4);
    if (!v1) {
        put_u32(out, static_cast<uint32_t>(op.m));
        put_u32(out, static_cast<uint32_t>(op.n_unique));
        put_u32(out, static_cast<uint32_t>(op.prec));
        put_u32(out, static_cast<uint32_t>(op.part));
        put_u32(out, static_cast<uint32_t>(op.nparts));
        for (int i = 0; i < op.m * op.m; ++i) {
            const char c = static_cast<char>(op.comp_map[i]);
            out.write(&c, 1);
        }
        for (auto mk : op.skew_mask)
            put_u32(out, mk);
    }
    for (uint32_t b = 0; b < (1u << op.d); ++b) {
        if (!op.owns(b))
            continue;
        for (int u = 0; u < op.n_unique; ++u) {
            put_i64(out, op.block_elems[b]);
            const char* p = host.data() + (op.branch_base[b] + u * op.block_elems[b]) * op.es();
            out.write(p, static_cast<std::streamsize>(op.block_elems[b] * op.es()));
        }
    }
    if (!out)
        fail(TS_ERR_IO, "write failure on kernel file: " + path);
}

std::shared_ptr<DeviceOperator> load_split(const std::string& path)
{
    std::ifstream in(path, std::ios::binary);
    if (!in)
        fail(TS_ERR_IO, "cannot open kernel file: " + path);
    char magic[4];
    if (!in.read(magic, 4) || std::memcmp(magic, kMagic, 4) != 0)
        fail(TS_ERR_IO, "not a kernel spectra file: " + path);
    const uint32_t version = get_u32(in);
    if (version != 1 && version != 2)
        fail(TS_ERR_IO, "unsupported kernel file version " + std::to_string(version));
    const uint32_t d = get_u32(in);
    if (d < 1 || d > 31)
        fail(TS_ERR_LOGIC, "kernel file has invalid level count");
    Shape levels(d);
    for (auto& n : levels) {
        n = get_i64(in);
        if (n < 1)
            fail(TS_ERR_LOGIC, "kernel file has invalid level size");
    }
    unsigned char hdr[4];
    if (!in.read(reinterpret_cast<char*>(hdr), 4))
        fail(TS_ERR_IO, "kernel file truncated");
    const unsigned sym = hdr[0], sto = hdr[1];
    if (sto > 1 || (version == 1 && sym > 2))
        fail(TS_ERR_LOGIC, "kernel file has invalid mode fields");
    auto op = std::make_shared<DeviceOperator>();
    op->levels = levels;
    op->d = static_cast<int>(d);
    op->s = volume(levels);
    op->compressed = sto == 1;
    if (version == 1) {
        op->m = 1;
        op->n_unique = 1;
        op->comp_map = {0};
        op->prec = 0;
        op->tskf_symmetry = static_cast<int>(sym);
        op->skew_mask = {sym == 2 ? (d >= 32 ? ~0u : ((1u << d) - 1)) : 0u};
    } else {
        op->m = static_cast<int>(get_u32(in));
        op->n_unique = static_cast<int>(get_u32(in));
        op->prec = static_cast<int>(get_u32(in));
        op->part = static_cast<int>(get_u32(in));
        op->nparts = static_cast<int>(get_u32(in));
        op->tskf_symmetry = static_cast<int>(sym);
        if (op->m < 1 || op->m > TSK_MAX_M || op->n_unique < 1 || op->n_unique > TSK_MAX_UNIQUE ||
            op->prec < 0 || op->prec > 1 || op->nparts < 1 ||
            (op->nparts & (op->nparts - 1)) != 0 || op->part < 0 || op->part >= op->nparts ||
            op->nparts > (1 << d))
            fail(TS_ERR_LOGIC, "kernel file has invalid extension fields");
        for (int i = 0; i < op->m * op->m; ++i) {
            char c;
            if (!in.read(&c, 1))
                fail(TS_ERR_IO, "kernel file truncated");
            if (c < 0 || c >= op->n_unique)
                fail(TS_ERR_LOGIC, "kernel file has invalid component map");
            op->comp_map.push_back(c);
        }
        for (int u = 0; u < op->n_unique; ++u)
            op->skew_mask.push_back(get_u32(in));
        while ((1 << op->q) < op->nparts)
            ++op->q;
    }
    for (int u = 0; u < op->n_unique; ++u)
        for (uint32_t a = 0; a < d; ++a)
            op->axis_sign.push_back(((op->skew_mask[u] >> a) & 1u) ? -1 : 1);
    const uint32_t nb = 1u << d;
    op->branch_base.assign(nb, 0);
    op->block_elems.assign(nb, 0);
    int64_t total = 0;
    for (uint32_t b = 0; b < nb; ++b) {
        int64_t e = 1;
        for (uint32_t a = 0; a < d; ++a)
            e *= op->compressed ? stored_len_host(levels[a], (b >> a) & 1u) : levels[a];
        op->block_elems[b] = e;
        if (op->owns(b)) {
            op->branch_base[b] = total;
            total += e * op->n_unique;
        }
    }
    op->spectra_elems = static_cast<uint64_t>(total);
    std::vector<char> host(static_cast<size_t>(total) * op->es());
    for (uint32_t b = 0; b < nb; ++b) {
        if (!op->owns(b))
            continue;
        for (int u = 0; u < op->n_unique; ++u) {
            const int64_t cnt = get_i64(in);
            if (cnt != op->block_elems[b])
                fail(TS_ERR_LOGIC, "kernel file block size mismatch");
            char* p = host.data() + (op->branch_base[b] + u * op->block_elems[b]) * op->es();
            if (!in.read(p, static_cast<std::streamsize>(cnt * op->es())))
                fail(TS_ERR_IO, "kernel file truncated");
        }
    }
    DeviceGuard guard(-1);
    cuda_check(cudaGetDevice(&op->device), "cudaGetDevice");
    op->spectra = DevBuf(host.size());
    cuda_check(cudaMemcpy(op->spectra.p, host.data(), host.size(), cudaMemcpyHostToDevice),
               "H2D spectra");
    fill_tables(*op, op->levels, op->tab);
    return op;
}

}  // namespace tsb
