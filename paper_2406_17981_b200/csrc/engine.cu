// Device engine of libtoesplit (B200), setup side: per-length twiddle
// tables, operator construction with on-device spectra precompute, and the
// full-embedding baseline operator. The apply paths live in sched.cpp
// (device buffers), transfer.cpp (host buffers of the reference ABI) and
// multi.cpp (several GPUs); TSKF files in tskf.cpp.
//
// Reference counterparts (relative to /root/reference/proj):
//   SplitOperator / build_spectra     src/core/engine_split.cpp:188-228
//   precompute_spectra (branchwise)   src/core/kernel.cpp:223-323
//   compress_spectra                  src/core/kernel.cpp:325-390
//   EmbedOperator                     src/core/engine_embed.cpp:61-168
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <numbers>
#include <vector>

#include "engine.hpp"

namespace tsb {


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

std::shared_ptr<AxisTables> make_tables(int64_t n, int prec)
{
    if (n > (int64_t(1) << 24))
        fail(TS_ERR_SHAPE, "axis length too large for the device engine");
    auto t = std::make_shared<AxisTables>();
    t->n = n;
    t->rad = radices(n);
    const size_t es = prec ? 8 : 16;
    t->roots = DevBuf(n * es, MEM_TABLES);
    t->phase = DevBuf(n * es, MEM_TABLES);
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

const Shape& operator_levels(const DeviceOperator& op) { return op.levels; }
uint64_t operator_kernel_elems(const DeviceOperator& op) { return op.spectra_elems; }

uint64_t DeviceOperator::table_bytes() const
{
    uint64_t b = 0;
    std::vector<const AxisTables*> seen;
    for (const auto* v : {&tab, &tab2})
        for (const auto& t : *v)
            if (t && std::find(seen.begin(), seen.end(), t.get()) == seen.end()) {
                seen.push_back(t.get());
                b += t->roots.bytes + t->phase.bytes;
            }
    return b;
}

void fill_tables(DeviceOperator& op, const Shape& lens, std::vector<std::shared_ptr<AxisTables>>& out)
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

tsk_axis axis_desc(const Shape& shape, const std::vector<std::shared_ptr<AxisTables>>& tabs, int axis,
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
    a.nrhs = 1;
    a.rstride = 0;
    a.nrad = static_cast<int32_t>(tabs[axis]->rad.size());
    for (int i = 0; i < a.nrad; ++i)
        a.rad[i] = tabs[axis]->rad[i];
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
        DevBuf buf(static_cast<size_t>(volume(half)) * 16, MEM_STAGING);
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
            tsk_axis ax = axis_desc(op.levels, tabs64, a, 1, 0, 0);
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
    op->spectra = DevBuf(static_cast<size_t>(total) * op->es(), MEM_SPECTRA);
    fill_tables(*op, op->levels, op->tab);

    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};

    Precompute pc{*op, g, st, {}, DevBuf(2 * sizeof(double), MEM_STAGING), 0, s0};
    {
        DeviceOperator tmp;
        tmp.prec = 0;
        fill_tables(tmp, op->levels, pc.tabs64);
    }
    // embedding + first fold in one sweep per (component, axis-0 parity): the
    // (2n)^d embedding is never materialised (setup peak: the half tensor)
    Shape half(d);
    for (int a = 0; a < d; ++a)
        half[a] = 2 * g.levels[a];
    half[0] = g.levels[0];
    DevBuf h0(static_cast<size_t>(volume(half)) * 16, MEM_STAGING);
    DevBuf lagbuf;
    for (int u = 0; u < g.n_unique; ++u) {
        pc.u = u;
        if (!g.dyadic) {
            const auto& lags = g.lags[u];
            if (!lagbuf.p)
                lagbuf = DevBuf(lags.size() * 16, MEM_STAGING);
            cuda_check(cudaMemcpyAsync(lagbuf.p, lags.data(), lags.size() * 16,
                                       cudaMemcpyHostToDevice, st),
                       "upload lags");
        }
        for (int odd = 0; odd < 2; ++odd) {
            if (op->q > 0 && (op->part & 1) != odd)
                continue;  // axis 0's other parity belongs to another partition
            launch_check(tsk_embed_fold0(d, g.levels.data(), g.dyadic ? nullptr : lagbuf.p,
                                         g.dyadic ? g.dyadic_ij[u].first : 0,
                                         g.dyadic ? g.dyadic_ij[u].second : 0, g.k,
                                         g.self_term.real(), g.self_term.imag(), s0.real(), s0.imag(),
                                         odd, h0.p, st),
                         "embed + fold");
            pc.recurse(h0.p, half, 1, static_cast<uint32_t>(odd));
        }
    }
    cuda_check(cudaStreamSynchronize(st), "precompute sync");
    op->precompute_ns = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
            .count());
    return op;
}

// ---------------------------------------------------------------- embed

// Full circulant embedding (the method the paper improves on; ref
// engine_embed.cpp:61-168) on this library's own FFT passes, for m x m block
// generators in complex64 / complex128: per unique component the (2n)^d
// symbol (or its (n+1)^d mirror corner) is computed on the device in
// complex128 and stored in the operator precision.
std::shared_ptr<DeviceOperator> create_embed_block(const BlockGenerator& g, const ts_split_options& opt)
{
    const auto t0 = std::chrono::steady_clock::now();
    if (opt.precision != TS_PREC_C128 && opt.precision != TS_PREC_C64)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid precision value");
    if (opt.storage != TS_STORAGE_AUTO && opt.storage != TS_STORAGE_FULL &&
        opt.storage != TS_STORAGE_COMPRESSED)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid storage value");
    if (g.m > TSK_MAX_M || g.n_unique > TSK_MAX_UNIQUE)
        fail(TS_ERR_SHAPE, "block arity too large for the embedding engine");
    const cplx s0{opt.s0_re, opt.s0_im};
    bool all_signed = true, any_skew = false;
    for (int v : g.axis_sign) {
        all_signed = all_signed && v != 0;
        any_skew = any_skew || v < 0;
    }
    const bool compress = opt.storage == TS_STORAGE_AUTO ? all_signed && (!any_skew || s0 == cplx{})
                                                         : opt.storage == TS_STORAGE_COMPRESSED;
    if (compress && !all_signed)
        fail(TS_ERR_SYMMETRY, "compression requires a symmetric or skew generator");
    DeviceGuard guard(opt.device);
    auto op = std::make_shared<DeviceOperator>();
    cuda_check(cudaGetDevice(&op->device), "cudaGetDevice");
    const int d = static_cast<int>(g.levels.size());
    op->is_embed = true;
    op->levels = g.levels;
    op->d = d;
    op->s = volume(g.levels);
    op->m = g.m;
    op->n_unique = g.n_unique;
    op->comp_map = g.comp_map;
    op->axis_sign = g.axis_sign;
    op->prec = opt.precision;
    op->embed_corner = compress;
    op->tskf_symmetry = g.scalar_symmetry >= 0 ? g.scalar_symmetry : 255;
    for (int u = 0; u < g.n_unique; ++u) {
        uint32_t mask = 0;
        for (int a = 0; a < d; ++a)
            if (g.axis_sign[u * d + a] < 0)
                mask |= 1u << a;
        op->skew_mask.push_back(mask);
    }
    Shape eshape(d);
    for (int a = 0; a < d; ++a)
        eshape[a] = 2 * g.levels[a];
    fill_tables(*op, eshape, op->tab2);  // operator precision, for the apply
    std::vector<std::shared_ptr<AxisTables>> tabs64;  // complex128, for the symbol
    {
        DeviceOperator tmp;
        tmp.prec = 0;
        fill_tables(tmp, eshape, tabs64);
    }
    const int64_t evol = volume(eshape);
    int64_t blk = evol;
    if (compress) {
        blk = 1;
        for (auto n : g.levels)
            blk *= n + 1;
    }
    op->block_elems.assign(1, blk);
    op->symbol = DevBuf(static_cast<size_t>(blk) * g.n_unique * op->es(), MEM_SPECTRA);
    op->spectra_elems = static_cast<uint64_t>(blk) * g.n_unique;
    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevBuf spec(static_cast<size_t>(evol) * 16, MEM_STAGING), lagbuf, chk(2 * sizeof(double), MEM_STAGING);
    for (int u = 0; u < g.n_unique; ++u) {
        if (g.dyadic) {
            launch_check(tsk_embed_dyadic(d, g.levels.data(), g.dyadic_ij[u].first, g.dyadic_ij[u].second,
                                          g.k, g.self_term.real(), g.self_term.imag(), s0.real(), s0.imag(),
                                          spec.p, st),
                         "embed dyadic");
        } else {
            const auto& lags = g.lags[u];
            if (!lagbuf.p)
                lagbuf = DevBuf(lags.size() * 16, MEM_STAGING);
            cuda_check(cudaMemcpyAsync(lagbuf.p, lags.data(), lags.size() * 16, cudaMemcpyHostToDevice, st),
                       "upload");
            launch_check(tsk_embed_generator(d, g.levels.data(), lagbuf.p, s0.real(), s0.imag(), spec.p, st),
                         "embed");
        }
        for (int a = 0; a < d; ++a) {
            tsk_axis x = axis_desc(eshape, tabs64, a, 1, 0, 0);
            x.src0 = spec.p;
            x.dst0 = spec.p;
            x.use_odd = 0;
            launch_check(tsk_fwd_split(&x, st), "symbol fft");
        }
        char* dst = static_cast<char*>(op->symbol.p) + static_cast<size_t>(u) * blk * op->es();
        if (compress) {
            launch_check(tsk_mirror_check(d, eshape.data(), 0, op->skew_mask[u], spec.p,
                                          static_cast<double*>(chk.p), st),
                         "mirror check");
            double h[2];
            cuda_check(cudaMemcpyAsync(h, chk.p, sizeof h, cudaMemcpyDeviceToHost, st), "check");
            cuda_check(cudaStreamSynchronize(st), "sync");
            if (!(h[1] <= 1e-9 * std::max(h[0], 1.0)))
                fail(TS_ERR_SYMMETRY, std::string("embedded spectrum is not mirror ") +
                                          (op->skew_mask[u] ? "antisymmetric" : "symmetric"));
            launch_check(tsk_store_block(d, eshape.data(), 0, 1, spec.p, dst, op->prec, st), "corner");
        } else {
            launch_check(tsk_convert(spec.p, 0, dst, op->prec, evol, st), "symbol");
        }
    }
    cuda_check(cudaStreamSynchronize(st), "sync");
    op->precompute_ns = static_cast<uint64_t>(
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
            .count());
    return op;
}

std::shared_ptr<DeviceOperator> create_embed(const Generator& g, cplx s0, ts_storage storage)
{
    ts_split_options o{};
    o.precision = TS_PREC_C128;
    o.storage = storage;
    o.device = -1;
    o.part = 0;
    o.nparts = 1;
    o.s0_re = s0.real();
    o.s0_im = s0.imag();
    return create_embed_block(block_from_scalar(g), o);
}

// pad -> d forward passes -> block symbol multiply -> d inverse passes ->
// project, all m components per launch (ref engine_embed.cpp:113-168)
void apply_embed(const DeviceOperator& op, const void* x, void* y, cudaStream_t st, void* work)
{
    Shape eshape(op.d);
    for (int a = 0; a < op.d; ++a)
        eshape[a] = 2 * op.levels[a];
    const int64_t evol = volume(eshape);
    const size_t es = op.es();
    char* wk = static_cast<char*>(work);
    // d = 3: pad / project are a memset plus one pitched 3-D copy per component
    // (copy-engine rates); other d: the index-mapping kernel
    auto corner_copy = [&](const void* src, bool src_big, void* dst) {
        const size_t rowb = static_cast<size_t>(op.levels[2]) * es;
        cudaMemcpy3DParms p{};
        const size_t bigp = 2 * rowb, smallp = rowb;
        p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(src), src_big ? bigp : smallp, rowb,
                                       static_cast<size_t>(src_big ? 2 * op.levels[1] : op.levels[1]));
        p.dstPtr = make_cudaPitchedPtr(dst, src_big ? smallp : bigp, rowb,
                                       static_cast<size_t>(src_big ? op.levels[1] : 2 * op.levels[1]));
        p.extent = make_cudaExtent(rowb, static_cast<size_t>(op.levels[1]), static_cast<size_t>(op.levels[0]));
        p.kind = cudaMemcpyDeviceToDevice;
        cuda_check(cudaMemcpy3DAsync(&p, st), "corner copy");
    };
    for (int c = 0; c < op.m; ++c) {
        const char* xc = static_cast<const char*>(x) + c * op.s * es;
        char* wc = wk + c * evol * es;
        if (op.d == 3) {
            cuda_check(cudaMemsetAsync(wc, 0, static_cast<size_t>(evol) * es, st), "pad zero");
            corner_copy(xc, false, wc);
        } else {
            launch_check(tsk_embed_corner(op.d, op.levels.data(), op.prec, xc, wc, 0, st), "pad");
        }
    }
    for (int a = 0; a < op.d; ++a) {
        tsk_axis f = axis_desc(eshape, op.tab2, a, op.m, evol, op.prec);
        f.src0 = wk;
        f.dst0 = wk;
        f.use_odd = 0;
        launch_check(tsk_fwd_split(&f, st), "embed fwd");
    }
    tsk_block_symbol bs{};
    bs.data = op.symbol.p;
    bs.block_elems = op.block_elems.empty() ? 0 : op.block_elems[0];
    bs.m = op.m;
    bs.n_unique = op.n_unique;
    bs.corner = op.embed_corner ? 1 : 0;
    for (int u = 0; u < op.n_unique; ++u)
        bs.skew_mask[u] = op.skew_mask[u];
    for (int i = 0; i < op.m * op.m; ++i)
        bs.comp_map[i] = static_cast<int8_t>(op.comp_map[i]);
    launch_check(tsk_block_symbol_multiply(op.d, op.levels.data(), op.prec, wk, evol, &bs, st), "symbol");
    for (int a = 0; a < op.d; ++a) {
        tsk_axis iv = axis_desc(eshape, op.tab2, a, op.m, evol, op.prec);
        iv.src0 = wk;
        iv.dst0 = wk;
        iv.use_odd = 0;
        iv.scale = 1.0 / static_cast<double>(eshape[a]);
        launch_check(tsk_inv_merge(&iv, st), "embed inv");
    }
    for (int c = 0; c < op.m; ++c) {
        char* yc = static_cast<char*>(y) + c * op.s * es;
        if (op.d == 3)
            corner_copy(wk + c * evol * es, true, yc);
        else
            launch_check(tsk_embed_corner(op.d, op.levels.data(), op.prec, wk + c * evol * es, yc, 1, st),
                         "project");
    }
}

}  // namespace tsb
