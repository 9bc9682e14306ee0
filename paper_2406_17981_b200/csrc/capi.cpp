// C ABI of libtoesplit.so.1 (B200 build): the 22 functions of the reference
// header (ref proj/include/toesplit.h:84-156, behaviour of
// ref proj/src/capi/capi.cpp) plus the toesplit_ext.h extensions. Every entry
// point is exception-free: failures become ts_status codes with a
// thread-local detail string (ref capi.cpp:27-68).
#include <cstring>
#include <fstream>
#include <new>
#include <sstream>
#include <string>

#include "engine.hpp"
#include "host.hpp"
#include "multi.hpp"
#include "tsk_launch.h"

using namespace tsb;

namespace {

thread_local std::string g_last_error;

template <typename Fn>
ts_status guarded(Fn&& fn)
{
    try {
        fn();
        g_last_error.clear();
        return TS_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of memory";
        return TS_ERR_RESOURCE;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return TS_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return TS_ERR_LOGIC;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return TS_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return TS_ERR_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return TS_ERR_INTERNAL;
    }
}

void need(bool ok, const char* what = "null argument")
{
    if (!ok)
        fail(TS_ERR_INVALID_ARGUMENT, what);
}

std::vector<cplx> from_interleaved(const double* p, int64_t count)
{
    need(p != nullptr, "null buffer");
    std::vector<cplx> v(static_cast<size_t>(count));
    std::memcpy(static_cast<void*>(v.data()), p, static_cast<size_t>(count) * sizeof(cplx));
    return v;
}

}  // namespace

extern "C" {

const char* ts_version(void) { return "1.0.0"; }

const char* ts_status_name(ts_status status)
{
    switch (status) {
    case TS_OK: return "ok";
    case TS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case TS_ERR_SHAPE: return "shape mismatch";
    case TS_ERR_SYMMETRY: return "symmetry violation";
    case TS_ERR_CAP_EXCEEDED: return "cap exceeded";
    case TS_ERR_RESOURCE: return "resource exhausted";
    case TS_ERR_IO: return "io error";
    case TS_ERR_LOGIC: return "logic error";
    case TS_ERR_INTERNAL: return "internal error";
    }
    return "unknown";
}

const char* ts_last_error(void) { return g_last_error.c_str(); }

ts_status ts_generator_create(int32_t d, const int64_t* levels, const double* lags,
                              ts_symmetry symmetry, ts_generator** out)
{
    return guarded([&] {
        need(out != nullptr, "null out pointer");
        Shape lv = check_levels(d, levels);
        int64_t count = 1;
        for (auto n : lv)
            count *= 2 * n - 1;
        auto g = make_generator(lv, from_interleaved(lags, count), symmetry);
        *out = new ts_generator{std::move(g)};
    });
}

ts_status ts_generator_random(int32_t d, const int64_t* levels, uint64_t seed, double variance,
                              ts_symmetry symmetry, ts_generator** out)
{
    return guarded([&] {
        need(out != nullptr, "null out pointer");
        if (symmetry != TS_SYM_GENERAL && symmetry != TS_SYM_SYMMETRIC && symmetry != TS_SYM_SKEW)
            fail(TS_ERR_INVALID_ARGUMENT, "invalid symmetry value");
        auto g = random_generator(check_levels(d, levels), seed, variance, symmetry);
        *out = new ts_generator{std::move(g)};
    });
}

ts_status ts_generator_from_json_file(const char* path, ts_generator** out)
{
    return guarded([&] {
        need(out && path);
        std::ifstream in(path);
        if (!in)
            fail(TS_ERR_IO, std::string("cannot open generator file: ") + path);
        std::ostringstream buf;
        buf << in.rdbuf();
        auto g = generator_from_json(buf.str());
        *out = new ts_generator{std::move(g)};
    });
}

ts_status ts_generator_to_json_file(const ts_generator* g, const char* path)
{
    return guarded([&] {
        need(g && path);
        std::ofstream out(path);
        if (!out)
            fail(TS_ERR_IO, std::string("cannot write generator file: ") + path);
        out << generator_to_json(g->g) << "\n";
        if (!out)
            fail(TS_ERR_IO, std::string("write failure on generator file: ") + path);
    });
}

int32_t ts_generator_dims(const ts_generator* g)
{
    return g ? static_cast<int32_t>(g->g.levels.size()) : 0;
}

ts_status ts_generator_levels(const ts_generator* g, int64_t* out_levels)
{
    return guarded([&] {
        need(g && out_levels);
        for (size_t a = 0; a < g->g.levels.size(); ++a)
            out_levels[a] = g->g.levels[a];
    });
}

void ts_generator_destroy(ts_generator* g) { delete g; }

ts_status ts_random_vector(int32_t d, const int64_t* levels, uint64_t seed, double variance,
                           double* out)
{
    return guarded([&] {
        need(out != nullptr, "null out buffer");
        random_vector_into(check_levels(d, levels), seed, variance, reinterpret_cast<cplx*>(out));
    });
}

ts_status ts_operator_create_split(const ts_generator* g, double s0_re, double s0_im,
                                   ts_storage storage, ts_operator** out)
{
    return guarded([&] {
        need(g && out);
        ts_split_options opt;
        ts_split_options_default(&opt);
        opt.storage = storage;
        opt.s0_re = s0_re;
        opt.s0_im = s0_im;
        auto dev = create_split(block_from_scalar(g->g), opt);
        *out = new ts_operator{OperatorHandle{std::move(dev)}};
    });
}

ts_status ts_operator_create_embed(const ts_generator* g, double s0_re, double s0_im,
                                   ts_storage storage, ts_operator** out)
{
    return guarded([&] {
        need(g && out);
        auto dev = create_embed(g->g, cplx{s0_re, s0_im}, storage);
        *out = new ts_operator{OperatorHandle{std::move(dev)}};
    });
}

ts_status ts_operator_apply(const ts_operator* op, const double* v, double* y,
                            const ts_policy* policy, ts_metrics* metrics)
{
    return guarded([&] {
        need(op && v && y);
        apply_host(*op->h.dev, v, y, policy, metrics);
    });
}

int32_t ts_operator_dims(const ts_operator* op)
{
    return op ? static_cast<int32_t>(operator_levels(*op->h.dev).size()) : 0;
}

ts_status ts_operator_levels(const ts_operator* op, int64_t* out_levels)
{
    return guarded([&] {
        need(op && out_levels);
        const Shape& lv = operator_levels(*op->h.dev);
        for (size_t a = 0; a < lv.size(); ++a)
            out_levels[a] = lv[a];
    });
}

ts_status ts_operator_kernel_elems(const ts_operator* op, uint64_t* out)
{
    return guarded([&] {
        need(op && out);
        *out = operator_kernel_elems(*op->h.dev);
    });
}

ts_status ts_operator_save_kernel(const ts_operator* op, const char* path)
{
    return guarded([&] {
        need(op && path);
        save_kernel(*op->h.dev, path);
    });
}

ts_status ts_operator_load_split(const char* path, ts_operator** out)
{
    return guarded([&] {
        need(path && out);
        auto dev = load_split(path);
        *out = new ts_operator{OperatorHandle{std::move(dev)}};
    });
}

void ts_operator_destroy(ts_operator* op) { delete op; }

ts_status ts_naive_matvec(const ts_generator* g, const double* v, double* y, int64_t cap)
{
    return guarded([&] {
        need(g && v && y);
        auto in = from_interleaved(v, volume(g->g.levels));
        auto out = naive_matvec(g->g, in.data(), cap);
        std::memcpy(y, out.data(), out.size() * sizeof(cplx));
    });
}

ts_status ts_predict(int32_t d, double n, ts_complexity* out)
{
    return guarded([&] {
        need(out != nullptr, "null out pointer");
        *out = predict(d, n);
    });
}

// ---------------------------------------------------------------- extensions

ts_status ts_block_generator_create(int32_t d, const int64_t* levels, int32_t m,
                                    int32_t n_unique, const int32_t* comp_map,
                                    const double* const* lags, const int32_t* axis_sign,
                                    ts_block_generator** out)
{
    return guarded([&] {
        need(out && comp_map && lags && axis_sign);
        Shape lv = check_levels(d, levels);
        if (m < 1 || m > TSK_MAX_M)
            fail(TS_ERR_INVALID_ARGUMENT, "block arity m must be in [1, 4]");
        if (n_unique < 1 || n_unique > 16)
            fail(TS_ERR_INVALID_ARGUMENT, "n_unique must be in [1, 16]");
        BlockGenerator b;
        b.levels = lv;
        b.m = m;
        b.n_unique = n_unique;
        std::vector<bool> used(static_cast<size_t>(n_unique), false);
        for (int i = 0; i < m * m; ++i) {
            if (comp_map[i] < 0 || comp_map[i] >= n_unique)
                fail(TS_ERR_INVALID_ARGUMENT, "component map entry out of range");
            used[comp_map[i]] = true;
            b.comp_map.push_back(comp_map[i]);
        }
        int64_t count = 1;
        for (auto n : lv)
            count *= 2 * n - 1;
        for (int u = 0; u < n_unique; ++u) {
            std::vector<int> sg;
            for (int a = 0; a < d; ++a) {
                const int v = axis_sign[u * d + a];
                if (v < -1 || v > 1)
                    fail(TS_ERR_INVALID_ARGUMENT, "axis sign must be -1, 0 or +1");
                sg.push_back(v);
                b.axis_sign.push_back(v);
            }
            auto l = from_interleaved(lags[u], count);
            validate_symmetry(lv, l, sg);
            b.lags.push_back(std::move(l));
        }
        *out = new ts_block_generator{std::move(b)};
    });
}

ts_status ts_block_generator_dyadic(int32_t d, const int64_t* levels, double k, double self_re,
                                    double self_im, ts_block_generator** out)
{
    return guarded([&] {
        need(out != nullptr, "null out pointer");
        auto b = block_dyadic(check_levels(d, levels), k, cplx{self_re, self_im});
        *out = new ts_block_generator{std::move(b)};
    });
}

ts_status ts_generator_get_lags(const ts_generator* g, double* out)
{
    return guarded([&] {
        need(g && out);
        std::memcpy(static_cast<void*>(out), g->g.lags.data(), g->g.lags.size() * sizeof(cplx));
    });
}

ts_status ts_block_generator_from_scalar(const ts_generator* g, ts_block_generator** out)
{
    return guarded([&] {
        need(g && out);
        *out = new ts_block_generator{block_from_scalar(g->g)};
    });
}

int32_t ts_block_generator_components(const ts_block_generator* g) { return g ? g->g.m : 0; }

void ts_block_generator_destroy(ts_block_generator* g) { delete g; }

void ts_split_options_default(ts_split_options* opt)
{
    if (!opt)
        return;
    opt->precision = TS_PREC_C128;
    opt->storage = TS_STORAGE_AUTO;
    opt->device = -1;
    opt->part = 0;
    opt->nparts = 1;
    opt->s0_re = 0.0;
    opt->s0_im = 0.0;
}

ts_status ts_operator_create_split_ex(const ts_block_generator* g, const ts_split_options* opt,
                                      ts_operator** out)
{
    return guarded([&] {
        need(g && out);
        ts_split_options o;
        ts_split_options_default(&o);
        if (opt)
            o = *opt;
        auto dev = create_split(g->g, o);
        *out = new ts_operator{OperatorHandle{std::move(dev)}};
    });
}

ts_status ts_operator_create_embed_ex(const ts_block_generator* g, const ts_split_options* opt,
                                      ts_operator** out)
{
    return guarded([&] {
        need(g && out);
        ts_split_options o;
        ts_split_options_default(&o);
        if (opt)
            o = *opt;
        auto dev = create_embed_block(g->g, o);
        *out = new ts_operator{OperatorHandle{std::move(dev)}};
    });
}

ts_status ts_operator_apply_device(const ts_operator* op, const void* x, void* y, void* stream,
                                   ts_metrics* metrics)
{
    return guarded([&] {
        need(op != nullptr);
        apply_device(*op->h.dev, x, y, stream, metrics);
    });
}

ts_status ts_operator_apply_batch_device(const ts_operator* op, const void* x, void* y, int64_t nrhs,
                                         void* stream, ts_metrics* metrics)
{
    return guarded([&] {
        need(op != nullptr);
        apply_batch_device(*op->h.dev, x, y, nrhs, stream, metrics);
    });
}

ts_status ts_operator_get_info(const ts_operator* op, ts_operator_info* out)
{
    return guarded([&] {
        need(op && out);
        operator_info(*op->h.dev, out);
    });
}

ts_status ts_operator_profile_device(const ts_operator* op, const void* x, void* y, void* stream,
                                     ts_launch_record* out, int32_t cap, int32_t* count)
{
    return guarded([&] {
        need(op && count);
        auto recs = profile_device(*op->h.dev, x, y, stream);
        const int32_t n = static_cast<int32_t>(recs.size());
        for (int32_t i = 0; i < n && i < cap && out; ++i)
            out[i] = recs[i];
        *count = n;
    });
}

int32_t ts_device_count(void) { return device_count(); }

ts_status ts_device_memory_stats(int32_t device, ts_memory_stats* out)
{
    return guarded([&] {
        need(out != nullptr);
        if (device < 0 || device >= device_count())
            fail(TS_ERR_INVALID_ARGUMENT, "invalid device ordinal");
        meter_stats(device, out);
    });
}

ts_status ts_device_memory_reset_peak(int32_t device)
{
    return guarded([&] {
        if (device < 0 || device >= device_count())
            fail(TS_ERR_INVALID_ARGUMENT, "invalid device ordinal");
        meter_reset_peak(device);
    });
}

ts_status ts_operator_create_split_multi(const ts_block_generator* g, const ts_split_options* opt,
                                         int32_t ndev, const int32_t* devices, ts_operator** out)
{
    return guarded([&] {
        need(g && out && devices && ndev > 0);
        ts_split_options o;
        ts_split_options_default(&o);
        if (opt)
            o = *opt;
        auto dev = create_split_multi(g->g, o, std::vector<int>(devices, devices + ndev));
        *out = new ts_operator{OperatorHandle{std::move(dev)}};
    });
}

ts_status ts_comm_unique_id(unsigned char out[128])
{
    return guarded([&] {
        need(out != nullptr);
        comm_unique_id(out);
    });
}

ts_status ts_comm_create(const unsigned char id[128], int32_t nranks, int32_t rank, int32_t device,
                         ts_comm** out)
{
    return guarded([&] {
        need(id && out);
        if (device < 0 || device >= device_count())
            fail(TS_ERR_INVALID_ARGUMENT, "invalid device ordinal");
        *out = reinterpret_cast<ts_comm*>(comm_create(id, nranks, rank, device));
    });
}

void ts_comm_destroy(ts_comm* comm) { comm_destroy(reinterpret_cast<Comm*>(comm)); }

ts_status ts_operator_apply_device_comm(const ts_operator* op, ts_comm* comm, const void* x, void* y,
                                        int32_t root, int32_t bcast_x, void* stream, ts_metrics* metrics)
{
    return guarded([&] {
        need(op && comm);
        apply_device_comm(*op->h.dev, reinterpret_cast<Comm*>(comm), x, y, root, bcast_x,
                          static_cast<cudaStream_t>(stream), metrics);
    });
}

}  // extern "C"
