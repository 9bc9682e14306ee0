// Host-side types of libtoesplit (B200 build). The C ABI (capi.cpp) is a thin
// exception-to-status shell over these; the device engine (engine.cu) owns
// spectra and kernels. Reference counterparts (relative to
// /root/reference/proj): errors.hpp, generator.hpp, instance.hpp,
// engine_split.hpp, engine_embed.hpp, kernel.hpp.
#pragma once

#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "toesplit.h"
#include "toesplit_ext.h"

namespace tsb {

using cplx = std::complex<double>;
using Shape = std::vector<int64_t>;

// One exception type carrying the ABI status (ref errors.hpp:8-30 +
// capi.cpp:43-67 mapping collapsed into the code field).
struct Error : std::runtime_error {
    ts_status code;
    Error(ts_status c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void fail(ts_status c, const std::string& what) { throw Error(c, what); }

int64_t volume(const Shape& s);
Shape check_levels(int32_t d, const int64_t* levels);

// ---- generators -------------------------------------------------------

// ref generator.hpp:9 single symmetry mode; per-axis signs generalise it:
// +1 symmetric, -1 skew, 0 general along that axis.
std::vector<int> signs_for_mode(int d, ts_symmetry mode);

struct Generator {  // ts_generator (ref generator.hpp:20-46)
    Shape levels;
    std::vector<cplx> lags;  // (2n_l - 1)^d
    ts_symmetry symmetry = TS_SYM_GENERAL;
};

Generator make_generator(Shape levels, std::vector<cplx> lags, ts_symmetry sym);
void validate_symmetry(const Shape& levels, const std::vector<cplx>& lags,
                       const std::vector<int>& axis_sign);

struct BlockGenerator {  // ts_block_generator
    Shape levels;
    int m = 1;
    int n_unique = 1;
    std::vector<int> comp_map;             // m*m
    std::vector<std::vector<cplx>> lags;   // per unique component (empty if analytic)
    std::vector<int> axis_sign;            // n_unique * d
    int scalar_symmetry = -1;              // ts_symmetry when wrapping a scalar generator
    bool dyadic = false;
    double k = 0.0;
    cplx self_term{};
    std::vector<std::pair<int, int>> dyadic_ij;  // unique u -> (i, j)
};

BlockGenerator block_from_scalar(const Generator& g);
BlockGenerator block_dyadic(const Shape& levels, double k, cplx self_term);

// ---- seeded instances (ref instance.hpp:11-55, instance.cpp:8-131) ------
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    uint64_t next();
    double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
SplitMix64 seeded_stream(uint64_t seed, uint64_t role);
Generator random_generator(const Shape& levels, uint64_t seed, double variance, ts_symmetry sym);
std::vector<cplx> random_vector(const Shape& levels, uint64_t seed, double variance);
void random_vector_into(const Shape& levels, uint64_t seed, double variance, cplx* out);

// ---- fixtures and oracle-side host services ---------------------------
Generator generator_from_json(const std::string& text);
std::string generator_to_json(const Generator& g);
std::vector<cplx> naive_matvec(const Generator& g, const cplx* v, int64_t cap);
ts_complexity predict(int32_t d, double n);

// ---- device engine ----------------------------------------------------
struct DeviceOperator;  // engine.cu

struct OperatorHandle {
    std::shared_ptr<DeviceOperator> dev;
};

std::shared_ptr<DeviceOperator> create_split(const BlockGenerator& g, const ts_split_options& opt);
std::shared_ptr<DeviceOperator> create_embed(const Generator& g, cplx s0, ts_storage storage);
std::shared_ptr<DeviceOperator> create_embed_block(const BlockGenerator& g, const ts_split_options& opt);
std::shared_ptr<DeviceOperator> load_split(const std::string& path);
void save_kernel(const DeviceOperator& op, const std::string& path);
void apply_host(const DeviceOperator& op, const double* v, double* y, const ts_policy* policy,
                ts_metrics* metrics);
void apply_device(const DeviceOperator& op, const void* x, void* y, void* stream,
                  ts_metrics* metrics);
void apply_batch_device(const DeviceOperator& op, const void* x, void* y, int64_t nrhs, void* stream,
                        ts_metrics* metrics);
std::vector<ts_launch_record> profile_device(const DeviceOperator& op, const void* x, void* y,
                                             void* stream);
const Shape& operator_levels(const DeviceOperator& op);
uint64_t operator_kernel_elems(const DeviceOperator& op);
void operator_info(const DeviceOperator& op, ts_operator_info* out);
int32_t device_count();

}  // namespace tsb

struct ts_generator {
    tsb::Generator g;
};
struct ts_block_generator {
    tsb::BlockGenerator g;
};
struct ts_operator {
    tsb::OperatorHandle h;
};
