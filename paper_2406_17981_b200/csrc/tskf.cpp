// TSKF kernel-spectra files (ref proj/src/core/kernel.cpp:456-537, format
// proj/README.md:158-170): version 1 byte-compatible with the reference for
// scalar complex128 whole-tree operators; version 2 (this library) adds
// precision, the m x m block map, per-component skew masks and the branch
// partition. Spectra are staged through host memory and uploaded to the
// current device on load.
#include <cuda_runtime.h>

#include <bit>
#include <cstring>
#include <fstream>

#include "engine.hpp"

namespace tsb {

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
    if (op.multi)
        fail(TS_ERR_INVALID_ARGUMENT, "save the per-GPU partition operators of a multi-GPU operator");
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
    op->spectra = DevBuf(host.size(), MEM_SPECTRA);
    cuda_check(cudaMemcpy(op->spectra.p, host.data(), host.size(), cudaMemcpyHostToDevice),
               "H2D spectra");
    fill_tables(*op, op->levels, op->tab);
    return op;
}

}  // namespace tsb
