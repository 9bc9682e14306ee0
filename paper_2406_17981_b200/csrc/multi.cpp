// Several GPUs for one split operator (the paper's outlook
// the reference itself is single-process CPU code).
//
// Partition: GPU g of P = 2^q owns the branch ids whose low q bits equal g
// (the axes split first), stores only those spectra and runs q single-child
// forward passes (K1'), its subtree, and q single-child inverse passes (K3');
// y = sum_g partial_g. Data movement is NCCL over NVLink / NVSwitch:
//   * x is broadcast from the root GPU (ncclBroadcast, in place on the root);
//   * the root-level inverse pass is launched per component vector and the
//     ncclReduce of component c (2 s reals, sum, in place on the root) runs on
//     a second stream as soon as that component's pass is done, overlapping
//     the pass over component c+1.
// Two drivers share this: one process driving P GPUs (ncclCommInitAll; the
// operator behaves like a single-GPU one to its caller) and one process per
// GPU (ts_comm: ncclCommInitRank, the torchrun layout).
//
// NCCL is dlopen'ed (libnccl.so.2; torch's copy when torch loaded it first),
// so the library carries no link-time NCCL dependency and loads on hosts
// without it; the multi-GPU calls then fail with TS_ERR_RESOURCE.
#include "multi.hpp"

#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only (resolved through dlsym)

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace tsb {

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclReduce) reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl()
{
    static const NcclApi api = [] {
        NcclApi a;
        void* h = nullptr;
        // TSK_NCCL_LIB: another implementation of these entry points (the tests'
        // single-process stand-in, tests/nccl_mock)
        if (const char* alt = getenv("TSK_NCCL_LIB"); alt && *alt)
            h = dlopen(alt, RTLD_NOW | RTLD_LOCAL);
        else
            for (const char* name : {"libnccl.so.2", "libnccl.so"})
                if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL)))
                    break;
        if (!h) {
            const char* e = dlerror();
            a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return a;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && a.why.empty())
                a.why = std::string("libnccl lacks ") + name;
        };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.init_rank, "ncclCommInitRank");
        sym(a.init_all, "ncclCommInitAll");
        sym(a.destroy, "ncclCommDestroy");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.reduce, "ncclReduce");
        sym(a.error_string, "ncclGetErrorString");
        a.ok = a.why.empty();
        return a;
    }();
    if (!api.ok)
        fail(TS_ERR_RESOURCE, "NCCL unavailable: " + api.why);
    return api;
}

void nccl_check(ncclResult_t r, const char* what)
{
    if (r == ncclSuccess)
        return;
    const char* s = nccl().error_string ? nccl().error_string(r) : "?";
    fail(r == ncclSystemError || r == ncclUnhandledCudaError ? TS_ERR_RESOURCE : TS_ERR_INTERNAL,
         std::string(what) + ": " + s);
}

ncclDataType_t real_type(const DeviceOperator& op) { return op.prec ? ncclFloat : ncclDouble; }

// Restores the caller's current device whatever the body switched to.
struct KeepDevice {
    int dev = -1;
    KeepDevice() { cudaGetDevice(&dev); }
    ~KeepDevice()
    {
        if (dev >= 0)
            cudaSetDevice(dev);
    }
};

cudaEvent_t new_event()
{
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    return e;
}

}  // namespace

// ---------------------------------------------------------------- one process, P GPUs

struct MultiGpu {
    std::vector<int> devices;
    std::vector<std::shared_ptr<DeviceOperator>> parts;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> cst, nst;  // per GPU: compute / reduce stream
    std::vector<DevBuf> xb, yb;           // per GPU g > 0: replicated x, partial y
    std::vector<std::vector<cudaEvent_t>> comp;  // per GPU, per component: root pass done
    std::vector<cudaEvent_t> done;        // per GPU: reduce done
    cudaEvent_t in_ev = nullptr;
    std::mutex mu;
    int64_t last_peak = 0;

    ~MultiGpu()
    {
        KeepDevice keep;
        for (size_t g = 0; g < devices.size(); ++g) {
            cudaSetDevice(devices[g]);
            if (g < cst.size() && cst[g])
                cudaStreamSynchronize(cst[g]);
            if (g < nst.size() && nst[g])
                cudaStreamSynchronize(nst[g]);
        }
        if (!comms.empty() && nccl().destroy)
            for (auto c : comms)
                if (c)
                    nccl().destroy(c);
        for (size_t g = 0; g < devices.size(); ++g) {
            cudaSetDevice(devices[g]);
            if (g < comp.size())
                for (auto e : comp[g])
                    cudaEventDestroy(e);
            if (g < done.size() && done[g])
                cudaEventDestroy(done[g]);
            if (g < cst.size() && cst[g])
                cudaStreamDestroy(cst[g]);
            if (g < nst.size() && nst[g])
                cudaStreamDestroy(nst[g]);
            if (g < xb.size())
                xb[g].reset();
            if (g < yb.size())
                yb[g].reset();
        }
        if (in_ev) {
            cudaSetDevice(devices[0]);
            cudaEventDestroy(in_ev);
        }
    }
};

std::shared_ptr<DeviceOperator> create_split_multi(const BlockGenerator& g, const ts_split_options& opt,
                                                   const std::vector<int>& devices)
{
    const int P = static_cast<int>(devices.size());
    const int d = static_cast<int>(g.levels.size());
    if (P < 1 || (P & (P - 1)) != 0 || P > (1 << std::min(d, 30)))
        fail(TS_ERR_INVALID_ARGUMENT, "device count must be a power of two <= 2^d");
    const int ndev = device_count();
    for (int i = 0; i < P; ++i) {
        if (devices[i] < 0 || devices[i] >= ndev)
            fail(TS_ERR_INVALID_ARGUMENT, "invalid device ordinal " + std::to_string(devices[i]));
        // (TSK_ALLOW_SHARED_DEVICE=1 lets tests place several parts on one
        // GPU under the single-process NCCL stand-in; real NCCL refuses it)
        static const bool shared_ok = [] {
            const char* e = getenv("TSK_ALLOW_SHARED_DEVICE");
            return e && e[0] == '1';
        }();
        for (int j = 0; j < i && !shared_ok; ++j)
            if (devices[j] == devices[i])
                fail(TS_ERR_INVALID_ARGUMENT, "device ordinals must be distinct (one part per GPU)");
    }
    const NcclApi& api = nccl();
    KeepDevice keep;
    auto mg = std::make_shared<MultiGpu>();
    mg->devices = devices;
    for (int p = 0; p < P; ++p) {
        ts_split_options o = opt;
        o.part = p;
        o.nparts = P;
        o.device = devices[p];
        mg->parts.push_back(create_split(g, o));
    }
    const auto& p0 = *mg->parts[0];
    mg->comms.assign(P, nullptr);
    nccl_check(api.init_all(mg->comms.data(), P, devices.data()), "ncclCommInitAll");
    mg->cst.assign(P, nullptr);
    mg->nst.assign(P, nullptr);
    mg->xb.resize(P);
    mg->yb.resize(P);
    mg->comp.resize(P);
    mg->done.assign(P, nullptr);
    for (int p = 0; p < P; ++p) {
        cuda_check(cudaSetDevice(devices[p]), "cudaSetDevice");
        cuda_check(cudaStreamCreateWithFlags(&mg->cst[p], cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&mg->nst[p], cudaStreamNonBlocking), "stream");
        if (p > 0) {
            mg->xb[p] = DevBuf(p0.vec_bytes(), MEM_WORK);
            mg->yb[p] = DevBuf(p0.vec_bytes(), MEM_WORK);
        }
        for (int c = 0; c < p0.m; ++c)
            mg->comp[p].push_back(new_event());
        mg->done[p] = new_event();
    }
    cuda_check(cudaSetDevice(devices[0]), "cudaSetDevice");
    mg->in_ev = new_event();

    // the caller-facing operator: whole-tree shape, no spectra of its own
    auto top = std::make_shared<DeviceOperator>();
    top->device = devices[0];
    top->levels = p0.levels;
    top->d = p0.d;
    top->s = p0.s;
    top->m = p0.m;
    top->n_unique = p0.n_unique;
    top->comp_map = p0.comp_map;
    top->skew_mask = p0.skew_mask;
    top->axis_sign = p0.axis_sign;
    top->prec = p0.prec;
    top->compressed = p0.compressed;
    top->tskf_symmetry = p0.tskf_symmetry;
    top->branch_base = p0.branch_base;
    top->block_elems = p0.block_elems;
    for (auto& p : mg->parts) {
        top->spectra_elems += p->spectra_elems;
        top->precompute_ns = std::max(top->precompute_ns, p->precompute_ns);
    }
    top->multi = mg;
    return top;
}

static int64_t multi_one(const DeviceOperator& op, MultiGpu& mg, const void* x, void* y, cudaStream_t st)
{
    const NcclApi& api = nccl();
    const int P = static_cast<int>(mg.devices.size());
    const size_t cnt = 2 * static_cast<size_t>(op.s) * static_cast<size_t>(op.m);  // reals
    const size_t cbytes = static_cast<size_t>(op.s) * op.es();                   // one component
    const ncclDataType_t ty = real_type(op);
    // x ready / y free on the caller's stream
    cuda_check(cudaSetDevice(mg.devices[0]), "cudaSetDevice");
    cuda_check(cudaEventRecord(mg.in_ev, st), "event");
    for (int p = 0; p < P; ++p) {
        cuda_check(cudaSetDevice(mg.devices[p]), "cudaSetDevice");
        cuda_check(cudaStreamWaitEvent(mg.cst[p], mg.in_ev, 0), "wait");
    }
    nccl_check(api.group_start(), "ncclGroupStart");
    for (int p = 0; p < P; ++p) {
        void* dst = p == 0 ? const_cast<void*>(x) : mg.xb[p].p;
        nccl_check(api.broadcast(p == 0 ? x : dst, dst, cnt, ty, 0, mg.comms[p], mg.cst[p]), "ncclBroadcast");
    }
    nccl_check(api.group_end(), "ncclGroupEnd");
    int64_t peak = 0;
    for (int p = 0; p < P; ++p) {
        cuda_check(cudaSetDevice(mg.devices[p]), "cudaSetDevice");
        const DeviceOperator& part = *mg.parts[p];
        CtxLease lease(part, mg.cst[p], false, 1);
        const void* xp = p == 0 ? x : mg.xb[p].p;
        void* yp = p == 0 ? y : mg.yb[p].p;
        auto hook = [&, p](int64_t c) {
            cuda_check(cudaEventRecord(mg.comp[p][c], mg.cst[p]), "event");
        };
        peak = std::max(peak, enqueue_apply_hooked(part, lease.c, xp, yp, 1, hook));
    }
    for (int c = 0; c < op.m; ++c) {
        for (int p = 0; p < P; ++p) {
            cuda_check(cudaSetDevice(mg.devices[p]), "cudaSetDevice");
            cuda_check(cudaStreamWaitEvent(mg.nst[p], mg.comp[p][c], 0), "wait");
        }
        nccl_check(api.group_start(), "ncclGroupStart");
        for (int p = 0; p < P; ++p) {
            char* src = static_cast<char*>(p == 0 ? y : mg.yb[p].p) + c * cbytes;
            char* dst = static_cast<char*>(y) + c * cbytes;
            nccl_check(api.reduce(src, p == 0 ? dst : src, cnt / op.m, ty, ncclSum, 0, mg.comms[p], mg.nst[p]),
                       "ncclReduce");
        }
        nccl_check(api.group_end(), "ncclGroupEnd");
    }
    for (int p = 0; p < P; ++p) {
        cuda_check(cudaSetDevice(mg.devices[p]), "cudaSetDevice");
        cuda_check(cudaEventRecord(mg.done[p], mg.nst[p]), "event");
        // the next call's broadcast / compute on this GPU waits for the reduce
        cuda_check(cudaStreamWaitEvent(mg.cst[p], mg.done[p], 0), "wait");
    }
    cuda_check(cudaSetDevice(mg.devices[0]), "cudaSetDevice");
    cuda_check(cudaStreamWaitEvent(st, mg.done[0], 0), "wait");
    return peak;
}

void multi_apply_device(const DeviceOperator& op, const void* x, void* y, int64_t nrhs, cudaStream_t st,
                        ts_metrics* metrics)
{
    MultiGpu& mg = *op.multi;
    std::lock_guard<std::mutex> lk(mg.mu);
    KeepDevice keep;
    int64_t peak = 0;
    for (int64_t r = 0; r < nrhs; ++r)
        peak = multi_one(op, mg, static_cast<const char*>(x) + op.vec_bytes() * r,
                         static_cast<char*>(y) + op.vec_bytes() * r, st);
    mg.last_peak = peak;
    if (metrics) {
        fill_counters(op, metrics, peak);  // whole-tree counts; peak per GPU
        const uint64_t k = static_cast<uint64_t>(nrhs);
        metrics->fft_forward *= k;
        metrics->fft_inverse *= k;
        metrics->diag_mults *= k;
        metrics->phase_mults *= k;
    }
}

void multi_info(const DeviceOperator& op, ts_operator_info* r)
{
    const MultiGpu& mg = *op.multi;
    r->ndevices = static_cast<int32_t>(mg.devices.size());
    r->nparts = r->ndevices;
    r->part = -1;
    r->table_bytes = 0;
    r->cached_bytes = 0;
    r->spectra_bytes = op.spectra_elems * op.es();
    r->workspace_bytes = 0;
    r->graph_replays = 0;
    for (const auto& p : mg.parts) {
        ts_operator_info pi{};
        operator_info(*p, &pi);
        r->table_bytes += pi.table_bytes;
        r->cached_bytes += pi.cached_bytes;
        r->workspace_bytes = std::max(r->workspace_bytes, pi.workspace_bytes);
        r->launches = std::max<uint64_t>(r->launches, pi.launches + static_cast<uint64_t>(op.m) - 1);
    }
    for (size_t g = 1; g < mg.xb.size(); ++g)
        r->cached_bytes += mg.xb[g].bytes + mg.yb[g].bytes;
}

// ---------------------------------------------------------------- one process per GPU

struct Comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    cudaStream_t nst = nullptr;
    std::vector<cudaEvent_t> comp;
    cudaEvent_t done = nullptr;
    std::mutex mu;
};

void comm_unique_id(unsigned char out[128])
{
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof id);
}

Comm* comm_create(const unsigned char idb[128], int nranks, int rank, int device)
{
    if (nranks < 1 || rank < 0 || rank >= nranks)
        fail(TS_ERR_INVALID_ARGUMENT, "0 <= rank < nranks required");
    const NcclApi& api = nccl();
    KeepDevice keep;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto c = std::make_unique<Comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId id;
    std::memcpy(&id, idb, sizeof id);
    nccl_check(api.init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank");
    cuda_check(cudaStreamCreateWithFlags(&c->nst, cudaStreamNonBlocking), "stream");
    c->done = new_event();
    return c.release();
}

void comm_destroy(Comm* c)
{
    if (!c)
        return;
    KeepDevice keep;
    cudaSetDevice(c->device);
    if (c->nst)
        cudaStreamSynchronize(c->nst);
    if (c->comm && nccl().destroy)
        nccl().destroy(c->comm);
    for (auto e : c->comp)
        cudaEventDestroy(e);
    if (c->done)
        cudaEventDestroy(c->done);
    if (c->nst)
        cudaStreamDestroy(c->nst);
    delete c;
}

void apply_device_comm(const DeviceOperator& op, Comm* comm, const void* x, void* y, int root, int bcast_x,
                       cudaStream_t st, ts_metrics* metrics)
{
    if (!comm)
        fail(TS_ERR_INVALID_ARGUMENT, "null communicator");
    if (op.multi || op.is_embed)
        fail(TS_ERR_INVALID_ARGUMENT, "collective apply takes a single-GPU partition operator");
    if (op.nparts != comm->nranks || op.part != comm->rank)
        fail(TS_ERR_INVALID_ARGUMENT, "operator partition must be (part = rank, nparts = nranks)");
    if (op.device != comm->device)
        fail(TS_ERR_INVALID_ARGUMENT, "operator and communicator live on different devices");
    if (root < 0 || root >= comm->nranks)
        fail(TS_ERR_INVALID_ARGUMENT, "invalid root rank");
    if (!x || !y || x == y)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must be distinct device buffers");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
        fail(TS_ERR_INVALID_ARGUMENT, "x and y must be 16-byte aligned device pointers");
    const NcclApi& api = nccl();
    std::lock_guard<std::mutex> lk(comm->mu);
    DeviceGuard guard(op.device);
    while (static_cast<int>(comm->comp.size()) < op.m)
        comm->comp.push_back(new_event());
    const size_t creals = 2 * static_cast<size_t>(op.s);
    const size_t cbytes = static_cast<size_t>(op.s) * op.es();
    const ncclDataType_t ty = real_type(op);
    if (bcast_x)
        nccl_check(api.broadcast(x, const_cast<void*>(x), creals * op.m, ty, root, comm->comm, st),
                   "ncclBroadcast");
    CtxLease lease(op, st, false, 1);
    auto hook = [&](int64_t c) {
        cuda_check(cudaEventRecord(comm->comp[c], st), "event");
        cuda_check(cudaStreamWaitEvent(comm->nst, comm->comp[c], 0), "wait");
        char* p = static_cast<char*>(y) + c * cbytes;
        nccl_check(api.reduce(p, p, creals, ty, ncclSum, root, comm->comm, comm->nst), "ncclReduce");
    };
    const int64_t peak = enqueue_apply_hooked(op, lease.c, x, y, 1, hook);
    cuda_check(cudaEventRecord(comm->done, comm->nst), "event");
    cuda_check(cudaStreamWaitEvent(st, comm->done, 0), "wait");
    if (metrics)
        fill_counters(op, metrics, peak);
}

}  // namespace tsb
