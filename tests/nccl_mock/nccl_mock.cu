// TEST INFRASTRUCTURE ONLY: a single-process stand-in for the NCCL entry
// points libtoesplit resolves at run time (multi.cpp), so the multi-GPU
// orchestration — partition operators, x broadcast, per-component reduce
// hooks and their stream/event ordering — runs on the one GPU of a test box
// with several "ranks" on the same device (TSK_NCCL_LIB=<this .so>,
// TSK_ALLOW_SHARED_DEVICE=1). Collectives of a group call execute at
// ncclGroupEnd as stream-ordered copies (broadcast) and a summing kernel on
// the root's stream (reduce), each rank's stream waiting for the data it
// reads and the root's result before it may reuse its buffers.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <vector>

struct ncclComm {
    int rank, nranks;
};

namespace {

struct Op {
    int kind;  // 0 broadcast, 1 reduce
    const void* send;
    void* recv;
    size_t count;
    ncclDataType_t ty;
    int root;
    ncclComm* comm;
    cudaStream_t st;
};

int g_depth = 0;
std::vector<Op> g_ops;

size_t esize(ncclDataType_t t) { return t == ncclDouble ? 8 : 4; }

template <typename T>
__global__ void k_acc(T* dst, const T* src, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

cudaEvent_t ev()
{
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
}

ncclResult_t run(std::vector<Op>& ops)
{
    if (ops.empty())
        return ncclSuccess;
    const Op* root = nullptr;
    for (auto& o : ops)
        if (o.comm->rank == o.root)
            root = &o;
    if (!root)
        return ncclInvalidUsage;
    const size_t bytes = root->count * esize(root->ty);
    std::vector<cudaEvent_t> evs;
    if (root->kind == 0) {
        cudaEvent_t r = ev();
        evs.push_back(r);
        cudaEventRecord(r, root->st);
        if (root->recv != root->send)
            cudaMemcpyAsync(root->recv, root->send, bytes, cudaMemcpyDeviceToDevice, root->st);
        for (auto& o : ops) {
            if (&o == root)
                continue;
            cudaStreamWaitEvent(o.st, r, 0);
            cudaMemcpyAsync(o.recv, root->send, bytes, cudaMemcpyDeviceToDevice, o.st);
            cudaEvent_t e = ev();
            evs.push_back(e);
            cudaEventRecord(e, o.st);
            cudaStreamWaitEvent(root->st, e, 0);  // the root's buffer stays until read
        }
    } else {
        for (auto& o : ops) {
            if (&o == root)
                continue;
            cudaEvent_t e = ev();
            evs.push_back(e);
            cudaEventRecord(e, o.st);
            cudaStreamWaitEvent(root->st, e, 0);
        }
        if (root->recv != root->send)
            cudaMemcpyAsync(root->recv, root->send, bytes, cudaMemcpyDeviceToDevice, root->st);
        for (auto& o : ops) {
            if (&o == root)
                continue;
            if (root->ty == ncclDouble)
                k_acc<<<1184, 256, 0, root->st>>>((double*)root->recv, (const double*)o.send, root->count);
            else
                k_acc<<<1184, 256, 0, root->st>>>((float*)root->recv, (const float*)o.send, root->count);
        }
        cudaEvent_t r = ev();
        evs.push_back(r);
        cudaEventRecord(r, root->st);
        for (auto& o : ops)
            if (&o != root)
                cudaStreamWaitEvent(o.st, r, 0);  // send buffers reusable after the sum
    }
    for (auto e : evs)
        cudaEventDestroy(e);  // destruction after the waits were enqueued is safe
    ops.clear();
    return cudaGetLastError() == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

ncclResult_t enqueue(const Op& o)
{
    if (o.ty != ncclFloat && o.ty != ncclDouble)
        return ncclInvalidArgument;
    if (g_depth == 0) {
        std::vector<Op> one{o};
        return run(one);
    }
    g_ops.push_back(o);
    return ncclSuccess;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id)
{
    std::memset(id, 0, sizeof *id);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t*, int, ncclUniqueId, int) { return ncclInvalidUsage; }

ncclResult_t ncclCommInitAll(ncclComm_t* comms, int ndev, const int*)
{
    for (int i = 0; i < ndev; ++i)
        comms[i] = new ncclComm{i, ndev};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm)
{
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart()
{
    ++g_depth;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd()
{
    if (--g_depth > 0)
        return ncclSuccess;
    // one collective per rank per kind, in call order: split by kind
    std::vector<Op> b, r;
    for (auto& o : g_ops)
        (o.kind == 0 ? b : r).push_back(o);
    g_ops.clear();
    ncclResult_t e = run(b);
    return e == ncclSuccess ? run(r) : e;
}

ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t ty, int root,
                           ncclComm_t comm, cudaStream_t st)
{
    return enqueue(Op{0, send, recv, count, ty, root, comm, st});
}

ncclResult_t ncclReduce(const void* send, void* recv, size_t count, ncclDataType_t ty, ncclRedOp_t op, int root,
                        ncclComm_t comm, cudaStream_t st)
{
    if (op != ncclSum)
        return ncclInvalidArgument;
    return enqueue(Op{1, send, recv, count, ty, root, comm, st});
}

const char* ncclGetErrorString(ncclResult_t) { return "nccl mock error"; }

}  // extern "C"
