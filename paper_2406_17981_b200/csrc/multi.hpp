// Several GPUs for one split operator: the 2^d branches
// partitioned over P = 2^q GPUs, x broadcast and the projected partial
// outputs summed with NCCL over NVLink, the reduce of component c overlapping
// the last inverse-merge pass of component c+1. NCCL is loaded at run time.
#pragma once

#include <cuda_runtime.h>

#include "engine.hpp"

namespace tsb {

std::shared_ptr<DeviceOperator> create_split_multi(const BlockGenerator& g, const ts_split_options& opt,
                                                   const std::vector<int>& devices);
void multi_apply_device(const DeviceOperator& op, const void* x, void* y, int64_t nrhs, cudaStream_t st,
                        ts_metrics* metrics);
void multi_info(const DeviceOperator& op, ts_operator_info* r);

struct Comm;  // one rank of a multi-process communicator
void comm_unique_id(unsigned char out[128]);
Comm* comm_create(const unsigned char id[128], int nranks, int rank, int device);
void comm_destroy(Comm* c);
void apply_device_comm(const DeviceOperator& op, Comm* comm, const void* x, void* y, int root, int bcast_x,
                       cudaStream_t st, ts_metrics* metrics);

}  // namespace tsb
