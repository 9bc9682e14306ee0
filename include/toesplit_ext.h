/*
 * toesplit_ext.h — additive B200 extensions to the toesplit C ABI.
 *
 * Nothing here changes toesplit.h (the reference ABI, ref
 * proj/include/toesplit.h); these are new symbols for what BASELINE.json's
 * configs need and the reference lacks (SURVEY.md §0 "gaps", §8(b)):
 *   - complex64 operators (complex128 remains the default),
 *   - m x m blocks (e.g. 3x3 dyadic Green tensors) with a unique-component
 *     map, so a block-symmetric G stores 6 of its 9 components,
 *   - per-axis symmetry signs, generalising ref generator.hpp:9's single mode
 *     (the off-diagonal dyadic G_ij is odd along axes i and j, even along the
 *     third),
 *   - device-pointer apply on a caller stream (no PCIe in the loop),
 *   - branch partitions: an operator that owns the subtree of branch ids whose
 *     low q bits equal `part` (nparts = 2^q) and returns that subtree's
 *     projected partial output; summing the partials over parts (an NCCL
 *     reduce across GPUs) gives y (paper outlook).
 *
 * Vector layout for m-component operators: m component tensors back to back
 * (SoA), each prod(levels) complex elements, row-major, level 1 outermost.
 * ts_operator_apply on an m-component operator reads/writes m*prod(levels)
 * interleaved complex doubles in that layout.
 */
#ifndef TOESPLIT_EXT_H
#define TOESPLIT_EXT_H

#include "toesplit.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ts_precision {
    TS_PREC_C128 = 0, /* complex<double>, the reference's only precision */
    TS_PREC_C64 = 1   /* complex<float> storage and arithmetic; spectra and
                         twiddles are computed in double and rounded */
} ts_precision;

typedef struct ts_block_generator ts_block_generator;

/* Explicit m x m block generator. comp_map[i*m+j] in [0, n_unique) names the
 * unique component used at block position (i, j); lags[u] is that component's
 * interleaved lag tensor (as ts_generator_create); axis_sign[u*d + a] is +1
 * (t_m == t_{-m} under negation of lag a), -1 (t_m == -t_{-m}) or 0 (no
 * symmetry), validated exactly like ref generator.cpp:38-62. */
ts_status ts_block_generator_create(int32_t d, const int64_t* levels, int32_t m,
                                    int32_t n_unique, const int32_t* comp_map,
                                    const double* const* lags, const int32_t* axis_sign,
                                    ts_block_generator** out);

/* The synthetic dyadic Green kernel of BASELINE.json configs[1..3] (d = 3,
 * m = 3, 6 unique components, per-axis parity (-1)^([i=a]+[j=a])):
 * G_ij(r) = (d_ij - rh_i rh_j) e^{ikr}/r + (d_ij - 3 rh_i rh_j) e^{ikr}/(k^2 r^3),
 * G(0) = (self_re + i self_im) I, on unit-spaced integer offsets. Lags are
 * evaluated analytically on the device at operator creation (never
 * materialised on the host). */
ts_status ts_block_generator_dyadic(int32_t d, const int64_t* levels, double k, double self_re,
                                    double self_im, ts_block_generator** out);

/* Copy a scalar generator's lag tensor (interleaved, prod(2 n_l - 1) complex)
 * into out — the reference ABI has no lag getter. */
ts_status ts_generator_get_lags(const ts_generator* g, double* out);

/* Wrap a scalar generator (m = 1); per-axis signs from its symmetry mode. */
ts_status ts_block_generator_from_scalar(const ts_generator* g, ts_block_generator** out);

int32_t ts_block_generator_components(const ts_block_generator* g);
void ts_block_generator_destroy(ts_block_generator* g);

typedef struct ts_split_options {
    int32_t precision; /* ts_precision */
    int32_t storage;   /* ts_storage */
    int32_t device;    /* CUDA ordinal, -1 = current */
    int32_t part;      /* owned branch subtree, 0 <= part < nparts */
    int32_t nparts;    /* 1, 2, 4, ... <= 2^d */
    double s0_re;      /* circulant padding value (result never depends on it) */
    double s0_im;
} ts_split_options;

/* Fill *opt with defaults: c128, AUTO, current device, part 0 of 1, s0 = 0. */
void ts_split_options_default(ts_split_options* opt);

ts_status ts_operator_create_split_ex(const ts_block_generator* g, const ts_split_options* opt,
                                      ts_operator** out);

/* The full circulant-embedding operator (ref engine_embed.cpp:61-168, the
 * method the paper improves on) for block generators, on this library's own
 * FFT passes: opt->precision (c64 / c128), opt->storage (AUTO: the (n+1)^d
 * mirror corner of each unique component's (2n)^d symbol when every component
 * has a sign on every axis and skew padding is zero), opt->device, opt->s0;
 * part / nparts are ignored. Applies like a split operator (ts_operator_apply,
 * _apply_device, _apply_batch_device). */
ts_status ts_operator_create_embed_ex(const ts_block_generator* g, const ts_split_options* opt,
                                      ts_operator** out);

/* y = T x on device memory: x, y hold m components of prod(levels) elements of
 * the operator's precision (float2 / double2), 16-byte aligned (else
 * TS_ERR_INVALID_ARGUMENT), may not alias; stream is a
 * cudaStream_t (NULL = legacy default stream). Asynchronous: returns after
 * enqueueing; metrics (nullable) carries counters, apply_ns = 0. Workspace is
 * stream-ordered per call, so concurrent calls on different streams are safe.
 * For a partition operator y receives the partial output of its subtree. */
ts_status ts_operator_apply_device(const ts_operator* op, const void* x, void* y, void* stream,
                                   ts_metrics* metrics);

/* nrhs right-hand sides in one call (an iterative solver's block of vectors):
 * x and y hold nrhs vectors back to back, each laid out as for
 * ts_operator_apply_device; same stream semantics. Counters in metrics are
 * summed over the vectors. */
ts_status ts_operator_apply_batch_device(const ts_operator* op, const void* x, void* y, int64_t nrhs,
                                         void* stream, ts_metrics* metrics);

typedef struct ts_operator_info {
    int32_t d;
    int32_t m;          /* vector components / block arity */
    int32_t n_unique;   /* stored components */
    int32_t precision;  /* ts_precision */
    int32_t storage;    /* resolved ts_storage (FULL or COMPRESSED) */
    int32_t is_embed;   /* 1 for full-embedding baseline operators */
    int32_t device;
    int32_t part;
    int32_t nparts;
    int32_t reserved;
    uint64_t elem_bytes;       /* 8 (c64) or 16 (c128) */
    uint64_t spectra_bytes;    /* device bytes of stored spectra */
    uint64_t workspace_bytes;  /* device working set of one apply_device call */
    uint64_t launches;         /* kernels per apply_device call */
    uint64_t table_bytes;      /* device bytes of twiddle / phase tables */
    uint64_t cached_bytes;     /* device bytes held by the operator's apply contexts
                                  (workspace kept across calls, host-path buffers) */
    uint64_t graph_replays;    /* applies served by a captured CUDA graph */
    int32_t ndevices;          /* 1, or P for a multi-GPU operator */
    int32_t reserved2;
} ts_operator_info;

ts_status ts_operator_get_info(const ts_operator* op, ts_operator_info* out);

/* One kernel launch of an apply, timed with CUDA events on the apply stream. */
typedef struct ts_launch_record {
    int32_t kind;          /* 1 = K1 fwd_split, 2 = K2 leaf_pair, 3 = K3 inv_merge,
                              4 = embed-engine pass */
    int32_t axis;
    int32_t single_child;  /* 1 for the partition path variants K1'/K2'/K3' */
    int32_t reserved;
    double ms;             /* device time of this launch */
    uint64_t alg_bytes;    /* algorithmic HBM bytes of this launch (SURVEY.md §8(d)
                              per-level pass model: vectors + spectra read once) */
} ts_launch_record;

/* As ts_operator_apply_device, with an event pair around every launch;
 * synchronizes the stream, then fills out[0..min(cap, launches)) and *count.
 * For profiling/bench only (events add a few microseconds per launch). */
ts_status ts_operator_profile_device(const ts_operator* op, const void* x, void* y, void* stream,
                                     ts_launch_record* out, int32_t cap, int32_t* count);

/* Number of visible CUDA devices (0 when none); never fails. */
int32_t ts_device_count(void);

/* Device-memory meter (the reference's AllocationMeter, ref
 * proj/src/core/tensor.cpp:49-66, for device bytes): every device buffer the
 * library allocates on `device` — spectra, tables, apply workspaces, staging —
 * counted live, by kind, with a high-water mark since the last reset.
 * Caller-owned buffers (x, y of apply_device) are not included. */
typedef struct ts_memory_stats {
    uint64_t live_bytes;
    uint64_t peak_bytes;
    uint64_t spectra_bytes;
    uint64_t table_bytes;
    uint64_t workspace_bytes;
    uint64_t staging_bytes;
} ts_memory_stats;

ts_status ts_device_memory_stats(int32_t device, ts_memory_stats* out);
/* peak := live */
ts_status ts_device_memory_reset_peak(int32_t device);

/* ---- multi-GPU: the 2^d branches partitioned over P = 2^q GPUs -----------
 * (the paper's outlook PAPER.md:97-99). GPU g owns the branch
 * ids whose low q bits equal g, stores only their spectra, runs q single-child
 * path levels, its subtree and q single-child inverse levels; the projected
 * partial outputs are summed by one NCCL reduce over NVLink, component by
 * component as the last inverse-merge pass finishes each (reduce of
 * component c overlaps the pass of component c+1). NCCL is loaded at run time
 * (libnccl.so.2); without it these calls fail with TS_ERR_RESOURCE. */

/* One process driving P GPUs. devices[0..ndev) (ndev a power of two <= 2^d,
 * distinct ordinals) receive parts 0..ndev-1; opt->part / opt->nparts /
 * opt->device are ignored. ts_operator_apply and ts_operator_apply_device
 * (x, y on devices[0], stream on devices[0]) then compute the whole product:
 * x is broadcast from devices[0], partials are reduced onto devices[0]. */
ts_status ts_operator_create_split_multi(const ts_block_generator* g, const ts_split_options* opt,
                                         int32_t ndev, const int32_t* devices, ts_operator** out);

/* One process per GPU (torchrun style): an NCCL communicator the library
 * owns. Rank 0 calls ts_comm_unique_id, ships the 128 bytes to the other
 * ranks out of band, and every rank calls ts_comm_create (collective). */
typedef struct ts_comm ts_comm;
ts_status ts_comm_unique_id(unsigned char out[128]);
ts_status ts_comm_create(const unsigned char id[128], int32_t nranks, int32_t rank, int32_t device,
                         ts_comm** out);
void ts_comm_destroy(ts_comm* comm);

/* Collective apply of a partition operator (part == rank, nparts == nranks,
 * created on the communicator's device). bcast_x != 0: x is valid on root
 * only and is broadcast into every rank's x buffer first; otherwise every
 * rank holds x. On root y receives the whole product, elsewhere y holds the
 * rank's partial (scratch). Asynchronous on stream like apply_device. */
ts_status ts_operator_apply_device_comm(const ts_operator* op, ts_comm* comm, const void* x, void* y,
                                        int32_t root, int32_t bcast_x, void* stream,
                                        ts_metrics* metrics);

#ifdef __cplusplus
}
#endif

#endif /* TOESPLIT_EXT_H */
