/*
 * tsk_launch.h — the thin extern "C" launcher layer between the C++ host
 * engine (scheduler, operators) and the sm_100a kernels (SURVEY.md §8(b)
 * "internal layering"). Launchers take device pointers, plain shape/stride
 * descriptors and a cudaStream_t (as void*), enqueue one kernel and return
 * the cudaError_t of the launch (as int). No torch types, no C++ types.
 *
 * Kernel families:
 *   K1 tsk_fwd_split  — replaces FftwProvider::forward on entry of a branch
 *                       node + phase_shift_axis child creation
 *                       (ref engine_split.cpp:67-73, fft.cpp:65-87,
 *                       tensor.cpp:227-254): even = F_a(t), odd = F_a(P_a t).
 *   K2 tsk_leaf_pair  — replaces the deepest level: both leaf FFTs, the
 *                       KernelSpectra::multiply_into of both leaves (1x1 or
 *                       m x m across components, full or mirror-compressed,
 *                       ref kernel.cpp:126-219), both inverse FFTs and the
 *                       deepest merge_loop (ref engine_split.cpp:13-37,89).
 *   K3 tsk_inv_merge  — replaces FftwProvider::inverse + its 1/n sweep +
 *                       merge_loop: out = scale * (B_a(e) + conj(P_a) B_a(o)).
 *  Single-child variants (partition path) are the same launchers with one of
 *  use_even / use_odd cleared.
 */
#ifndef TSK_LAUNCH_H
#define TSK_LAUNCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSK_MAX_D 31
#define TSK_MAX_RADICES 24
#define TSK_MAX_UNIQUE 16
#define TSK_MAX_M 4

/* One batched single-axis pass over a tensor viewed as [outer][n][inner],
 * for ncomp component tensors cstride elements apart. */
typedef struct tsk_axis {
    int64_t outer;
    int64_t inner;
    int64_t n;
    int32_t ncomp;
    int32_t prec; /* 0 = c128 (double2), 1 = c64 (float2) */
    int64_t cstride;
    const void* src0; /* K1/K2: input; K3: even child */
    const void* src1; /* K3: odd child */
    void* dst0;       /* K1: even out; K2/K3: output */
    void* dst1;       /* K1: odd out */
    const void* roots; /* n entries exp(-2 pi i k / n), element type of prec */
    const void* phase; /* n entries exp(-i pi k / n) */
    int32_t use_even;
    int32_t use_odd;
    double scale; /* K3/K2 output scale (1/(2n) for a merge) */
    int32_t nrad;
    int32_t rad[TSK_MAX_RADICES];
    /* K2 only: right-hand sides of a batched leaf pass (0 or 1 = one), the
     * ncomp coupled components of RHS r start rstride elements after RHS r-1 */
    int64_t nrhs;
    int64_t rstride;
} tsk_axis;

/* Spectra description for the leaf pass (leaf axis = d-1, inner = 1). */
typedef struct tsk_spectra {
    const void* data;          /* element type of prec */
    int64_t branch_base[2];    /* element offset of the even/odd leaf branch */
    int64_t block_elems[2];    /* elements per unique-component block */
    uint32_t branch_bits[2];   /* branch ids of the even/odd leaf */
    int32_t compressed;
    int32_t d;
    int32_t m;
    int32_t n_unique;
    int64_t levels[TSK_MAX_D];
    uint32_t skew_mask[TSK_MAX_UNIQUE]; /* bit a: component is skew along a */
    int8_t comp_map[TSK_MAX_M * TSK_MAX_M];
} tsk_spectra;

int tsk_fwd_split(const tsk_axis* a, void* stream);
int tsk_inv_merge(const tsk_axis* a, void* stream);
int tsk_leaf_pair(const tsk_axis* a, const tsk_spectra* sp, void* stream);

/* ---- setup / auxiliary kernels ---------------------------------------- */

/* kernel.cpp:50-82 on the device: (2n)^d embedded first column (c128) from
 * a (2n-1)^d lag tensor (c128). */
int tsk_embed_generator(int32_t d, const int64_t* levels, const void* lags, double s0_re,
                        double s0_im, void* out, void* stream);
/* Analytic dyadic G_ij evaluated straight into the embedded layout (c128). */
int tsk_embed_dyadic(int32_t d, const int64_t* levels, int32_t i, int32_t j, double k,
                     double self_re, double self_im, double s0_re, double s0_im, void* out,
                     void* stream);
/* Embedding + first branchwise fold along axis 0 in one sweep (the (2n)^d
 * embedding is never materialised): out (n_0 x 2n_1 x ... x 2n_{d-1}, c128)
 * = lo + hi (odd = 0) or e^{-i pi k/n_0} (lo - hi) (odd = 1). Source: the lag
 * tensor `lags` (as tsk_embed_generator), or with lags == NULL the analytic
 * dyadic G_ij (as tsk_embed_dyadic). Bit-identical to embed + fold_axis. */
int tsk_embed_fold0(int32_t d, const int64_t* levels, const void* lags, int32_t dyadic_i, int32_t dyadic_j,
                    double k, double self_re, double self_im, double s0_re, double s0_im, int32_t odd,
                    void* out, void* stream);
/* kernel.cpp:223-258 fold along `axis` of a tensor of shape `shape` (c128):
 * even = lo + hi, odd = e^{-i pi k/n} (lo - hi); out has shape[axis]/2. */
int tsk_fold_axis(int32_t d, const int64_t* shape, int32_t axis, int32_t odd, const void* in,
                  void* out, void* stream);
/* max over the block of |f|, and of |f(k) - sign_a f(mirror_a(k))| for every
 * axis (ref kernel.cpp:350-366), written as two doubles to out2 (device). */
int tsk_mirror_check(int32_t d, const int64_t* levels, uint32_t branch_bits, uint32_t skew_mask,
                     const void* block, double* out2, void* stream);
/* Gather the stored (mirror-compressed or full) part of a full c128 block
 * into dst with precision prec. */
int tsk_store_block(int32_t d, const int64_t* levels, uint32_t branch_bits, int32_t compressed,
                    const void* block, void* dst, int32_t prec, void* stream);
/* element-wise conversions between c128 and the operator precision */
int tsk_convert(const void* src, int32_t src_prec, void* dst, int32_t dst_prec, int64_t count,
                void* stream);
/* full-embedding engine pieces (ts_operator_create_embed):
 * pad/extract the leading corner of a (2n)^d tensor */
int tsk_embed_corner(int32_t d, const int64_t* levels, int32_t prec, const void* src, void* dst,
                     int32_t extract, void* stream);
/* m x m block symbol of the full-embedding engine: n_unique blocks of
 * block_elems elements (full (2n)^d or (n+1)^d mirror corner), comp_map and
 * per-unique-component skew masks as in tsk_spectra. */
typedef struct tsk_block_symbol {
    const void* data;
    int64_t block_elems;
    int32_t m;
    int32_t n_unique;
    int32_t corner;
    int32_t reserved;
    uint32_t skew_mask[TSK_MAX_UNIQUE];
    int8_t comp_map[TSK_MAX_M * TSK_MAX_M];
} tsk_block_symbol;
/* work_c[(2n)^d] <- sum_c' S_{map(c,c')} work_c' for the m component tensors
 * (cstride elements apart), per frequency; mirrored corner entries take the
 * component's sign per mirrored skew axis (ref engine_embed.cpp:136-147). */
int tsk_block_symbol_multiply(int32_t d, const int64_t* levels, int32_t prec, void* work, int64_t cstride,
                              const tsk_block_symbol* sym, void* stream);
/* work *= symbol, full (2n)^d symbol or (n+1)^d mirror corner with sign */
int tsk_symbol_multiply(int32_t d, const int64_t* levels, int32_t prec, void* work,
                        const void* symbol, int32_t corner, int32_t skew, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TSK_LAUNCH_H */
