/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the split-FFT block-Toeplitz
 * MVM. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it; the product library never links or calls it.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2406.17981,
 * /root/reference/proj), every function citing the reference file:line it
 * follows. Buffers are interleaved (re, im) doubles, row-major, level 1
 * (axis 0) outermost, exactly as proj/include/toesplit.h:8.
 *
 * Parity pin: tests/test_oracle_cpu.py checks this restatement against
 *  - the reference's own known-answer tests (worked 2x2, [1,3,0,2] parity
 *    blocks, symmetric n=2 DFT, spt_brn phase, skew zeros),
 *  - golden vectors in tests/golden/ produced by the UNMODIFIED reference
 *    compiled from its sources (oracle/_ref, FFTW-API shim), and
 *  - that build itself, live, when oracle/_ref/libtoesplit_ref.so exists.
 *
 * Extension beyond the reference (needed by BASELINE.json's dyadic 3x3
 * configs): per-axis symmetry signs. axis_sign[a] = +1 (symmetric along a),
 * -1 (skew along a), 0 (general). The reference's single mode maps to all
 * +1 (TS_SYM_SYMMETRIC), all -1 (TS_SYM_SKEW) or all 0 (TS_SYM_GENERAL).
 */
#ifndef TOESPLIT_ORACLE_H
#define TOESPLIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror ts_status (proj/include/toesplit.h:20-30) */
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ESHAPE = 2, ORC_ESYM = 3, ORC_ECAP = 4, ORC_ERES = 5 };

/* ---- seeded instances (proj/src/core/instance.cpp:8-131) -------------- */
uint64_t orc_splitmix_next(uint64_t* state);
/* lags: (2n_l-1)^d interleaved; symmetry 0 general, 1 symmetric, 2 skew */
int orc_random_lags(int d, const int64_t* levels, uint64_t seed, double variance, int symmetry,
                    double* out_lags);
int orc_random_vector(int d, const int64_t* levels, uint64_t seed, double variance, double* out);

/* Synthetic dyadic Green kernel of BASELINE.json configs[1]: component (i,j)
 * lags, k = wavenumber, self term (self_re + i self_im) * delta_ij. */
int orc_dyadic_lags(int d, const int64_t* levels, int i, int j, double k, double self_re,
                    double self_im, double* out_lags);
int orc_dyadic_lags_slab(int d, const int64_t* levels, int i, int j, double k, double self_re,
                         double self_im, int64_t row0, int64_t row1, double* out);

/* Exact per-axis symmetry check (proj/src/core/generator.cpp:38-62). */
int orc_validate_symmetry(int d, const int64_t* levels, const double* lags, const int* axis_sign);

/* ---- spectra (proj/src/core/kernel.cpp) ------------------------------- */
/* total stored complex elements of the 2^d blocks */
int64_t orc_spectra_elems(int d, const int64_t* levels, int compressed);
/* blocks concatenated in ascending branch-id order, each row-major in its
 * stored shape. compressed requires every axis_sign != 0. */
int orc_precompute(int d, const int64_t* levels, const double* lags, double s0_re, double s0_im,
                   int compressed, const int* axis_sign, double* out_blocks);

/* ---- engines ----------------------------------------------------------- */
/* counters[0..4] = fft_forward, fft_inverse, diag_mults, phase_mults,
 * peak_live_elems (proj/src/core/engine_split.hpp:25-32). May be NULL. */
int orc_split_apply(int d, const int64_t* levels, const double* blocks, int compressed,
                    const int* axis_sign, const double* v, double* y, int64_t* counters);
/* Branch-partitioned partial output: the contribution of the subtree whose
 * branch ids have low q bits == part (P = 2^q parts). Sum over parts == full
 * apply. Restates the paper's multi-device outlook. */
int orc_split_apply_partial(int d, const int64_t* levels, const double* blocks, int compressed,
                            const int* axis_sign, const double* v, double* y, int part, int nparts);
int orc_embed_apply(int d, const int64_t* levels, const double* lags, double s0_re, double s0_im,
                    const double* v, double* y);
int orc_naive_matvec(int d, const int64_t* levels, const double* lags, const double* v, double* y,
                     int64_t cap);

/* ---- pieces, exposed for the reference's unit-level known answers ------ */
int orc_fft_axis(int d, const int64_t* shape, double* t, int axis, int inverse);
int orc_phase_axis(int d, const int64_t* shape, double* t, int axis, int conjugate);
int orc_embed_generator(int d, const int64_t* levels, const double* lags, double s0_re,
                        double s0_im, double* out);

/* ---- closed-form model (proj/src/core/analysis.cpp:21-56) -------------- */
int orc_predict(int d, double n, double out[9]);

#ifdef __cplusplus
}
#endif

#endif
