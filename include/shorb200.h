/*
 * shorb200 -- B200-native hot path of the Shor simulator (arXiv 1801.01434).
 *
 * Plain C ABI of libshorb200.so (built for sm_100a).  Every entry point takes
 * plain pointers and sizes; device pointers are prefixed d_, the `stream`
 * argument is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Functions return SHB_OK or an error code; shb_last_error() describes the
 * last failure of the calling thread.  Nothing here aborts the process.
 *
 * Each function cites the reference interface it replaces
 * (/root/reference/pkg/src/shorsim/<file>:<line>).  The Python drop-in in
 * paper_1801_01434_b200/ (ctypes, _native.py) is the reference-facing layer;
 * INTEGRATION.md shows the binding the reference itself would add.
 */
#ifndef SHORB200_H
#define SHORB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHB_ABI_VERSION 1

enum shb_status {
    SHB_OK = 0,
    SHB_EINVAL = 1, /* argument error      -> ValueError in the Python layer */
    SHB_ECUDA = 2,  /* CUDA runtime error  -> RuntimeError                   */
    SHB_ENOMEM = 3, /* device allocation   -> MemoryError                    */
    SHB_ERANGE = 4  /* capacity too small  -> ValueError                     */
};

enum shb_precision { SHB_FP64 = 0, SHB_FP32 = 1 };

int shb_abi_version(void);
const char *shb_last_error(void);
/* SM count / name of `device` (for grid sizing and reports). */
int shb_device_info(int device, int *sm_count, char *name, int name_len);
/* Number of kernels this library has launched in this process (bench.py's
 * gpu_launches evidence). */
uint64_t shb_kernel_launches(void);
/* Measured FP64 FMA throughput of the current device (TFLOP/s) over about
 * `seconds` of independent DFMA chains: the roofline denominator of the QFT
 * kernel (MEASURED_PEAKS.json carries HBM and bf16 peaks only). */
int shb_fp64_peak(double seconds, double *tflops, void *stream);

/* ------------------------------------------------------------------ modexp
 * qstate.entangle_modexp (qstate.py:64-83): part 2 of the register.
 * d_residues[i] = x^(a_begin + i) mod n for i < count, n in [2, 2^32).
 * Sharding: rank g passes its own a_begin / count slice.
 */
int shb_modexp(uint32_t *d_residues, uint64_t a_begin, uint64_t count,
               uint64_t x, uint64_t n, void *stream);

/* ---------------------------------------------------------------- collapse
 * qstate.measure_part2 (qstate.py:95-97): np.bincount of residue classes
 * with the (uniform) weights factored out -> exact integer class counts.
 * d_counts[v] += #{i : d_residues[i] == v}; accumulates, so shards can add
 * into one buffer.  d_counts must hold ncls entries (ncls > max residue).
 */
int shb_class_counts(const uint32_t *d_residues, uint64_t count,
                     uint64_t *d_counts, uint64_t ncls, void *stream);

/* qstate.measure_part2 (qstate.py:101): mask = residues == k.
 * Writes the ascending indices a_begin + i with d_residues[i] == k into
 * d_support (capacity entries) by warp-ballot + prefix-sum compaction and
 * returns their number in *m_out (host).  SHB_ERANGE if capacity < M.
 */
int shb_compact_eq(const uint32_t *d_residues, uint64_t count, uint32_t k,
                   uint64_t a_begin, uint64_t *d_support, uint64_t capacity,
                   uint64_t *m_out, void *stream);

/* Arithmetic-progression descriptor of an ascending index set:
 * a0 = first index, stride = gcd of all gaps (1 if a single element),
 * length = (last - a0)/stride + 1 (0 for an empty set).  Host outputs. */
int shb_support_progression(const uint64_t *d_support, uint64_t m,
                            uint64_t *a0, uint64_t *stride, uint64_t *length,
                            void *stream);

/* Same descriptor for the nonzero entries of a dense complex128 state of
 * length q (interleaved re, im).  Used by the dense_dft drop-in. */
int shb_state_progression(const double *d_state, uint64_t q, uint64_t *a0,
                          uint64_t *stride, uint64_t *length, void *stream);

/* d_amps[j] = d_state[a0 + j*stride] (complex128), j < length. */
int shb_gather_progression(const double *d_state, uint64_t a0, uint64_t stride,
                           uint64_t length, double *d_amps, void *stream);

/* *uniform = 1 if all `length` complex128 amplitudes are bitwise equal, and
 * the common value in (*amp_re, *amp_im): selects the uniform-comb kernel. */
int shb_progression_is_uniform(const double *d_amps, uint64_t length,
                               int *uniform, double *amp_re, double *amp_im,
                               void *stream);

/* d_amps[j] = amp for j < length where the support index a0 + j*stride is in
 * d_support[0..m), 0 otherwise (collapsed register -> progression amplitudes). */
int shb_fill_progression(const uint64_t *d_support, uint64_t m, uint64_t a0,
                         uint64_t stride, uint64_t length, double amp_re,
                         double amp_im, double *d_amps, void *stream);

/* --------------------------------------------------------------------- QFT
 * qft.dense_dft / qft.tiled_dft (qft.py:270-317) and the compiled inner loop
 * _kernels.partial_row_sums (_kernels.py:16-30), B200 form:
 *
 *   out[i] = scale * sum_{t < tiles} sum_{a_j in tile t} amps[j] e^{+2 pi i a_j c / q}
 *   a_j = a0 + j*stride (j < length),  c = c_begin + i (i < c_count)
 *
 * tile t covers a in [t*q/tiles, (t+1)*q/tiles); tile partials are added in
 * ascending t (qft.py:138-141).  Only the support is visited: q*M phase terms.
 * d_amps: complex128[length]; d_out: complex128[c_count];
 * d_prob (nullable): float64[c_count] = |out|^2 as np.abs(.)**2 (qstate.py:111);
 * d_block_sums (nullable): per-CTA sums of d_prob, see shb_dft_num_blocks.
 * precision: SHB_FP64 (<=1e-9 relative) or SHB_FP32 (<=1e-4 relative).
 * Sharding: rank g passes its own c_begin / c_count.
 */
int shb_dft(const double *d_amps, uint64_t length, uint64_t a0,
            uint64_t stride, uint64_t q, uint64_t c_begin, uint64_t c_count,
            uint32_t tiles, double scale, int precision, double *d_out,
            double *d_prob, double *d_block_sums, void *stream);
uint64_t shb_dft_num_blocks(uint64_t c_count, int precision);

/* Same transform for a uniform comb: every one of the `length` progression
 * amplitudes equals (amp_re + i amp_im) -- the collapsed register of
 * measure_part2 (qstate.py:101-104).  The amplitude is factored
 * out of the sum (out = scale * amp * sum_j e^{...}); no amplitude array. */
int shb_dft_uniform(double amp_re, double amp_im, uint64_t length, uint64_t a0,
                    uint64_t stride, uint64_t q, uint64_t c_begin,
                    uint64_t c_count, uint32_t tiles, double scale,
                    int precision, double *d_out, double *d_prob,
                    double *d_block_sums, void *stream);

/* ---------------------------------------------------------------- sampling
 * qstate.sample_part1 / l2_norm (qstate.py:108-118).
 */
/* d_prob[i] = |d_state[i]|^2 computed as hypot(re, im)^2 (qstate.py:111). */
int shb_probabilities(const double *d_state, uint64_t count, double *d_prob,
                      void *stream);

/* Deterministic (fixed-order tree) sum of count doubles -> *out (host). */
int shb_sum(const double *d_x, uint64_t count, double *out, void *stream);

/* Exact emulation of np.cumsum(p)[-1] (strict left-to-right float64 adds,
 * qstate.py:112): bit-identical to numpy for any input. */
int shb_cumsum_total(const double *d_prob, uint64_t count, double *total,
                     void *stream);

/* Exact emulation of np.searchsorted(np.cumsum(p), target, side="right")
 * (qstate.py:113): first i with cumsum[i] > target, or count if none. */
int shb_cumsum_search(const double *d_prob, uint64_t count, double target,
                      uint64_t *index, void *stream);

/* The whole Born-rule read (qstate.py:112-114) for a draw u:
 * target = u * cumsum[-1], *index = searchsorted(cumsum, target, "right")
 * (un-clamped; the caller clamps to q-1), *total = cumsum[-1] (nullable). */
int shb_sample_index(const double *d_prob, uint64_t count, double u,
                     uint64_t *index, double *total, void *stream);

/* ------------------------------------------------- host-buffer drop-ins
 * These own their device memory (current device) and take HOST buffers:
 * the C-level equivalents of the reference calls, for FFI users.
 */
/* qft.dense_dft (tiles == 1) / qft.tiled_dft (tiles >= 2) on a host
 * complex128[q] state -> host complex128[q] output, scaled by 1/sqrt(q). */
int shb_dense_dft_host(const double *state, uint64_t q, uint32_t tiles,
                       int precision, double *out);

/* _kernels.partial_row_sums(out, state, roots, q, k0, k1, j0, j1)
 * (_kernels.py:16): out[k-k0] = sum_{j0<=j<j1} roots[(j k) mod q] state[j],
 * unscaled.  `roots` is accepted for signature parity and may be NULL: the
 * kernel generates its phases exactly from the integer index. */
int shb_partial_row_sums_host(double *out, const double *state,
                              const double *roots, uint64_t q, uint64_t k0,
                              uint64_t k1, uint64_t j0, uint64_t j1);

/* --------------------------------------------- exact host-side helpers
 * Closed-form emulation of numpy reductions over a constant vector; used by
 * measure_part2 for odd register widths where 1/sqrt(q) is inexact.
 */
/* np.cumsum(np.full(count, w))[-1] == the per-bin accumulation of
 * np.bincount(weights=...) (qstate.py:97) for uniform weights. */
double shb_host_seqsum_const(double w, uint64_t count);
/* np.full(count, w).sum() (numpy pairwise summation, qstate.py:102). */
double shb_host_pairwise_sum_const(double w, uint64_t count);

#ifdef __cplusplus
}
#endif

#endif /* SHORB200_H */
