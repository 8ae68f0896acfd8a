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
    SHB_ERANGE = 4, /* capacity too small  -> ValueError                     */
    SHB_EIO = 5     /* file I/O            -> OSError                        */
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
/* The same for the FP64 tensor path (DMMA m8n8k4, the QFT's default FP64
 * engine): independent accumulator chains, about `seconds` long. */
int shb_fp64_dmma_peak(double seconds, double *tflops, void *stream);

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

/* As shb_progression_is_uniform, plus *real = 1 if every imaginary part is
 * zero (selects the real-amplitude DMMA form of shb_dft_real). */
int shb_progression_kind(const double *d_amps, uint64_t length, int *uniform,
                         int *real, double *amp_re, double *amp_im,
                         void *stream);

/* d_amps[j] = amp for j < length where the support index a0 + j*stride is in
 * d_support[0..m), 0 otherwise (collapsed register -> progression amplitudes). */
int shb_fill_progression(const uint64_t *d_support, uint64_t m, uint64_t a0,
                         uint64_t stride, uint64_t length, double amp_re,
                         double amp_im, double *d_amps, void *stream);

/* --------------------------------------------------------------------- QFT
 * qft.dense_dft / qft.tiled_dft (qft.py:95-142) and the compiled inner loop
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

/* shb_dft for a real amplitude stream: the imaginary parts of d_amps are
 * ignored (the caller has checked them to be zero, shb_progression_kind).
 * FP64 with tiles == 1 runs the real-A DMMA form: 2 real products per phase
 * term (amp*cos, amp*sin) instead of a complex multiply.  Other cases behave
 * exactly as shb_dft. */
int shb_dft_real(const double *d_amps, uint64_t length, uint64_t a0,
                 uint64_t stride, uint64_t q, uint64_t c_begin,
                 uint64_t c_count, uint32_t tiles, double scale, int precision,
                 double *d_out, double *d_prob, double *d_block_sums,
                 void *stream);

/* Name of the kernel the three DFT entry points launch for these arguments
 * (uniform: shb_dft_uniform; real: shb_dft_real), and the flops one phase
 * term costs in it (*flops_per_term: 8 complex multiply-add, 4 real
 * amplitude x complex phase).  Static string; for roofline reporting. */
const char *shb_dft_engine(int uniform, int real, uint64_t q, int precision,
                           uint32_t tiles, int *flops_per_term);

/* Same transform for a uniform comb: every one of the `length` progression
 * amplitudes equals (amp_re + i amp_im) -- the collapsed register of
 * measure_part2 (qstate.py:101-104).  The amplitude is factored
 * out of the sum (out = scale * amp * sum_j e^{...}); no amplitude array. */
int shb_dft_uniform(double amp_re, double amp_im, uint64_t length, uint64_t a0,
                    uint64_t stride, uint64_t q, uint64_t c_begin,
                    uint64_t c_count, uint32_t tiles, double scale,
                    int precision, double *d_out, double *d_prob,
                    double *d_block_sums, void *stream);

/* ------------------------------------------------------ gate-level QFT
 * The reference's circuit engine primitives (qft.py:164-212) on a device
 * complex128[q] vector (interleaved re, im), bit-identical to numpy's
 * arithmetic.  circuit_qft (qft.py:215-231) is built from them in the
 * Python layer, so the "circuit" engine cross-checks the DFT kernels
 * independently.  SHB_EINVAL for the reference's argument errors. */
/* apply_hadamard (qft.py:164-177): (u, v) -> ((u+v)/sqrt2, (u-v)/sqrt2) over
 * the index pairs differing in bit `qubit`; in place. */
int shb_apply_hadamard(double *state, uint64_t q, int qubit, void *stream);
/* apply_controlled_phase (qft.py:180-196): amplitudes whose index has both
 * bits set are multiplied by (phase_re + i phase_im) = np.exp(1j*angle)
 * (computed by the caller); in place. */
int shb_apply_controlled_phase(double *state, uint64_t q, int control, int target,
                               double phase_re, double phase_im, void *stream);
/* bit_reverse_permute (qft.py:199-212): out[reverse_bits_w(a)] = in[a];
 * out of place. */
int shb_bit_reverse_permute(const double *in, double *out, uint64_t q, void *stream);

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

/* Continuations from a running value s_in, for a shard of a longer vector
 * whose earlier elements summed left to right to s_in (the sharded read
 * chains them rank to rank):
 *   *s_out  = the running sum after the last element (s_in if count == 0);
 *   *index  = first i with running sum s_in + p[0] + ... + p[i] > target,
 *             or count if none. */
int shb_cumsum_total_from(const double *d_prob, uint64_t count, double s_in,
                          double *s_out, void *stream);
int shb_cumsum_search_from(const double *d_prob, uint64_t count, double s_in,
                           double target, uint64_t *index, void *stream);

/* The whole Born-rule read (qstate.py:112-114) for a draw u:
 * target = u * cumsum[-1], *index = searchsorted(cumsum, target, "right")
 * (un-clamped; the caller clamps to q-1), *total = cumsum[-1] (nullable). */
int shb_sample_index(const double *d_prob, uint64_t count, double u,
                     uint64_t *index, double *total, void *stream);

/* Split form of the sequential cumsum, for a vector sharded over ranks or
 * devices (the sharded Born-rule read, distributed.py / shb_sample):
 *   shb_cumsum_records  -- per-tile binade records from a HINT of the running
 *                          value entering this shard (parallel on every shard;
 *                          the result stays exact whatever the hint);
 *   shb_cumsum_walk     -- the exact walk from the exact s_in: *s_out, and the
 *                          exact running value at every tile start in d_tile_S;
 *                          this is the only step that chains shard to shard;
 *   shb_cumsum_find     -- searchsorted(cumsum, target, "right") in the shard
 *                          from d_tile_S and the shard's total (*index = count
 *                          when no running value exceeds target).
 * Buffers: d_recs holds shb_cumsum_tiles(count) * shb_cumsum_record_bytes()
 * bytes, d_tile_S shb_cumsum_tiles(count) doubles. */
uint64_t shb_cumsum_tiles(uint64_t count);
uint64_t shb_cumsum_record_bytes(void);
int shb_cumsum_records(const double *d_prob, uint64_t count, double s_hint, void *d_recs, void *stream);
int shb_cumsum_walk(const double *d_prob, uint64_t count, const void *d_recs, double s_in,
                    double *d_tile_S, double *s_out, void *stream);
int shb_cumsum_find(const double *d_prob, uint64_t count, const double *d_tile_S, double total,
                    double target, uint64_t *index, void *stream);

/* ------------------------------------------------- host-buffer drop-ins
 * These own their device memory (current device) and take HOST buffers:
 * the C-level equivalents of the reference calls, for FFI users.
 */
/* qft.dense_dft (tiles == 1) / qft.tiled_dft (tiles >= 2) on a host
 * complex128[q] state -> host complex128[q] output, scaled by 1/sqrt(q).
 * Both copies overlap the DFT (output slices; a speculative start from the
 * state's head when it holds a uniform progression, confirmed by a scan of
 * the whole state).  Page-locked host buffers make the overlap real. */
int shb_dense_dft_host(const double *state, uint64_t q, uint32_t tiles,
                       int precision, double *out);

/* _kernels.partial_row_sums(out, state, roots, q, k0, k1, j0, j1)
 * (_kernels.py:16): out[k-k0] = sum_{j0<=j<j1} roots[(j k) mod q] state[j],
 * unscaled.  `roots` may be NULL; a non-NULL table must be the reference's
 * e^{+2 pi i j/q} table (spot-checked at six indices, SHB_EINVAL otherwise):
 * the kernel generates those phases itself from the exact integer index, so
 * a different table could not be honoured and is rejected, not ignored. */
int shb_partial_row_sums_host(double *out, const double *state,
                              const double *roots, uint64_t q, uint64_t k0,
                              uint64_t k1, uint64_t j0, uint64_t j1);

/* ------------------------------------------------- register handle (ctx)
 * The whole attempt of shor.single_attempt (shor.py:73-133) on one opaque
 * register that owns its device memory, for FFI callers that hold no device
 * pointers.  The register is sharded over the handle's
 * devices: part 2 (residues) by index a, the spectrum by output c.  One host
 * thread drives every shard; the only cross-shard exchanges are the class
 * counts (host sum), the support geometry (host gcd) and, for sampling, the
 * exact running value of the sequential CDF carried shard to shard (the
 * split cumsum above: records on every shard at once, then the walk).
 *
 * Stage order (each call checks it, SHB_EINVAL otherwise):
 *   shb_init -> shb_ctx_modexp          init_uniform + entangle_modexp (qstate.py:56-83)
 *            -> shb_measure(u) | shb_ctx_class_counts + shb_collapse(k)
 *                                        measure_part2 (qstate.py:86-105)
 *            -> shb_ctx_dft              qft.transform "dense"/"tiled" (qft.py:95-142)
 *            -> shb_sample(u)            sample_part1 (qstate.py:108-114)
 * shb_norm, the shb_copy_* readers and shb_dump_state work at any stage that
 * has the data.  A handle is not reentrant: one handle per concurrent run.
 */
typedef struct shb_ctx shb_ctx;

/* Handle over devices 0..ngpu-1 (ngpu <= 0: every visible device). */
int shb_init(int ngpu, shb_ctx **ctx);
/* Handle over an explicit device list; a device may repeat (several shards
 * on one device, e.g. to exercise the sharded path on a single GPU). */
int shb_init_devices(const int *devices, int ndev, shb_ctx **ctx);
void shb_free(shb_ctx *ctx);
/* *stage: 0 empty, 1 entangled, 2 collapsed, 3 transformed; *q register
 * size, *n modulus (0 before shb_ctx_modexp).  Outputs are nullable. */
int shb_ctx_state(const shb_ctx *ctx, int *stage, uint64_t *q, uint64_t *n,
                  int *nshards);

/* init_uniform(2^w) then entangle_modexp(reg, x, n) (qstate.py:56-83):
 * residues[a] = x^a mod n on the shards.  Same ValueErrors as the reference
 * (n < 2, gcd(x, n) != 1); w in [1, 32].  Discards any previous register. */
int shb_ctx_modexp(shb_ctx *ctx, uint64_t x, uint64_t n, uint32_t w);

/* Exact residue-class counts of part 2 (the integer form of the bincount at
 * qstate.py:97): counts_out[v] for v < ncls; ncls must be >= n (SHB_ERANGE). */
int shb_ctx_class_counts(shb_ctx *ctx, uint64_t *counts_out, uint64_t ncls);

/* Collapse part 1 onto {a : residue[a] == k} (qstate.py:101-104): *M_out =
 * support size, *amp_out = the surviving amplitude (real; imaginary part +0),
 * rounded exactly as the reference divides by sqrt(sum of kept weights). */
int shb_collapse(shb_ctx *ctx, uint32_t k, uint64_t *M_out, double *amp_out);

/* measure_part2 with the draw u = s.uniform() (qstate.py:86-105): the
 * outcome k from the exact class counts (shb_host_measure_class), then
 * shb_collapse(k).  k, M and the amplitude are bit-identical to the
 * reference. */
int shb_measure(shb_ctx *ctx, double u, uint32_t *k_out, uint64_t *M_out,
                double *amp_out);

/* The QFT of the collapsed register (qft.dense_dft for tiles == 1,
 * qft.tiled_dft for tiles >= 2, tiles | q), with |V|^2 fused. */
int shb_ctx_dft(shb_ctx *ctx, int precision, uint32_t tiles);

/* l2_norm (qstate.py:117-118) of the register at its current stage. */
int shb_norm(shb_ctx *ctx, double *out);

/* sample_part1 with the draw u (qstate.py:108-114) on the transformed
 * register: norm check (1e-9 FP64, 1e-4 FP32), exact sequential cumsum,
 * m = min(searchsorted(cum, u * cum[-1], "right"), q - 1). */
int shb_sample(shb_ctx *ctx, double u, uint64_t *m_out);

/* Host readers.  Spectrum rows [c0, c1) as interleaved complex128; the
 * support (ascending, capacity entries; *m_out = M even on SHB_ERANGE);
 * residues [a0, a1) widened to int64 like the reference array (qstate.py:39). */
int shb_copy_spectrum(shb_ctx *ctx, uint64_t c0, uint64_t c1, double *host_out);
int shb_copy_support(shb_ctx *ctx, uint64_t *host_out, uint64_t capacity,
                     uint64_t *m_out);
int shb_copy_residues(shb_ctx *ctx, uint64_t a0, uint64_t a1, int64_t *host_out);

/* qstate.dump_state (qstate.py:121-130) of the transformed register:
 * "QREG" header + q little-endian complex128, streamed shard by shard.
 * SHB_EIO if the file cannot be written. */
int shb_dump_state(shb_ctx *ctx, const char *path);

/* --------------------------------------------- exact host-side helpers
 * Closed-form emulation of numpy reductions over a constant vector; used by
 * measure_part2 for odd register widths where 1/sqrt(q) is inexact.
 */
/* The host half of measure_part2 (qstate.py:95-104) for the uniform register
 * of size q, from exact class counts counts[0..ncls): nclasses = last
 * nonzero class + 1; probs = bincount sums; k = min(searchsorted(cumsum,
 * u * cum[-1], "right"), nclasses - 1); M = counts[k]; amplitude as numpy's
 * complex division rounds it.  No device work. */
int shb_host_measure_class(const uint64_t *counts, uint64_t ncls, uint64_t q,
                           double u, uint32_t *k_out, uint64_t *M_out,
                           double *amp_out);
/* np.cumsum(np.full(count, w))[-1] == the per-bin accumulation of
 * np.bincount(weights=...) (qstate.py:97) for uniform weights. */
double shb_host_seqsum_const(double w, uint64_t count);
/* np.full(count, w).sum() (numpy pairwise summation, qstate.py:102). */
double shb_host_pairwise_sum_const(double w, uint64_t count);

#ifdef __cplusplus
}
#endif

#endif /* SHORB200_H */
