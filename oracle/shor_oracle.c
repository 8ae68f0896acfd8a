/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the Shor hot path.
 *
 * This file restates, in plain C, the arithmetic of the reference `shorsim`
 * package (/root/reference/pkg/src/shorsim) for the three hot-path stages so
 * that the B200 kernels can be checked against it.  Only tests/, the
 * __graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path (paper_1801_01434_b200) never
 * links or calls anything in oracle/.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile -> oracle/_build/liboracle.so
 * Compiled with -ffp-contract=off so no multiply-add is fused: the reference
 * kernel is numba-compiled without fastmath, which never contracts either.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <pthread.h>

/* Minimal static-chunk parallel-for over rows (pthreads; no OpenMP so the
 * recipe builds with any gcc in the image). */
typedef struct {
    void (*body)(void *ctx, int64_t lo, int64_t hi);
    void *ctx;
    int64_t lo, hi;
} oracle_span;

static void *oracle_span_run(void *arg)
{
    oracle_span *s = (oracle_span *)arg;
    s->body(s->ctx, s->lo, s->hi);
    return NULL;
}

static void oracle_parallel_for(int64_t n, int nthreads,
                                void (*body)(void *, int64_t, int64_t),
                                void *ctx)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = (int)(n > 0 ? n : 1);
    pthread_t tid[256];
    oracle_span spans[256];
    /* interleave rows across threads in small blocks for load balance */
    for (int t = 0; t < nthreads; t++) {
        spans[t].body = body;
        spans[t].ctx = ctx;
        spans[t].lo = n * t / nthreads;
        spans[t].hi = n * (t + 1) / nthreads;
    }
    for (int t = 1; t < nthreads; t++)
        pthread_create(&tid[t], NULL, oracle_span_run, &spans[t]);
    oracle_span_run(&spans[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(tid[t], NULL);
}

/*
 * roots[idx] exactly as qft.build_twiddles builds its table
 * (qft.py:79: np.exp((2j*np.pi/q) * np.arange(q))).
 * (2j*pi/q) is the complex (0, fl(2*pi)/q); multiplying by (idx + 0j) gives
 * (0, fl(t*idx)); numpy's exp of a purely imaginary argument is
 * (cos(y), sin(y)) from libm.  Checked bitwise against numpy on every width
 * the tests use (tests/test_oracle_golden.py::test_root_table_bitwise).
 */
static inline void oracle_root(uint64_t q, uint64_t idx, double *re, double *im)
{
    const double t = (2.0 * M_PI) / (double)q;
    const double y = t * (double)idx;
    *re = cos(y);
    *im = sin(y);
}

void oracle_roots(uint64_t q, uint64_t n, const uint64_t *idx, double *out)
{
    for (uint64_t i = 0; i < n; i++)
        oracle_root(q, idx[i], &out[2 * i], &out[2 * i + 1]);
}

/*
 * Rows of the reference dense transform restricted to the support.
 *
 * Reference: _kernels.partial_row_sums (_kernels.py:16-30) called by
 * qft.dense_dft (qft.py:95-112) with j0=0, j1=q:
 *     acc = 0; for j ascending: acc += roots[(j*k) mod q] * state[j]
 * then out *= 1/sqrt(q) (qft.py:111).
 * Terms with state[j] == 0 add an exact (+-0, +-0) and leave acc unchanged,
 * so summing over the nonzero support only, in ascending order, is bitwise
 * identical to the reference (pinned by the n=15 / n=221 golden spectra).
 *
 * The complex product follows numba's expansion
 *     (ar*br - ai*bi, ar*bi + ai*br)
 * and the accumulator add is component-wise.
 *
 * supp[] must be ascending.  amps[] is interleaved (re, im).
 * If apply_scale != 0 each row is multiplied by scale as `out *= scale`
 * does for a complex array and a real scalar (numpy promotes the scalar to
 * (scale + 0j) and performs a full complex multiply).
 */
typedef struct {
    uint64_t q, nsupp;
    const uint64_t *supp, *rows;
    const double *amps;
    int apply_scale;
    double scale;
    double *out;
} dft_rows_ctx;

static void dft_rows_body(void *vctx, int64_t lo, int64_t hi)
{
    const dft_rows_ctx *x = (const dft_rows_ctx *)vctx;
    const uint64_t mask = x->q - 1;
    for (int64_t r = lo; r < hi; r++) {
        const uint64_t c = x->rows[r];
        double acc_re = 0.0, acc_im = 0.0;
        for (uint64_t s = 0; s < x->nsupp; s++) {
            const uint64_t jk = (x->supp[s] * c) & mask; /* exact: q | 2^64 */
            double rr, ri;
            oracle_root(x->q, jk, &rr, &ri);
            const double ar = x->amps[2 * s], ai = x->amps[2 * s + 1];
            const double pr = rr * ar - ri * ai;
            const double pi = rr * ai + ri * ar;
            acc_re = acc_re + pr;
            acc_im = acc_im + pi;
        }
        if (x->apply_scale) {
            /* (acc_re + i acc_im) * (scale + 0i) */
            const double o_re = acc_re * x->scale - acc_im * 0.0;
            const double o_im = acc_re * 0.0 + acc_im * x->scale;
            acc_re = o_re;
            acc_im = o_im;
        }
        x->out[2 * r] = acc_re;
        x->out[2 * r + 1] = acc_im;
    }
}

void oracle_dft_rows(uint64_t q, uint64_t nsupp, const uint64_t *supp,
                     const double *amps, uint64_t nrows, const uint64_t *rows,
                     int apply_scale, double scale, double *out, int nthreads)
{
    dft_rows_ctx ctx = {q, nsupp, supp, rows, amps, apply_scale, scale, out};
    oracle_parallel_for((int64_t)nrows, nthreads, dft_rows_body, &ctx);
}

/*
 * The same rows computed the way the reference engine really iterates:
 * every j in [j0, j1), zeros included, with the incremental twiddle index of
 * _kernels.py:24-29 (jk += k; if jk >= q: jk -= q).  O(q) per row; used only
 * to time the reference algorithm and to cross-check oracle_dft_rows.
 * state[] is the dense interleaved complex vector of length q.
 */
typedef struct {
    uint64_t q, j0, j1;
    const double *state;
    const uint64_t *rows;
    double *out;
} literal_ctx;

static void literal_body(void *vctx, int64_t lo, int64_t hi)
{
    const literal_ctx *x = (const literal_ctx *)vctx;
    for (int64_t r = lo; r < hi; r++) {
        const uint64_t k = x->rows[r];
        double acc_re = 0.0, acc_im = 0.0;
        uint64_t jk = (x->j0 * k) & (x->q - 1);
        for (uint64_t j = x->j0; j < x->j1; j++) {
            double rr, ri;
            oracle_root(x->q, jk, &rr, &ri);
            const double ar = x->state[2 * j], ai = x->state[2 * j + 1];
            acc_re = acc_re + (rr * ar - ri * ai);
            acc_im = acc_im + (rr * ai + ri * ar);
            jk += k;
            if (jk >= x->q) jk -= x->q;
        }
        x->out[2 * r] = acc_re;
        x->out[2 * r + 1] = acc_im;
    }
}

void oracle_dense_rows_literal(uint64_t q, const double *state, uint64_t j0,
                               uint64_t j1, uint64_t nrows,
                               const uint64_t *rows, double *out, int nthreads)
{
    literal_ctx ctx = {q, j0, j1, state, rows, out};
    oracle_parallel_for((int64_t)nrows, nthreads, literal_body, &ctx);
}

/*
 * residues[i] = x^(a_begin + i) mod n, by the incremental recurrence the
 * SPEC states for entangle_modexp (the reference walks one
 * cycle and tiles it, qstate.py:77-82, which yields the same values).
 */
void oracle_modexp(uint64_t x, uint64_t n, uint64_t a_begin, uint64_t count,
                   uint32_t *residues)
{
    /* seed: x^a_begin mod n by square-and-multiply (numtheory.modpow) */
    unsigned __int128 base = x % n, acc = 1 % n;
    uint64_t e = a_begin;
    while (e) {
        if (e & 1) acc = (acc * base) % n;
        base = (base * base) % n;
        e >>= 1;
    }
    uint64_t r = (uint64_t)acc;
    const uint64_t xm = x % n;
    for (uint64_t i = 0; i < count; i++) {
        residues[i] = (uint32_t)r;
        r = (uint64_t)(((unsigned __int128)r * xm) % n);
    }
}

/* bincount of residues (qstate.py:97) with unit weights: exact counts */
void oracle_class_counts(const uint32_t *residues, uint64_t count,
                         uint64_t ncls, uint64_t *counts)
{
    memset(counts, 0, ncls * sizeof(uint64_t));
    for (uint64_t i = 0; i < count; i++) counts[residues[i]]++;
}

/*
 * qstate.sample_part1 tail (qstate.py:112-114):
 *   cum = np.cumsum(probs)            -- strictly sequential float64 adds
 *   m = searchsorted(cum, u*cum[-1], side="right"); min(m, q-1)
 */
uint64_t oracle_cumsum_search(const double *p, uint64_t L, double u,
                              double *total_out)
{
    double s = 0.0;
    for (uint64_t i = 0; i < L; i++) s = s + p[i];
    const double target = u * s;
    if (total_out) *total_out = s;
    double c = 0.0;
    for (uint64_t i = 0; i < L; i++) {
        c = c + p[i];
        if (c > target) return i;
    }
    return L - 1; /* searchsorted returns L; the reference clamps to q-1 */
}

/*
 * Accuracy reference (not the reference's arithmetic): rows of the DFT of a
 * uniform comb amp * sum_{j<M} |c0 + j r>, scaled by `scale`, from the
 * geometric-series closed form in 80-bit long double,
 *     V_c = amp scale e^{i pi K/q} sin(pi M t/q) / sin(pi t/q),
 *     t = r c mod q as a signed residue in (-q/2, q/2],
 *     K = 2 c0 c + (M-1) t mod 2q,
 * and V_c = amp scale M e^{2 pi i c0 c/q} when t = 0.  Every angle is an
 * exact integer residue times pi/q, and each sine argument is folded into
 * [-pi/2, pi/2] (sin(pi - x) = sin x) so a small sine keeps its relative
 * accuracy; the only errors are long double roundings (~1e-18 relative) and
 * the final rounding to double.  The reference's own sequential sum
 * (oracle_dft_rows) carries up to ~M 2^-53 relative error on a peak row;
 * this function tells which side of a disagreement is the accurate one.
 */
static const long double ORACLE_PI_L = 3.141592653589793238462643383279502884L;

/* k mod 2q as a signed residue in (-q, q] */
static __int128 oracle_mod2q(__int128 k, uint64_t q)
{
    const __int128 q2 = 2 * (__int128)q;
    k %= q2;
    if (k < 0) k += q2;
    if (k > (__int128)q) k -= q2;
    return k;
}

/* sin(pi k / q) for any integer k, argument folded into [-pi/2, pi/2] */
static long double oracle_sinpi_over(__int128 k, uint64_t q)
{
    k = oracle_mod2q(k, q);
    const __int128 h = (__int128)(q / 2);
    if (k > h) k = (__int128)q - k;
    else if (k < -h) k = -(__int128)q - k;
    return sinl(ORACLE_PI_L * (long double)k / (long double)q);
}

void oracle_comb_rows_exact(uint64_t q, uint64_t r, uint64_t c0, uint64_t M,
                            double amp_re, double amp_im, double scale,
                            uint64_t nrows, const uint64_t *rows, double *out)
{
    for (uint64_t i = 0; i < nrows; i++) {
        const __int128 c = (__int128)rows[i];
        __int128 t = (__int128)(((unsigned __int128)r * (unsigned __int128)rows[i]) % q);
        if (t > (__int128)(q / 2)) t -= (__int128)q;
        long double mag;
        __int128 K;
        if (t == 0) {
            mag = (long double)M;
            K = oracle_mod2q(2 * (__int128)c0 * c, q);
        } else {
            mag = oracle_sinpi_over((__int128)M * t, q) / oracle_sinpi_over(t, q);
            K = oracle_mod2q(2 * (__int128)c0 * c + (__int128)(M - 1) * t, q);
        }
        const long double ph = ORACLE_PI_L * (long double)K / (long double)q;
        const long double s = mag * (long double)scale;
        const long double er = cosl(ph), ei = sinl(ph);
        out[2 * i] = (double)(s * (er * amp_re - ei * amp_im));
        out[2 * i + 1] = (double)(s * (er * amp_im + ei * amp_re));
    }
}
