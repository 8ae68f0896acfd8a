// C ABI plumbing for libshorb200.so: error state, device info, scratch
// allocation, the host-buffer drop-ins and the exact host-side helpers.
#include <math.h>
#include <float.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <map>

#include "shb_internal.cuh"

namespace shb {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;

void note_launch(unsigned n) { __atomic_fetch_add(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

int set_error(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int check_cuda(cudaError_t e, const char *what)
{
    if (e == cudaSuccess) return SHB_OK;
    const int code = (e == cudaErrorMemoryAllocation) ? SHB_ENOMEM : SHB_ECUDA;
    cudaGetLastError();  // clear sticky-free errors so later calls can proceed
    return set_error(code, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int sm_count()
{
    static thread_local int cached_dev = -1, cached = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
    }
    return cached > 0 ? cached : 148;
}

// Keep the stream-ordered pool's memory mapped between calls: with the default
// release threshold (0) every multi-GiB scratch buffer is unmapped at the next
// synchronisation and re-mapped by the next call (seconds at 16 GiB).
static void keep_pool_mapped()
{
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

int scratch_alloc(Scratch &s, size_t bytes, cudaStream_t st)
{
    keep_pool_mapped();
    s.st = st;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&s.ptr, bytes, st);
    if (e == cudaErrorMemoryAllocation) {
        // give cached pool memory back (e.g. a previous q = 2^32 call) and retry once
        cudaGetLastError();
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            cudaStreamSynchronize(st);
            cudaMemPoolTrimTo(pool, 0);
        }
        e = cudaMallocAsync(&s.ptr, bytes, st);
    }
    if (e != cudaSuccess) {
        s.ptr = nullptr;
        return check_cuda(e, "cudaMallocAsync(scratch)");
    }
    return SHB_OK;
}

// ---------------------------------------------------------------------------
// Exact closed-form emulation of numpy reductions over a constant vector.

// np.cumsum(np.full(n, w))[-1]: strict left-to-right float64 adds.  Within one
// binade of the running sum S (ulp u) adding w moves S by a fixed number of
// ulps d = round(w/u), so whole runs of adds are one multiply; the add that
// leaves the binade is done in floating point.  Round-half-even ties only
// depend on the parity of S/u, which is even after the first tied add.
static double seqsum_const_impl(double w, uint64_t n)
{
    if (n == 0) return 0.0;
    if (!(w > 0.0) || !isfinite(w)) {
        double s = w;  // cumsum seeds with the first element
        for (uint64_t i = 1; i < n; i++) s = s + w;
        return s;
    }
    double S = w;
    uint64_t done = 1;
    const double two53 = 9007199254740992.0;
    while (done < n) {
        if (!isfinite(S)) {
            return S;
        }
        double u, B;
        if (S < ldexp(1.0, -1021)) {
            u = ldexp(1.0, -1074);
            B = ldexp(1.0, -1021);
        } else {
            int e;
            frexp(S, &e);  // S in [2^(e-1), 2^e)
            u = ldexp(1.0, e - 53);
            B = ldexp(1.0, e);
        }
        const double Su = S / u;   // exact integer < 2^53
        const double x = w / u;    // exact (w <= S)
        const double kf = floor(x);
        const double frac = x - kf;
        double d;
        if (frac < 0.5) {
            d = kf;
        } else if (frac > 0.5) {
            d = kf + 1.0;
        } else {
            if (fmod(Su, 2.0) != 0.0) {  // odd: this one add decides by parity
                S = S + w;
                done++;
                continue;
            }
            d = (fmod(kf, 2.0) == 0.0) ? kf : kf + 1.0;
        }
        if (d == 0.0) return S;  // every further add rounds back to S
        // largest k with Su + k*d < 2^53 (stays strictly inside the binade)
        const double room = two53 - Su;  // exact, > 0
        double ksafe = ceil(room / d) - 1.0;
        if (ksafe < 0) ksafe = 0;
        const uint64_t rem = n - done;
        const uint64_t take = (ksafe >= (double)rem) ? rem : (uint64_t)ksafe;
        S = (Su + (double)take * d) * u;  // exact: integer < 2^53 times power of 2
        done += take;
        (void)B;
        if (done < n) {  // the add that crosses into the next binade
            S = S + w;
            done++;
        }
    }
    return S;
}

// numpy's pairwise summation (umath loops_utils pairwise_sum) specialised to
// a constant input: blocks of <= 128 use 8 interleaved accumulators, larger
// spans split at n/2 rounded down to a multiple of 8.  Memoised by length.
struct PairwiseConst {
    double w;
    std::map<uint64_t, double> memo;
    double run(uint64_t n)
    {
        auto it = memo.find(n);
        if (it != memo.end()) return it->second;
        double res;
        if (n < 8) {
            res = -0.0;
            for (uint64_t i = 0; i < n; i++) res += w;
        } else if (n <= 128) {
            // r[k] = w + w + ... ((n - n%8)/8 copies, sequential)
            const uint64_t per = (n - n % 8) / 8;
            double r = seqsum_const_impl(w, per);
            res = ((r + r) + (r + r)) + ((r + r) + (r + r));
            for (uint64_t i = n - n % 8; i < n; i++) res += w;
        } else {
            uint64_t n2 = n / 2;
            n2 -= n2 % 8;
            res = run(n2) + run(n - n2);
        }
        memo[n] = res;
        return res;
    }
};

// FP64 FMA throughput probe: 8 independent DFMA chains per thread, a grid of
// 4 CTAs x 256 threads per SM.  The roofline denominator of the QFT kernel.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double *out, int iters, double a, double b)
{
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it += 4) {
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
            for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) s += x[i];
    if (s == 1234.5) out[0] = s;  // keep the chains alive
}

// FP64 tensor path (DMMA m8n8k4) probe: 4 independent accumulator chains per
// warp, B operands cycling through registers, as in the DFT's DMMA kernel.
__global__ void __launch_bounds__(256) dmma_probe_kernel(double *out, int iters, double a, double b)
{
    double d[4][2], g[8];
#pragma unroll
    for (int i = 0; i < 4; i++) d[i][0] = d[i][1] = threadIdx.x * 1e-6 + i;
#pragma unroll
    for (int i = 0; i < 8; i++) g[i] = b + i * 1e-3;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++)
#pragma unroll
            for (int i = 0; i < 4; i++)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(d[i][0]), "+d"(d[i][1])
                             : "d"(a), "d"(g[k]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) s += d[i][0] + d[i][1];
    if (s == 1234.5) out[0] = s;
}

}  // namespace shb

using namespace shb;

extern "C" {

int shb_abi_version(void) { return SHB_ABI_VERSION; }

uint64_t shb_kernel_launches(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

const char *shb_last_error(void) { return g_err; }

int shb_device_info(int device, int *sm, char *name, int name_len)
{
    cudaDeviceProp p;
    SHB_TRY_CUDA(cudaGetDeviceProperties(&p, device));
    if (sm) *sm = p.multiProcessorCount;
    if (name && name_len > 0) {
        strncpy(name, p.name, (size_t)name_len - 1);
        name[name_len - 1] = 0;
    }
    return SHB_OK;
}

int shb_fp64_peak(double seconds, double *tflops, void *stream)
{
    if (!tflops) return set_error(SHB_EINVAL, "null output");
    cudaStream_t st = as_stream(stream);
    Scratch sink;
    SHB_TRY(scratch_alloc(sink, sizeof(double), st));
    const unsigned grid = (unsigned)sm_count() * 4;
    const int iters = 1 << 16;
    cudaEvent_t e0, e1;
    SHB_TRY_CUDA(cudaEventCreate(&e0));
    SHB_TRY_CUDA(cudaEventCreate(&e1));
    fp64_probe_kernel<<<grid, 256, 0, st>>>((double *)sink.ptr, 1024, 0.999999, 1e-7);  // warm-up
    SHB_LAUNCHED();
    // size the timed loop to roughly `seconds`
    int reps = 1;
    float ms = 0.f;
    for (;;) {
        SHB_TRY_CUDA(cudaEventRecord(e0, st));
        for (int r = 0; r < reps; r++) {
            fp64_probe_kernel<<<grid, 256, 0, st>>>((double *)sink.ptr, iters, 0.999999, 1e-7);
            SHB_LAUNCHED();
        }
        SHB_TRY_CUDA(cudaEventRecord(e1, st));
        SHB_TRY_CUDA(cudaEventSynchronize(e1));
        SHB_TRY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (ms >= seconds * 1000.0 * 0.5 || reps >= (1 << 16)) break;
        reps *= 2;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 16.0 * (double)iters * 256.0 * grid * reps;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return SHB_OK;
}

int shb_fp64_dmma_peak(double seconds, double *tflops, void *stream)
{
    if (!tflops) return set_error(SHB_EINVAL, "null output");
    cudaStream_t st = as_stream(stream);
    Scratch sink;
    SHB_TRY(scratch_alloc(sink, sizeof(double), st));
    const unsigned grid = (unsigned)sm_count() * 2;
    const int iters = 1 << 12;
    cudaEvent_t e0, e1;
    SHB_TRY_CUDA(cudaEventCreate(&e0));
    SHB_TRY_CUDA(cudaEventCreate(&e1));
    dmma_probe_kernel<<<grid, 256, 0, st>>>((double *)sink.ptr, 64, 0.999999, 1e-7);  // warm-up
    SHB_LAUNCHED();
    int reps = 1;
    float ms = 0.f;
    for (;;) {
        SHB_TRY_CUDA(cudaEventRecord(e0, st));
        for (int r = 0; r < reps; r++) {
            dmma_probe_kernel<<<grid, 256, 0, st>>>((double *)sink.ptr, iters, 0.999999, 1e-7);
            SHB_LAUNCHED();
        }
        SHB_TRY_CUDA(cudaEventRecord(e1, st));
        SHB_TRY_CUDA(cudaEventSynchronize(e1));
        SHB_TRY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (ms >= seconds * 1000.0 * 0.5 || reps >= (1 << 16)) break;
        reps *= 2;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // one DMMA m8n8k4 = 256 multiply-adds = 512 flops per warp instruction
    const double flops = 512.0 * 32.0 * (double)iters * (256 / 32) * grid * reps;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return SHB_OK;
}

double shb_host_seqsum_const(double w, uint64_t count) { return seqsum_const_impl(w, count); }

double shb_host_pairwise_sum_const(double w, uint64_t count)
{
    PairwiseConst p{w, {}};
    return p.run(count);
}

int shb_host_measure_class(const uint64_t *counts, uint64_t ncls, uint64_t q, double u, uint32_t *k_out,
                           uint64_t *M_out, double *amp_out)
{
    if (!counts || !k_out || !M_out || !amp_out) return set_error(SHB_EINVAL, "null argument");
    if (q < 2 || (q & (q - 1))) return set_error(SHB_EINVAL, "q must be a power of two >= 2");
    uint64_t nclasses = ncls;
    while (nclasses > 0 && counts[nclasses - 1] == 0) nclasses--;
    if (nclasses == 0) return set_error(SHB_EINVAL, "all class counts are zero");
    if (nclasses - 1 > 0xFFFFFFFFull) return set_error(SHB_EINVAL, "residue class exceeds 32 bits");
    // init_uniform's amplitude (qstate.py:59) and its weight np.abs(a)**2 (qstate.py:95)
    const double a = 1.0 / sqrt((double)q);
    const double w0 = a * a;
    // bincount (qstate.py:97) per bin, then np.cumsum (qstate.py:98): both sequential
    double cum = 0.0, total = 0.0;
    {
        std::map<uint64_t, double> memo;
        for (uint64_t v = 0; v < nclasses; v++) {
            const uint64_t c = counts[v];
            if (c == 0) continue;
            auto it = memo.find(c);
            const double p = it != memo.end() ? it->second : (memo[c] = seqsum_const_impl(w0, c));
            total = total + p;
        }
    }
    // searchsorted(cum, u * cum[-1], side="right") (qstate.py:99), clamped (qstate.py:100)
    const double target = u * total;
    uint64_t k = 0;
    {
        std::map<uint64_t, double> memo;
        for (k = 0; k < nclasses; k++) {
            const uint64_t c = counts[k];
            if (c) {
                auto it = memo.find(c);
                const double p = it != memo.end() ? it->second : (memo[c] = seqsum_const_impl(w0, c));
                cum = cum + p;
            }
            if (cum > target) break;
        }
    }
    if (k > nclasses - 1) k = nclasses - 1;
    const uint64_t M = counts[k];
    // kept = sqrt(weights[mask].sum()) (pairwise, qstate.py:102); amplitude / kept is a
    // complex / complex division in numpy: Smith's form, (a + 0*rat) * (1 / kept)
    PairwiseConst pw{w0, {}};
    const double kept = sqrt(pw.run(M));
    *k_out = (uint32_t)k;
    *M_out = M;
    *amp_out = a * (1.0 / kept);
    return SHB_OK;
}

// ---------------------------------------------------------------------------
// Host-buffer drop-ins: the C-level form of qft.dense_dft / tiled_dft and of
// the _kernels.partial_row_sums seam.  Device memory is stream-ordered and
// freed before return.

// The state's progression descriptor and kernel choice (what the DFT launch needs).
struct ProgKind {
    uint64_t a0 = 0, stride = 1, len = 0;
    int uni = 0, real = 0;
    double ur = 0.0, ui = 0.0;
};

static int scan_progression(const double *d_state, uint64_t n, Scratch &d_amps, ProgKind &k, cudaStream_t s)
{
    SHB_TRY(shb_state_progression(d_state, n, &k.a0, &k.stride, &k.len, s));
    SHB_TRY(scratch_alloc(d_amps, (k.len ? k.len : 1) * 16, s));
    if (k.len) SHB_TRY(shb_gather_progression(d_state, k.a0, k.stride, k.len, (double *)d_amps.ptr, s));
    if (k.len) SHB_TRY(shb_progression_kind((const double *)d_amps.ptr, k.len, &k.uni, &k.real, &k.ur, &k.ui, s));
    return SHB_OK;
}

static int dft_host_common(const double *state_host, uint64_t nstate, uint64_t index_base,
                           uint64_t q, uint64_t c_begin, uint64_t c_count, uint32_t tiles,
                           double scale, int precision, double *out_host)
{
    struct StreamGuard {
        cudaStream_t s = nullptr;
        ~StreamGuard() {
            if (s) cudaStreamDestroy(s);
        }
    } st_g, cp_g, up_g;
    SHB_TRY_CUDA(cudaStreamCreateWithFlags(&st_g.s, cudaStreamNonBlocking));  // DFT
    SHB_TRY_CUDA(cudaStreamCreateWithFlags(&cp_g.s, cudaStreamNonBlocking));  // D2H of output slices
    SHB_TRY_CUDA(cudaStreamCreateWithFlags(&up_g.s, cudaStreamNonBlocking));  // bulk H2D + full scan
    cudaStream_t st = st_g.s, cp = cp_g.s, up = up_g.s;
    int rc = SHB_OK;
    {
        Scratch d_state, d_amps, d_head_amps, d_out;
        // declared after the buffers, so destroyed before them on EVERY exit
        // path: the stream-ordered frees (on st) are enqueued only once every
        // stream -- including a D2H copy still reading d_out on cp -- drained
        struct DrainGuard {
            cudaStream_t a, b, c;
            ~DrainGuard() {
                cudaStreamSynchronize(a);
                cudaStreamSynchronize(b);
                cudaStreamSynchronize(c);
            }
        } drain{cp, up, st};
        SHB_TRY(scratch_alloc(d_state, nstate * 16, st));
        SHB_TRY(scratch_alloc(d_out, c_count * 16, st));
        SHB_TRY_CUDA(cudaStreamSynchronize(st));  // the allocations are visible to every stream
        // output slices: slice i's D2H copy (second stream) overlaps slice i+1's
        // DFT when out_host is page-locked (pageable memory serialises the copy).
        // Outputs are independent sums, so slicing changes no value.
        const int nslice = c_count >= (1ull << 22) ? 8 : 1;
        cudaEvent_t ev[8];
        int nev = 0;
        struct EventGuard {
            cudaEvent_t *e;
            int *n;
            ~EventGuard() {
                for (int i = 0; i < *n; i++) cudaEventDestroy(e[i]);
            }
        } ev_guard{ev, &nev};
        for (; nev < nslice; nev++) SHB_TRY_CUDA(cudaEventCreateWithFlags(&ev[nev], cudaEventDisableTiming));
        double *dout = (double *)d_out.ptr;
        // every slice's DFT is enqueued before any D2H copy is issued: a copy to
        // pageable memory blocks the host until it is done, and the DFTs of the
        // later slices must already be queued behind it
        auto launch_slice = [&](int i, const ProgKind &k, const double *amps) -> int {
            const uint64_t lo = c_count * i / nslice, hi = c_count * (i + 1) / nslice;
            int r = k.uni ? shb_dft_uniform(k.ur, k.ui, k.len, k.a0 + index_base, k.stride, q, c_begin + lo, hi - lo,
                                            tiles, scale, precision, dout + 2 * lo, nullptr, nullptr, st)
                          : (k.real ? shb_dft_real : shb_dft)(amps, k.len, k.a0 + index_base, k.stride, q,
                                                              c_begin + lo, hi - lo, tiles, scale, precision,
                                                              dout + 2 * lo, nullptr, nullptr, st);
            if (r != SHB_OK) return r;
            SHB_TRY_CUDA(cudaEventRecord(ev[i], st));
            return SHB_OK;
        };
        auto copy_slice = [&](int i) -> int {
            const uint64_t lo = c_count * i / nslice, hi = c_count * (i + 1) / nslice;
            SHB_TRY_CUDA(cudaStreamWaitEvent(cp, ev[i], 0));
            SHB_TRY_CUDA(cudaMemcpyAsync(out_host + 2 * lo, dout + 2 * lo, (hi - lo) * 16, cudaMemcpyDeviceToHost, cp));
            return SHB_OK;
        };

        // Speculative start.  A large state is uploaded as a head (1/64) and
        // the rest; if the head holds a uniform progression, the DFT of the
        // first output slice starts at once, assuming the progression runs to
        // the end of the state (a full comb, as a collapsed register is),
        // while the rest uploads and the whole state is scanned on `up`.  The
        // scan then decides: the same descriptor -> the speculative slice is
        // exactly the slice the plain path computes and the others follow;
        // anything else -> the plain path (the speculative slice is redone).
        const uint64_t head = nslice > 1 && nstate >= (1ull << 24) ? nstate / 64 : nstate;
        ProgKind spec;
        bool speculating = false;
        SHB_TRY_CUDA(cudaMemcpyAsync(d_state.ptr, state_host, head * 16, cudaMemcpyHostToDevice, st));
        if (head < nstate) {
            SHB_TRY_CUDA(cudaMemcpyAsync((double *)d_state.ptr + 2 * head, state_host + 2 * head,
                                         (nstate - head) * 16, cudaMemcpyHostToDevice, up));
            ProgKind h;
            SHB_TRY(scan_progression((const double *)d_state.ptr, head, d_head_amps, h, st));
            if (h.uni && h.len >= 2) {
                spec = h;
                spec.len = (nstate - 1 - h.a0) / h.stride + 1;
                speculating = true;
                SHB_TRY(launch_slice(0, spec, nullptr));
            }
        }
        // the whole-state scan: on `up` behind the bulk upload (the head's copy on
        // st is complete -- its scan synchronised st), on st when there is no split
        ProgKind k;
        SHB_TRY(scan_progression((const double *)d_state.ptr, nstate, d_amps, k, head < nstate ? up : st));
        const bool confirmed = speculating && k.uni && k.a0 == spec.a0 && k.stride == spec.stride &&
                               k.len == spec.len && k.ur == spec.ur && k.ui == spec.ui;
        // refuted: slice 0 is recomputed (stream order on st) before its copy
        for (int i = confirmed ? 1 : 0; i < nslice && rc == SHB_OK; i++)
            rc = launch_slice(i, k, (const double *)d_amps.ptr);
        for (int i = 0; i < nslice && rc == SHB_OK; i++) rc = copy_slice(i);
        SHB_TRY_CUDA(cudaStreamSynchronize(cp));
        SHB_TRY_CUDA(cudaStreamSynchronize(st));
        if (rc != SHB_OK) return rc;
    }
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    return rc;
}

/* The reference passes its twiddle table (qft.py:79) to partial_row_sums.
 * The device derives every phase from the exact integer index instead, which
 * equals the table up to the table's own rounding; a table that is not
 * e^{+2 pi i j/q} at all would be silently replaced, so it is rejected.
 * Spot checks at j = 0, 1, q/8, q/4, q/2, q-1 (5e-15 absolute). */
static int check_roots_table(const double *roots, uint64_t q)
{
    if (!roots) return SHB_OK;
    const uint64_t idx[6] = {0, 1, q / 8, q / 4, q / 2, q - 1};
    for (int i = 0; i < 6; i++) {
        const uint64_t j = idx[i] % q;
        const double a = (2.0 * M_PI / (double)q) * (double)j;  // qft.py:79's own expression
        const double cs = cos(a), sn = sin(a);
        if (fabs(roots[2 * j] - cs) > 5e-15 || fabs(roots[2 * j + 1] - sn) > 5e-15)
            return set_error(SHB_EINVAL, "roots[%llu] is not e^{+2 pi i j/q}: the device computes the reference "
                             "twiddle table's values itself and cannot honour a different table",
                             (unsigned long long)j);
    }
    return SHB_OK;
}

int shb_dense_dft_host(const double *state, uint64_t q, uint32_t tiles, int precision, double *out)
{
    if (!state || !out) return set_error(SHB_EINVAL, "null buffer");
    if (q < 2 || (q & (q - 1))) return set_error(SHB_EINVAL, "q must be a power of two >= 2, got %llu",
                                                 (unsigned long long)q);
    if (tiles < 1 || q % tiles) return set_error(SHB_EINVAL, "tiles %u does not divide q", tiles);
    return dft_host_common(state, q, 0, q, 0, q, tiles, 1.0 / sqrt((double)q), precision, out);
}

int shb_partial_row_sums_host(double *out, const double *state, const double *roots, uint64_t q,
                              uint64_t k0, uint64_t k1, uint64_t j0, uint64_t j1)
{
    if (!state || !out) return set_error(SHB_EINVAL, "null buffer");
    if (q < 2 || (q & (q - 1))) return set_error(SHB_EINVAL, "q must be a power of two >= 2");
    if (k1 < k0 || k1 > q || j1 < j0 || j1 > q) return set_error(SHB_EINVAL, "row/column range outside [0, q)");
    SHB_TRY(check_roots_table(roots, q));
    if (k1 == k0) return SHB_OK;
    if (j1 == j0) {
        memset(out, 0, (k1 - k0) * 16);
        return SHB_OK;
    }
    return dft_host_common(state + 2 * j0, j1 - j0, j0, q, k0, k1 - k0, 1, 1.0, SHB_FP64, out);
}

}  // extern "C"
