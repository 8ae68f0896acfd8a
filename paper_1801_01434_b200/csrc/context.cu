// The register handle (shb_ctx): one Shor attempt over device-resident,
// sharded state, driven from one host thread.
//
// Layout per shard g of G (devices may repeat):
//   residues  uint32[a_count]   a in [g*q/G, (g+1)*q/G)          (4 B / index)
//   support   uint64[m_g]       the shard's indices with residue k
//   spectrum  complex128[c_count], prob float64[c_count], per-CTA prob sums
//             c in [g*q/G, (g+1)*q/G)
// Cross-shard steps are tiny or copies: class counts are summed on the host,
// the support geometry (a0, stride) is combined with a host gcd, and the
// Born-rule read copies every shard's probabilities to shard 0's device
// (peer copy over NVLink when the devices differ) and runs the exact
// sequential-cumsum search there.  Every number is bitwise the same for any
// shard count: outputs are independent sums and the DFT engine is keyed on q.
#include <errno.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <vector>

#include "shb_internal.cuh"

using namespace shb;

namespace {

struct Shard {
    int dev = 0;
    cudaStream_t st = nullptr;
    uint64_t a_begin = 0, a_count = 0, c_begin = 0, c_count = 0;
    uint32_t *res = nullptr;
    std::vector<uint64_t> counts;  // host copy of this shard's class counts
    uint64_t *support = nullptr;
    uint64_t m = 0;
    double *spec = nullptr, *prob = nullptr, *bsums = nullptr;
    uint64_t nb = 0;
    void *recs = nullptr;      // split-cumsum records of this shard's probabilities
    double *tile_S = nullptr;  // exact running value at each of its tile starts
};

struct DeviceGuard {
    int prev = 0;
    DeviceGuard() { cudaGetDevice(&prev); }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// cudaMalloc with one retry after handing cached stream-ordered pool memory
// back (the scratch pool keeps its blocks mapped between calls).
int dev_alloc(void **p, size_t bytes)
{
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            cudaDeviceSynchronize();
            cudaMemPoolTrimTo(pool, 0);
        }
        e = cudaMalloc(p, bytes ? bytes : 16);
    }
    if (e != cudaSuccess) {
        *p = nullptr;
        return check_cuda(e, "cudaMalloc(register)");
    }
    return SHB_OK;
}

template <class T>
void dev_free(int dev, T *&p)
{
    if (p) {
        cudaSetDevice(dev);
        cudaFree(p);
        p = nullptr;
    }
}

}  // namespace

struct shb_ctx {
    std::vector<Shard> sh;
    int stage = 0;  // 0 empty, 1 entangled, 2 collapsed, 3 transformed
    uint64_t q = 0, x = 0, n = 0;
    uint32_t w = 0;
    bool counted = false;
    std::vector<uint64_t> counts;  // summed over shards, n entries
    uint32_t k = 0;
    uint64_t M = 0, a0 = 0, stride = 1, len = 0;
    double amp = 0.0;
    int precision = SHB_FP64;

    void release_from(int stage_keep)
    {
        DeviceGuard g;
        for (auto &s : sh) {
            if (stage_keep < 3) {
                dev_free(s.dev, s.spec);
                dev_free(s.dev, s.prob);
                dev_free(s.dev, s.bsums);
                dev_free(s.dev, s.recs);
                dev_free(s.dev, s.tile_S);
                s.nb = 0;
            }
            if (stage_keep < 2) {
                dev_free(s.dev, s.support);
                s.m = 0;
            }
            if (stage_keep < 1) {
                dev_free(s.dev, s.res);
                s.counts.clear();
            }
        }
        if (stage_keep < 1) {
            counted = false;
            counts.clear();
        }
        if (stage > stage_keep) stage = stage_keep;
    }

    int sync_all()
    {
        for (auto &s : sh) {
            SHB_TRY_CUDA(cudaSetDevice(s.dev));
            SHB_TRY_CUDA(cudaStreamSynchronize(s.st));
        }
        return SHB_OK;
    }
};

namespace {

int need(const shb_ctx *c, int stage, const char *what)
{
    if (!c) return set_error(SHB_EINVAL, "null register handle");
    if (c->stage < stage) {
        static const char *names[] = {"empty", "entangled", "collapsed", "transformed"};
        return set_error(SHB_EINVAL, "%s needs a %s register (current stage: %s)", what, names[stage],
                         names[c->stage]);
    }
    return SHB_OK;
}

int compute_counts(shb_ctx *c)
{
    if (c->counted) return SHB_OK;
    if (c->n > (1ull << 28)) return set_error(SHB_EINVAL, "class histogram is limited to n <= 2^28");
    DeviceGuard g;
    std::vector<uint64_t *> dcounts(c->sh.size(), nullptr);
    int rc = SHB_OK;
    for (size_t i = 0; i < c->sh.size() && rc == SHB_OK; i++) {
        Shard &s = c->sh[i];
        s.counts.assign(c->n, 0);
        if (!s.a_count) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        rc = dev_alloc((void **)&dcounts[i], c->n * 8);
        if (rc == SHB_OK) rc = check_cuda(cudaMemsetAsync(dcounts[i], 0, c->n * 8, s.st), "memset(counts)");
        if (rc == SHB_OK) rc = shb_class_counts(s.res, s.a_count, dcounts[i], c->n, s.st);
        if (rc == SHB_OK)
            rc = check_cuda(cudaMemcpyAsync(s.counts.data(), dcounts[i], c->n * 8, cudaMemcpyDeviceToHost, s.st),
                            "copy(counts)");
    }
    if (rc == SHB_OK) rc = c->sync_all();
    for (size_t i = 0; i < c->sh.size(); i++) dev_free(c->sh[i].dev, dcounts[i]);
    if (rc != SHB_OK) return rc;
    c->counts.assign(c->n, 0);
    for (auto &s : c->sh)
        for (uint64_t v = 0; v < c->n; v++) c->counts[v] += s.counts[v];
    c->counted = true;
    return SHB_OK;
}

}  // namespace

extern "C" {

int shb_init_devices(const int *devices, int ndev, shb_ctx **out)
{
    if (!out) return set_error(SHB_EINVAL, "null output handle");
    *out = nullptr;
    if (!devices || ndev < 1 || ndev > 1024) return set_error(SHB_EINVAL, "need 1..1024 devices, got %d", ndev);
    int count = 0;
    SHB_TRY_CUDA(cudaGetDeviceCount(&count));
    for (int i = 0; i < ndev; i++)
        if (devices[i] < 0 || devices[i] >= count)
            return set_error(SHB_EINVAL, "device %d is not visible (%d devices)", devices[i], count);
    DeviceGuard g;
    shb_ctx *c = new shb_ctx;
    c->sh.resize(ndev);
    for (int i = 0; i < ndev; i++) {
        Shard &s = c->sh[i];
        s.dev = devices[i];
        cudaError_t e = cudaSetDevice(s.dev);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            shb_free(c);
            return check_cuda(e, "shb_init: stream");
        }
        // shard 0 reads every shard's probabilities: map peers where the hardware allows
        if (s.dev != devices[0]) {
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, devices[0], s.dev);
            if (ok) {
                cudaSetDevice(devices[0]);
                if (cudaDeviceEnablePeerAccess(s.dev, 0) != cudaSuccess) cudaGetLastError();
            }
        }
    }
    *out = c;
    return SHB_OK;
}

int shb_init(int ngpu, shb_ctx **out)
{
    int count = 0;
    SHB_TRY_CUDA(cudaGetDeviceCount(&count));
    if (ngpu <= 0) ngpu = count;
    if (ngpu > count) return set_error(SHB_EINVAL, "asked for %d devices, %d visible", ngpu, count);
    std::vector<int> devs(ngpu);
    for (int i = 0; i < ngpu; i++) devs[i] = i;
    return shb_init_devices(devs.data(), ngpu, out);
}

void shb_free(shb_ctx *c)
{
    if (!c) return;
    c->release_from(0);
    DeviceGuard g;
    for (auto &s : c->sh)
        if (s.st) {
            cudaSetDevice(s.dev);
            cudaStreamDestroy(s.st);
        }
    delete c;
}

int shb_ctx_state(const shb_ctx *c, int *stage, uint64_t *q, uint64_t *n, int *nshards)
{
    if (!c) return set_error(SHB_EINVAL, "null register handle");
    if (stage) *stage = c->stage;
    if (q) *q = c->q;
    if (n) *n = c->n;
    if (nshards) *nshards = (int)c->sh.size();
    return SHB_OK;
}

int shb_ctx_modexp(shb_ctx *c, uint64_t x, uint64_t n, uint32_t w)
{
    if (!c) return set_error(SHB_EINVAL, "null register handle");
    if (w < 1 || w > 32) return set_error(SHB_EINVAL, "register width %u outside [1, 32]", w);
    if (n < 2) return set_error(SHB_EINVAL, "modulus must be >= 2");
    if (n > 0xFFFFFFFFull) return set_error(SHB_EINVAL, "modulus %llu exceeds 32-bit residue storage",
                                            (unsigned long long)n);
    if (gcd_u64(x, n) != 1)
        return set_error(SHB_EINVAL, "x=%llu shares a factor with n=%llu", (unsigned long long)x,
                         (unsigned long long)n);
    c->release_from(0);
    c->q = 1ull << w;
    c->w = w;
    c->x = x;
    c->n = n;
    const uint64_t G = c->sh.size();
    DeviceGuard g;
    for (uint64_t i = 0; i < G; i++) {
        Shard &s = c->sh[i];
        s.a_begin = c->q * i / G;
        s.a_count = c->q * (i + 1) / G - s.a_begin;
        s.c_begin = s.a_begin;
        s.c_count = s.a_count;
        if (!s.a_count) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY(dev_alloc((void **)&s.res, s.a_count * 4));
        SHB_TRY(shb_modexp(s.res, s.a_begin, s.a_count, x, n, s.st));
    }
    SHB_TRY(c->sync_all());
    c->stage = 1;
    return SHB_OK;
}

int shb_ctx_class_counts(shb_ctx *c, uint64_t *counts_out, uint64_t ncls)
{
    SHB_TRY(need(c, 1, "shb_ctx_class_counts"));
    if (!counts_out) return set_error(SHB_EINVAL, "null counts buffer");
    if (ncls < c->n)
        return set_error(SHB_ERANGE, "counts capacity %llu is below the modulus %llu", (unsigned long long)ncls,
                         (unsigned long long)c->n);
    SHB_TRY(compute_counts(c));
    memcpy(counts_out, c->counts.data(), c->n * 8);
    if (ncls > c->n) memset(counts_out + c->n, 0, (ncls - c->n) * 8);
    return SHB_OK;
}

int shb_collapse(shb_ctx *c, uint32_t k, uint64_t *M_out, double *amp_out)
{
    SHB_TRY(need(c, 1, "shb_collapse"));
    if (c->stage >= 2) return set_error(SHB_EINVAL, "part 2 was already measured");
    if (k >= c->n) return set_error(SHB_EINVAL, "outcome k=%u is not a residue mod n=%llu", k,
                                    (unsigned long long)c->n);
    SHB_TRY(compute_counts(c));
    const uint64_t M = c->counts[k];
    if (M == 0) return set_error(SHB_EINVAL, "outcome k=%u has probability 0", k);
    // the amplitude exactly as measure_part2 rounds it: the host half of the
    // recipe evaluated at this k (counts of other classes do not enter it)
    const double a = 1.0 / sqrt((double)c->q);
    const double kept = sqrt(shb_host_pairwise_sum_const(a * a, M));
    const double amp = a * (1.0 / kept);

    c->release_from(1);  // a failed earlier collapse may have left shard supports
    DeviceGuard g;
    for (auto &s : c->sh) {
        s.m = 0;
        const uint64_t cap = s.counts[k];
        if (!cap) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY(dev_alloc((void **)&s.support, cap * 8));
        SHB_TRY(shb_compact_eq(s.res, s.a_count, k, s.a_begin, s.support, cap, &s.m, s.st));
        if (s.m != cap) return set_error(SHB_ECUDA, "compaction found %llu of %llu indices",
                                         (unsigned long long)s.m, (unsigned long long)cap);
    }
    // support geometry: per-shard progressions joined by a host gcd over the
    // shard strides and the gaps between consecutive shards
    uint64_t a0 = 0, stride = 0, last = 0;
    bool first = true;
    for (auto &s : c->sh) {
        if (!s.m) continue;
        uint64_t b0 = 0, bs = 1, bl = 0;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY(shb_support_progression(s.support, s.m, &b0, &bs, &bl, s.st));
        if (bl != s.m) return set_error(SHB_ECUDA, "shard support is not an arithmetic progression");
        if (first) {
            a0 = b0;
            first = false;
        } else {
            stride = gcd_u64(stride, b0 - last);
        }
        if (s.m > 1) stride = gcd_u64(stride, bs);
        last = b0 + (s.m - 1) * bs;
    }
    if (stride == 0) stride = 1;
    const uint64_t len = (last - a0) / stride + 1;
    // {a : x^a = k (mod n)} is a full comb of stride ord(x); anything else is a bug
    if (len != M) return set_error(SHB_ECUDA, "collapsed support (M=%llu) does not fill its progression (%llu)",
                                   (unsigned long long)M, (unsigned long long)len);
    c->k = k;
    c->M = M;
    c->amp = amp;
    c->a0 = a0;
    c->stride = stride;
    c->len = len;
    c->stage = 2;
    if (M_out) *M_out = M;
    if (amp_out) *amp_out = amp;
    return SHB_OK;
}

int shb_measure(shb_ctx *c, double u, uint32_t *k_out, uint64_t *M_out, double *amp_out)
{
    SHB_TRY(need(c, 1, "shb_measure"));
    if (c->stage >= 2) return set_error(SHB_EINVAL, "part 2 was already measured");
    SHB_TRY(compute_counts(c));
    uint32_t k = 0;
    uint64_t M = 0;
    double amp = 0.0;
    SHB_TRY(shb_host_measure_class(c->counts.data(), c->n, c->q, u, &k, &M, &amp));
    uint64_t M2 = 0;
    double amp2 = 0.0;
    SHB_TRY(shb_collapse(c, k, &M2, &amp2));
    if (M2 != M || amp2 != amp) return set_error(SHB_ECUDA, "collapse disagrees with the class draw");
    if (k_out) *k_out = k;
    if (M_out) *M_out = M;
    if (amp_out) *amp_out = amp;
    return SHB_OK;
}

int shb_ctx_dft(shb_ctx *c, int precision, uint32_t tiles)
{
    SHB_TRY(need(c, 2, "shb_ctx_dft"));
    if (c->stage >= 3) return set_error(SHB_EINVAL, "the register was already transformed");
    if (precision != SHB_FP64 && precision != SHB_FP32) return set_error(SHB_EINVAL, "unknown precision %d",
                                                                          precision);
    if (tiles < 1 || c->q % tiles) return set_error(SHB_EINVAL, "tiles %u does not divide q=%llu", tiles,
                                                    (unsigned long long)c->q);
    const double scale = 1.0 / sqrt((double)c->q);
    c->release_from(2);
    DeviceGuard g;
    for (auto &s : c->sh) {
        if (!s.c_count) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        s.nb = shb_dft_num_blocks(s.c_count, precision);
        SHB_TRY(dev_alloc((void **)&s.spec, s.c_count * 16));
        SHB_TRY(dev_alloc((void **)&s.prob, s.c_count * 8));
        SHB_TRY(dev_alloc((void **)&s.bsums, (s.nb ? s.nb : 1) * 8));
        // launch every shard before waiting on any: distinct devices run concurrently
        SHB_TRY(shb_dft_uniform(c->amp, 0.0, c->len, c->a0, c->stride, c->q, s.c_begin, s.c_count, tiles, scale,
                                precision, s.spec, s.prob, s.bsums, s.st));
    }
    SHB_TRY(c->sync_all());
    c->precision = precision;
    c->stage = 3;
    return SHB_OK;
}

int shb_norm(shb_ctx *c, double *out)
{
    SHB_TRY(need(c, 1, "shb_norm"));
    if (!out) return set_error(SHB_EINVAL, "null output");
    if (c->stage == 1) {  // the uniform register: sqrt(q) * 1/sqrt(q)
        *out = sqrt((double)c->q) * (1.0 / sqrt((double)c->q));
        return SHB_OK;
    }
    if (c->stage == 2) {
        *out = sqrt((double)c->M) * fabs(c->amp);
        return SHB_OK;
    }
    DeviceGuard g;
    double total = 0.0;
    for (auto &s : c->sh) {
        if (!s.c_count) continue;
        double part = 0.0;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY(shb_sum(s.bsums, s.nb, &part, s.st));
        total += part;
    }
    *out = sqrt(total);
    return SHB_OK;
}

int shb_sample(shb_ctx *c, double u, uint64_t *m_out)
{
    SHB_TRY(need(c, 3, "shb_sample"));
    if (!m_out) return set_error(SHB_EINVAL, "null output");
    double norm = 0.0;
    SHB_TRY(shb_norm(c, &norm));
    const double tol = c->precision == SHB_FP64 ? 1e-9 : 1e-4;  // _NORM_TOL (qstate.py:17) / FP32 accuracy
    if (!(fabs(norm - 1.0) <= tol)) return set_error(SHB_EINVAL, "register is not normalized (|amp| = %.17g)", norm);
    // The exact sequential CDF over the c-shards without moving the
    // probabilities: every shard builds its binade records at once (from a hint
    // of the value entering it: the approximate sums of the shards before it),
    // then the exact running value is carried shard to shard through the
    // records-driven walk, and the shard that first passes u * total is
    // searched (the same split as distributed._sharded_sample).
    DeviceGuard g;
    std::vector<double> approx(c->sh.size(), 0.0);
    for (size_t i = 0; i < c->sh.size(); i++) {
        Shard &s = c->sh[i];
        if (!s.c_count) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY(shb_sum(s.prob, s.c_count, &approx[i], s.st));
    }
    double hint = 0.0;
    for (size_t i = 0; i < c->sh.size(); i++) {
        Shard &s = c->sh[i];
        if (s.c_count) {
            SHB_TRY_CUDA(cudaSetDevice(s.dev));
            const uint64_t nt = shb_cumsum_tiles(s.c_count);
            if (!s.recs) SHB_TRY(dev_alloc(&s.recs, nt * shb_cumsum_record_bytes()));
            if (!s.tile_S) SHB_TRY(dev_alloc((void **)&s.tile_S, nt * sizeof(double)));
            SHB_TRY(shb_cumsum_records(s.prob, s.c_count, hint, s.recs, s.st));  // async on every device
        }
        hint += approx[i];
    }
    std::vector<double> enter(c->sh.size(), 0.0), leave(c->sh.size(), 0.0);
    double run = 0.0;
    for (size_t i = 0; i < c->sh.size(); i++) {
        Shard &s = c->sh[i];
        enter[i] = run;
        if (s.c_count) {
            SHB_TRY_CUDA(cudaSetDevice(s.dev));
            SHB_TRY(shb_cumsum_walk(s.prob, s.c_count, s.recs, run, s.tile_S, &run, s.st));
        }
        leave[i] = run;
    }
    const double target = u * run;  // s.uniform() * cum[-1] (qstate.py:113)
    uint64_t idx = c->q;
    for (size_t i = 0; i < c->sh.size(); i++) {
        Shard &s = c->sh[i];
        if (!s.c_count || !(leave[i] > target)) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        uint64_t local = 0;
        SHB_TRY(shb_cumsum_find(s.prob, s.c_count, s.tile_S, leave[i], target, &local, s.st));
        idx = s.c_begin + local;
        break;
    }
    *m_out = idx < c->q - 1 ? idx : c->q - 1;
    return SHB_OK;
}

int shb_copy_spectrum(shb_ctx *c, uint64_t c0, uint64_t c1, double *host)
{
    SHB_TRY(need(c, 3, "shb_copy_spectrum"));
    if (c1 < c0 || c1 > c->q) return set_error(SHB_EINVAL, "rows [%llu, %llu) outside [0, q)",
                                               (unsigned long long)c0, (unsigned long long)c1);
    if (c1 > c0 && !host) return set_error(SHB_EINVAL, "null output");
    DeviceGuard g;
    for (auto &s : c->sh) {
        const uint64_t lo = c0 > s.c_begin ? c0 : s.c_begin;
        const uint64_t hi = c1 < s.c_begin + s.c_count ? c1 : s.c_begin + s.c_count;
        if (lo >= hi) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY_CUDA(cudaMemcpyAsync(host + 2 * (lo - c0), s.spec + 2 * (lo - s.c_begin), (hi - lo) * 16,
                                     cudaMemcpyDeviceToHost, s.st));
    }
    return c->sync_all();
}

int shb_copy_support(shb_ctx *c, uint64_t *host, uint64_t capacity, uint64_t *m_out)
{
    SHB_TRY(need(c, 2, "shb_copy_support"));
    if (m_out) *m_out = c->M;
    if (capacity < c->M) return set_error(SHB_ERANGE, "support has %llu entries, capacity %llu",
                                          (unsigned long long)c->M, (unsigned long long)capacity);
    if (c->M && !host) return set_error(SHB_EINVAL, "null output");
    DeviceGuard g;
    uint64_t off = 0;
    for (auto &s : c->sh) {
        if (!s.m) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        SHB_TRY_CUDA(cudaMemcpyAsync(host + off, s.support, s.m * 8, cudaMemcpyDeviceToHost, s.st));
        off += s.m;
    }
    return c->sync_all();
}

int shb_copy_residues(shb_ctx *c, uint64_t a0, uint64_t a1, int64_t *host)
{
    SHB_TRY(need(c, 1, "shb_copy_residues"));
    if (a1 < a0 || a1 > c->q) return set_error(SHB_EINVAL, "indices [%llu, %llu) outside [0, q)",
                                               (unsigned long long)a0, (unsigned long long)a1);
    if (a1 > a0 && !host) return set_error(SHB_EINVAL, "null output");
    DeviceGuard g;
    const uint64_t chunk = 1ull << 22;
    std::vector<uint32_t> buf;
    for (auto &s : c->sh) {
        const uint64_t lo = a0 > s.a_begin ? a0 : s.a_begin;
        const uint64_t hi = a1 < s.a_begin + s.a_count ? a1 : s.a_begin + s.a_count;
        if (lo >= hi) continue;
        SHB_TRY_CUDA(cudaSetDevice(s.dev));
        for (uint64_t p = lo; p < hi; p += chunk) {
            const uint64_t e = hi - p < chunk ? hi - p : chunk;
            buf.resize(e);
            SHB_TRY_CUDA(cudaMemcpyAsync(buf.data(), s.res + (p - s.a_begin), e * 4, cudaMemcpyDeviceToHost, s.st));
            SHB_TRY_CUDA(cudaStreamSynchronize(s.st));
            for (uint64_t i = 0; i < e; i++) host[p - a0 + i] = (int64_t)buf[i];
        }
    }
    return SHB_OK;
}

int shb_dump_state(shb_ctx *c, const char *path)
{
    SHB_TRY(need(c, 3, "shb_dump_state"));
    if (!path) return set_error(SHB_EINVAL, "null path");
    FILE *f = fopen(path, "wb");
    if (!f) return set_error(SHB_EIO, "cannot open %s: %s", path, strerror(errno));
    // qstate.py:18-20: magic, version 1, width, reserved (little-endian u32s)
    unsigned char hdr[16] = {'Q', 'R', 'E', 'G'};
    const uint32_t fields[3] = {1u, c->w, 0u};
    for (int i = 0; i < 3; i++)
        for (int b = 0; b < 4; b++) hdr[4 + 4 * i + b] = (unsigned char)(fields[i] >> (8 * b));
    int rc = fwrite(hdr, 1, 16, f) == 16 ? SHB_OK : set_error(SHB_EIO, "write %s failed", path);
    const uint64_t chunk = 1ull << 22;  // 64 MiB of complex128 per copy
    std::vector<double> buf;
    DeviceGuard g;
    for (auto &s : c->sh) {
        if (rc != SHB_OK) break;
        if (cudaSetDevice(s.dev) != cudaSuccess) {
            rc = check_cuda(cudaGetLastError(), "cudaSetDevice");
            break;
        }
        for (uint64_t p = 0; p < s.c_count && rc == SHB_OK; p += chunk) {
            const uint64_t e = s.c_count - p < chunk ? s.c_count - p : chunk;
            buf.resize(2 * e);
            rc = check_cuda(cudaMemcpy(buf.data(), s.spec + 2 * p, e * 16, cudaMemcpyDeviceToHost), "copy(spectrum)");
            if (rc == SHB_OK && fwrite(buf.data(), 16, e, f) != e) rc = set_error(SHB_EIO, "write %s failed", path);
        }
    }
    if (fclose(f) != 0 && rc == SHB_OK) rc = set_error(SHB_EIO, "close %s failed", path);
    return rc;
}

}  // extern "C"
