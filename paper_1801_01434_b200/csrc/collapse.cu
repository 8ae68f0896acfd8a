// Stage 2 of the hot path: measurement collapse of part 2
// (qstate.measure_part2, qstate.py:86-105) -- stream compaction of
// {a : residues[a] == k} -- and the support-geometry reductions that turn a
// support (or the nonzero pattern of a dense state) into the arithmetic
// progression the DFT kernel walks.
//
// Compaction is two-pass and deterministic: pass 1 counts matches per
// 4096-element tile (warp ballot + popc), a single-CTA scan turns the counts
// into output offsets, pass 2 re-derives each warp's match masks and writes
// indices in ascending order.  HBM-bound: 4 B read per exponent per pass,
// 8 B written per support element.
#include "shb_internal.cuh"

namespace shb {

constexpr int CMP_THREADS = 256;
constexpr int CMP_ITEMS = 16;                                // per lane
constexpr int CMP_TILE = CMP_THREADS * CMP_ITEMS;            // 4096
constexpr int CMP_WARP_SPAN = 32 * CMP_ITEMS;                // 512 per warp

__global__ void __launch_bounds__(CMP_THREADS)
    compact_count_kernel(const uint32_t *__restrict__ res, uint64_t count, uint32_t k,
                         uint32_t *__restrict__ tile_counts)
{
    __shared__ uint32_t warp_cnt[CMP_THREADS / 32];
    const uint64_t tile0 = (uint64_t)blockIdx.x * CMP_TILE;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t w0 = tile0 + (uint64_t)wid * CMP_WARP_SPAN;
    uint32_t c = 0;
#pragma unroll
    for (int it = 0; it < CMP_ITEMS; it++) {
        const uint64_t i = w0 + (uint64_t)it * 32 + lane;
        const bool hit = (i < count) && (res[i] == k);
        c += __popc(__ballot_sync(0xffffffffu, hit));
    }
    if (lane == 0) warp_cnt[wid] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < CMP_THREADS / 32; w++) t += warp_cnt[w];
        tile_counts[blockIdx.x] = t;
    }
}

// Exclusive scan of the tile counts (one CTA; ~1M tiles at q = 2^32).
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS)
    tile_scan_kernel(const uint32_t *__restrict__ counts, uint64_t ntiles,
                     uint64_t *__restrict__ offsets, uint64_t *__restrict__ total)
{
    __shared__ uint64_t warp_tmp[SCAN_THREADS / 32];
    const uint64_t per = (ntiles + SCAN_THREADS - 1) / SCAN_THREADS;
    const uint64_t lo = per * threadIdx.x;
    const uint64_t hi = lo + per < ntiles ? lo + per : ntiles;
    uint64_t s = 0;
    for (uint64_t i = lo; i < hi; i++) s += counts[i];
    uint64_t tot;
    uint64_t run = block_exclusive_scan_u64<SCAN_THREADS>(s, warp_tmp, tot);
    for (uint64_t i = lo; i < hi; i++) {
        offsets[i] = run;
        run += counts[i];
    }
    if (threadIdx.x == 0) *total = tot;
}

__global__ void __launch_bounds__(CMP_THREADS)
    compact_write_kernel(const uint32_t *__restrict__ res, uint64_t count, uint32_t k,
                         uint64_t a_begin, const uint64_t *__restrict__ tile_offsets,
                         uint64_t *__restrict__ support)
{
    __shared__ uint32_t warp_cnt[CMP_THREADS / 32];
    const uint64_t tile0 = (uint64_t)blockIdx.x * CMP_TILE;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t w0 = tile0 + (uint64_t)wid * CMP_WARP_SPAN;
    uint32_t masks[CMP_ITEMS];
    uint32_t c = 0;
#pragma unroll
    for (int it = 0; it < CMP_ITEMS; it++) {
        const uint64_t i = w0 + (uint64_t)it * 32 + lane;
        const bool hit = (i < count) && (res[i] == k);
        masks[it] = __ballot_sync(0xffffffffu, hit);
        c += __popc(masks[it]);
    }
    if (lane == 0) warp_cnt[wid] = c;
    __syncthreads();
    uint64_t off = tile_offsets[blockIdx.x];
    for (int w = 0; w < wid; w++) off += warp_cnt[w];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int it = 0; it < CMP_ITEMS; it++) {
        const uint32_t m = masks[it];
        if (m & (1u << lane)) support[off + __popc(m & lt)] = a_begin + w0 + (uint64_t)it * 32 + lane;
        off += __popc(m);
    }
}

// ----------------------------------------------------- progression geometry
struct Geo {
    uint64_t first, last, g;  // first = UINT64_MAX when empty
};

__device__ inline Geo geo_merge(Geo a, Geo b)
{
    if (a.first == ~0ull) return b;
    if (b.first == ~0ull) return a;
    Geo r;
    r.first = a.first < b.first ? a.first : b.first;
    r.last = a.last > b.last ? a.last : b.last;
    uint64_t g = gcd_u64(a.g, b.g);
    g = gcd_u64(g, a.first - r.first);
    g = gcd_u64(g, b.first - r.first);
    r.g = g;
    return r;
}

__device__ inline Geo geo_shfl(Geo v, int o)
{
    Geo r;
    r.first = __shfl_down_sync(0xffffffffu, v.first, o);
    r.last = __shfl_down_sync(0xffffffffu, v.last, o);
    r.g = __shfl_down_sync(0xffffffffu, v.g, o);
    return r;
}

template <int NT>
__device__ inline Geo geo_block_reduce(Geo v)
{
    __shared__ Geo tmp[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = geo_merge(v, geo_shfl(v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) tmp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = (lane < NT / 32) ? tmp[lane] : Geo{~0ull, 0, 0};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = geo_merge(v, geo_shfl(v, o));
    }
    return v;
}

__device__ inline void geo_add(Geo &t, uint64_t idx)
{
    if (t.first == ~0ull) {
        t.first = idx;
        t.last = idx;
        t.g = 0;
    } else {
        t.g = gcd_u64(t.g, idx - t.last);
        t.last = idx;
    }
}

constexpr int GEO_THREADS = 256;

__global__ void __launch_bounds__(GEO_THREADS)
    support_geo_kernel(const uint64_t *__restrict__ s, uint64_t m, Geo *__restrict__ part)
{
    Geo t{~0ull, 0, 0};
    const uint64_t stride = (uint64_t)gridDim.x * GEO_THREADS;
    // indices seen by one thread ascend, so consecutive gaps suffice
    for (uint64_t i = (uint64_t)blockIdx.x * GEO_THREADS + threadIdx.x; i < m; i += stride) geo_add(t, s[i]);
    Geo b = geo_block_reduce<GEO_THREADS>(t);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void __launch_bounds__(GEO_THREADS)
    state_geo_kernel(const double2 *__restrict__ st, uint64_t q, Geo *__restrict__ part)
{
    Geo t{~0ull, 0, 0};
    const uint64_t stride = (uint64_t)gridDim.x * GEO_THREADS;
    for (uint64_t i = (uint64_t)blockIdx.x * GEO_THREADS + threadIdx.x; i < q; i += stride) {
        const double2 v = st[i];
        if (v.x != 0.0 || v.y != 0.0) geo_add(t, i);
    }
    Geo b = geo_block_reduce<GEO_THREADS>(t);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
}

static int finish_geo(const Geo *d_part, int nblk, cudaStream_t st, uint64_t *a0, uint64_t *stride,
                      uint64_t *length)
{
    Geo h[1024];
    SHB_TRY_CUDA(cudaMemcpyAsync(h, d_part, sizeof(Geo) * nblk, cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    uint64_t first = ~0ull, last = 0;
    for (int b = 0; b < nblk; b++)
        if (h[b].first != ~0ull) {
            if (h[b].first < first) first = h[b].first;
            if (h[b].last > last) last = h[b].last;
        }
    if (first == ~0ull) {
        *a0 = 0;
        *stride = 1;
        *length = 0;
        return SHB_OK;
    }
    uint64_t g = 0;
    for (int b = 0; b < nblk; b++)
        if (h[b].first != ~0ull) g = gcd_u64(gcd_u64(g, h[b].g), h[b].first - first);
    if (g == 0) g = 1;  // single element
    *a0 = first;
    *stride = g;
    *length = (last - first) / g + 1;
    return SHB_OK;
}

__global__ void gather_prog_kernel(const double2 *__restrict__ st, uint64_t a0, uint64_t stride,
                                   uint64_t len, double2 *__restrict__ amps)
{
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += step)
        amps[j] = st[a0 + j * stride];
}

__global__ void fill_const_kernel(double2 *__restrict__ amps, uint64_t len, double2 v)
{
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += step) amps[j] = v;
}

__global__ void scatter_support_kernel(const uint64_t *__restrict__ s, uint64_t m, uint64_t a0,
                                       uint64_t stride, double2 *__restrict__ amps, double2 v)
{
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += step)
        amps[(s[i] - a0) / stride] = v;
}

// all amplitudes of a progression equal to the first one?
__global__ void uniform_check_kernel(const double2 *__restrict__ amps, uint64_t len, unsigned int *__restrict__ diff)
{
    const double2 a0 = amps[0];
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    bool d = false, cplx = false;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += step) {
        const double2 v = amps[j];
        // bitwise comparison: -0.0 and +0.0 or NaN payloads are not "equal"
        d |= (__double_as_longlong(v.x) != __double_as_longlong(a0.x)) ||
             (__double_as_longlong(v.y) != __double_as_longlong(a0.y));
        cplx |= !(v.y == 0.0);  // bit 1: some imaginary part is nonzero (or NaN)
    }
    const bool bd = __syncthreads_or(d), bc = __syncthreads_or(cplx);
    if (threadIdx.x == 0 && (bd || bc)) atomicOr(diff, (bd ? 1u : 0u) | (bc ? 2u : 0u));
}

static unsigned grid_for(uint64_t n, int threads, int per_sm)
{
    uint64_t b = (n + threads - 1) / threads;
    const uint64_t cap = (uint64_t)sm_count() * per_sm;
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (unsigned)b;
}

}  // namespace shb

using namespace shb;

extern "C" int shb_compact_eq(const uint32_t *d_residues, uint64_t count, uint32_t k, uint64_t a_begin,
                              uint64_t *d_support, uint64_t capacity, uint64_t *m_out, void *stream)
{
    if (!m_out) return set_error(SHB_EINVAL, "null m_out");
    *m_out = 0;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    const uint64_t ntiles = (count + CMP_TILE - 1) / CMP_TILE;
    if (ntiles > 0x7FFFFFFFull) return set_error(SHB_EINVAL, "register too large for one compaction");
    Scratch counts, offsets, total;
    SHB_TRY(scratch_alloc(counts, ntiles * sizeof(uint32_t), st));
    SHB_TRY(scratch_alloc(offsets, ntiles * sizeof(uint64_t), st));
    SHB_TRY(scratch_alloc(total, sizeof(uint64_t), st));
    compact_count_kernel<<<(unsigned)ntiles, CMP_THREADS, 0, st>>>(d_residues, count, k, (uint32_t *)counts.ptr);
    SHB_LAUNCHED();
    tile_scan_kernel<<<1, SCAN_THREADS, 0, st>>>((const uint32_t *)counts.ptr, ntiles, (uint64_t *)offsets.ptr,
                                                 (uint64_t *)total.ptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    uint64_t M = 0;
    SHB_TRY_CUDA(cudaMemcpyAsync(&M, total.ptr, sizeof M, cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    *m_out = M;
    if (M > capacity)
        return set_error(SHB_ERANGE, "support of %llu entries exceeds capacity %llu", (unsigned long long)M,
                         (unsigned long long)capacity);
    if (M == 0) return SHB_OK;
    compact_write_kernel<<<(unsigned)ntiles, CMP_THREADS, 0, st>>>(d_residues, count, k, a_begin,
                                                                   (const uint64_t *)offsets.ptr, d_support);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

extern "C" int shb_support_progression(const uint64_t *d_support, uint64_t m, uint64_t *a0, uint64_t *stride,
                                       uint64_t *length, void *stream)
{
    if (!a0 || !stride || !length) return set_error(SHB_EINVAL, "null output");
    cudaStream_t st = as_stream(stream);
    if (m == 0) {
        *a0 = 0;
        *stride = 1;
        *length = 0;
        return SHB_OK;
    }
    const unsigned nblk = grid_for(m, GEO_THREADS, 4) > 1024 ? 1024 : grid_for(m, GEO_THREADS, 4);
    Scratch part;
    SHB_TRY(scratch_alloc(part, sizeof(Geo) * nblk, st));
    support_geo_kernel<<<nblk, GEO_THREADS, 0, st>>>(d_support, m, (Geo *)part.ptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return finish_geo((const Geo *)part.ptr, (int)nblk, st, a0, stride, length);
}

extern "C" int shb_state_progression(const double *d_state, uint64_t q, uint64_t *a0, uint64_t *stride,
                                     uint64_t *length, void *stream)
{
    if (!a0 || !stride || !length) return set_error(SHB_EINVAL, "null output");
    cudaStream_t st = as_stream(stream);
    if (q == 0) {
        *a0 = 0;
        *stride = 1;
        *length = 0;
        return SHB_OK;
    }
    const unsigned g = grid_for(q, GEO_THREADS, 4);
    const unsigned nblk = g > 1024 ? 1024 : g;
    Scratch part;
    SHB_TRY(scratch_alloc(part, sizeof(Geo) * nblk, st));
    state_geo_kernel<<<nblk, GEO_THREADS, 0, st>>>((const double2 *)d_state, q, (Geo *)part.ptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return finish_geo((const Geo *)part.ptr, (int)nblk, st, a0, stride, length);
}

extern "C" int shb_gather_progression(const double *d_state, uint64_t a0, uint64_t stride, uint64_t length,
                                      double *d_amps, void *stream)
{
    if (length == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    gather_prog_kernel<<<grid_for(length, 256, 8), 256, 0, st>>>((const double2 *)d_state, a0, stride, length,
                                                                (double2 *)d_amps);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

extern "C" int shb_progression_kind(const double *d_amps, uint64_t length, int *uniform, int *real,
                                    double *amp_re, double *amp_im, void *stream)
{
    if (!uniform) return set_error(SHB_EINVAL, "null output");
    *uniform = 0;
    if (real) *real = 1;
    if (length == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    Scratch diff;
    SHB_TRY(scratch_alloc(diff, sizeof(unsigned int), st));
    SHB_TRY_CUDA(cudaMemsetAsync(diff.ptr, 0, sizeof(unsigned int), st));
    uniform_check_kernel<<<grid_for(length, 256, 8), 256, 0, st>>>((const double2 *)d_amps, length,
                                                                  (unsigned int *)diff.ptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    unsigned int h = 1;
    double a[2] = {0.0, 0.0};
    SHB_TRY_CUDA(cudaMemcpyAsync(&h, diff.ptr, sizeof h, cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaMemcpyAsync(a, d_amps, sizeof a, cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    *uniform = (h & 1u) ? 0 : 1;
    if (real) *real = (h & 2u) ? 0 : 1;
    if (amp_re) *amp_re = a[0];
    if (amp_im) *amp_im = a[1];
    return SHB_OK;
}

extern "C" int shb_progression_is_uniform(const double *d_amps, uint64_t length, int *uniform, double *amp_re,
                                          double *amp_im, void *stream)
{
    return shb_progression_kind(d_amps, length, uniform, nullptr, amp_re, amp_im, stream);
}

extern "C" int shb_fill_progression(const uint64_t *d_support, uint64_t m, uint64_t a0, uint64_t stride,
                                    uint64_t length, double amp_re, double amp_im, double *d_amps, void *stream)
{
    if (length == 0) return SHB_OK;
    if (stride == 0) return set_error(SHB_EINVAL, "stride must be >= 1");
    cudaStream_t st = as_stream(stream);
    const double2 v = make_double2(amp_re, amp_im);
    if (m == length) {  // a full comb: every progression slot is occupied
        fill_const_kernel<<<grid_for(length, 256, 8), 256, 0, st>>>((double2 *)d_amps, length, v);
        SHB_LAUNCHED();
    } else {
        SHB_TRY_CUDA(cudaMemsetAsync(d_amps, 0, length * 16, st));
        scatter_support_kernel<<<grid_for(m, 256, 8), 256, 0, st>>>(d_support, m, a0, stride, (double2 *)d_amps, v);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}
