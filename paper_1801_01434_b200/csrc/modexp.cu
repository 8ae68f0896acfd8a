// Stage 1 of the hot path: part 2 of the register, residues[a] = x^a mod n
// (qstate.entangle_modexp, qstate.py:64-83), plus the exact residue-class
// histogram that measure_part2 needs (qstate.py:95-97).
//
// HBM-bound: 4 bytes written per exponent (uint32 residues; n < 2^32).
// Each warp owns a contiguous span of exponents; lane l seeds x^(a0+l) by
// square-and-multiply, then every lane steps by x^32 so that one warp store
// covers 32 consecutive residues (128 B, fully coalesced).  The modular
// product uses Barrett reduction: 32-bit when n < 2^16 (every config of the
// paper path: q >= n^2 and q <= 2^32), 64-bit otherwise.
#include "shb_internal.cuh"

namespace shb {

struct Barrett64 {
    uint64_t n, mu;  // mu = floor((2^64 - 1) / n)
    __device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b) const
    {
        const uint64_t t = a * b;  // a, b < n < 2^32 -> exact
        const uint64_t qh = __umul64hi(t, mu);
        uint64_t r = t - qh * n;
        if (r >= n) r -= n;
        if (r >= n) r -= n;
        return r;
    }
};

struct Barrett32 {
    uint32_t n, mu;  // mu = floor((2^32 - 1) / n), n < 2^16
    __device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b) const
    {
        const uint32_t t = (uint32_t)a * (uint32_t)b;  // < 2^32
        const uint32_t qh = __umulhi(t, mu);
        uint32_t r = t - qh * n;
        if (r >= n) r -= n;
        if (r >= n) r -= n;
        return r;
    }
};

template <class R>
__device__ __forceinline__ uint64_t powmod(const R &red, uint64_t base, uint64_t e, uint64_t one)
{
    uint64_t acc = one;
    while (e) {
        if (e & 1) acc = red.mulmod(acc, base);
        base = red.mulmod(base, base);
        e >>= 1;
    }
    return acc;
}

constexpr int MODEXP_THREADS = 256;
constexpr int MODEXP_ITERS = 64;  // residues per lane per warp span -> 2048 per warp

template <class R>
__global__ void __launch_bounds__(MODEXP_THREADS)
    modexp_kernel(uint32_t *__restrict__ out, uint64_t a_begin, uint64_t count, uint64_t xm,
                  uint64_t x32, uint64_t xjump, R red, uint64_t one)
{
    const uint64_t span = 32ull * MODEXP_ITERS;
    const uint64_t warp = (uint64_t)blockIdx.x * (MODEXP_THREADS / 32) + (threadIdx.x >> 5);
    const uint64_t nwarps = (uint64_t)gridDim.x * (MODEXP_THREADS / 32);
    const int lane = threadIdx.x & 31;
    uint64_t w0 = warp * span;
    if (w0 >= count) return;
    // seed once by square-and-multiply; later spans jump by x^(nwarps*span)
    uint64_t seed = powmod(red, xm, a_begin + w0 + lane, one);
    for (; w0 < count; w0 += nwarps * span) {
        uint64_t r = seed;
        const uint64_t lim = (count - w0 < span) ? count - w0 : span;
#pragma unroll 4
        for (uint64_t k = lane; k < lim; k += 32) {
            out[w0 + k] = (uint32_t)r;
            r = red.mulmod(r, x32);
        }
        seed = red.mulmod(seed, xjump);
    }
}

// Exact class counts.  For n small enough the histogram lives in shared
// memory (one 32-bit counter per class per CTA), flushed with 64-bit atomics;
// otherwise counts go straight to global 64-bit atomics.
constexpr int HIST_THREADS = 1024;

__global__ void __launch_bounds__(HIST_THREADS)
    class_counts_smem(const uint32_t *__restrict__ res, uint64_t count,
                      unsigned long long *__restrict__ counts, uint32_t ncls,
                      unsigned int *__restrict__ bad)
{
    uint32_t oob = 0;
    extern __shared__ uint32_t hist[];
    for (uint32_t v = threadIdx.x; v < ncls; v += blockDim.x) hist[v] = 0;
    __syncthreads();
    // a CTA covers 16 residues per thread per step: four coalesced 16-byte loads
    // in flight per thread before its 16 shared atomics (memory-level parallelism)
    const uint64_t per_cta = (uint64_t)blockDim.x * 16;
    const bool aligned = (reinterpret_cast<uintptr_t>(res) & 15) == 0;
    uint64_t base = (uint64_t)blockIdx.x * per_cta;
    for (; aligned && base + per_cta <= count; base += (uint64_t)gridDim.x * per_cta) {
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; j++)
            v[j] = __ldcs(reinterpret_cast<const uint4 *>(res + base + (uint64_t)j * blockDim.x * 4) + threadIdx.x);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t r4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int t = 0; t < 4; t++) {
                if (r4[t] < ncls) atomicAdd(&hist[r4[t]], 1u);
                else oob = 1;
            }
        }
    }
    // the ragged tail chunk (or every chunk of an unaligned buffer), one residue per thread per step
    for (; base < count; base += (uint64_t)gridDim.x * per_cta) {
        const uint64_t hi = base + per_cta < count ? base + per_cta : count;
        for (uint64_t i = base + threadIdx.x; i < hi; i += blockDim.x) {
            const uint32_t r = res[i];
            if (r < ncls) atomicAdd(&hist[r], 1u);
            else oob = 1;
        }
    }
    if (oob) atomicOr(bad, 1u);
    __syncthreads();
    for (uint32_t v = threadIdx.x; v < ncls; v += blockDim.x)
        if (hist[v]) atomicAdd(&counts[v], (unsigned long long)hist[v]);
}

__global__ void class_counts_global(const uint32_t *__restrict__ res, uint64_t count,
                                    unsigned long long *__restrict__ counts, uint64_t ncls,
                                    unsigned int *__restrict__ bad)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint32_t r = res[i];
        if (r < ncls) atomicAdd(&counts[r], 1ull);
        else atomicOr(bad, 1u);
    }
}

}  // namespace shb

using namespace shb;

extern "C" int shb_modexp(uint32_t *d_residues, uint64_t a_begin, uint64_t count, uint64_t x,
                          uint64_t n, void *stream)
{
    if (n < 2) return set_error(SHB_EINVAL, "modulus must be >= 2");
    if (n > 0xFFFFFFFFull) return set_error(SHB_EINVAL, "modulus %llu exceeds the 32-bit residue storage",
                                            (unsigned long long)n);
    if (count == 0) return SHB_OK;
    if (!d_residues) return set_error(SHB_EINVAL, "null residue buffer");
    cudaStream_t st = as_stream(stream);
    const uint64_t xm = x % n;
    const uint64_t one = 1 % n;
    const uint64_t span = 32ull * MODEXP_ITERS;
    const uint64_t warps_needed = (count + span - 1) / span;
    const uint64_t blocks_needed = (warps_needed + MODEXP_THREADS / 32 - 1) / (MODEXP_THREADS / 32);
    const uint64_t cap = (uint64_t)sm_count() * 8;
    const unsigned grid = (unsigned)(blocks_needed < cap ? blocks_needed : cap);
    // x^32 mod n on the host (exact with 128-bit products)
    unsigned __int128 b = xm, acc = one;
    for (int i = 0; i < 32; i++) acc = (acc * b) % n;
    const uint64_t x32 = (uint64_t)acc;
    // x^(grid_warps * span) mod n: the per-warp jump between grid-stride spans
    uint64_t jump_e = (uint64_t)grid * (MODEXP_THREADS / 32) * span;
    unsigned __int128 jb = xm, jacc = one;
    while (jump_e) {
        if (jump_e & 1) jacc = (jacc * jb) % n;
        jb = (jb * jb) % n;
        jump_e >>= 1;
    }
    const uint64_t xjump = (uint64_t)jacc;
    if (n < 65536) {
        Barrett32 red{(uint32_t)n, (uint32_t)(0xFFFFFFFFu / (uint32_t)n)};
        modexp_kernel<<<grid, MODEXP_THREADS, 0, st>>>(d_residues, a_begin, count, xm, x32, xjump, red, one);
        SHB_LAUNCHED();
    } else {
        Barrett64 red{n, ~0ull / n};
        modexp_kernel<<<grid, MODEXP_THREADS, 0, st>>>(d_residues, a_begin, count, xm, x32, xjump, red, one);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

extern "C" int shb_class_counts(const uint32_t *d_residues, uint64_t count, uint64_t *d_counts,
                                uint64_t ncls, void *stream)
{
    if (ncls == 0) return set_error(SHB_EINVAL, "ncls must be >= 1");
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    Scratch bad;
    SHB_TRY(scratch_alloc(bad, sizeof(unsigned int), st));
    SHB_TRY_CUDA(cudaMemsetAsync(bad.ptr, 0, sizeof(unsigned int), st));
    const size_t smem = ncls * sizeof(uint32_t);
    if (smem <= 200 * 1024) {
        SHB_TRY_CUDA(cudaFuncSetAttribute(class_counts_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          200 * 1024));
        const uint64_t per_block = (uint64_t)HIST_THREADS * 4 * 16;
        uint64_t blocks = (count + per_block - 1) / per_block;
        const uint64_t cap = (uint64_t)sm_count();
        if (blocks > cap) blocks = cap;
        class_counts_smem<<<(unsigned)blocks, HIST_THREADS, smem, st>>>(
            d_residues, count, (unsigned long long *)d_counts, (uint32_t)ncls, (unsigned int *)bad.ptr);
        SHB_LAUNCHED();
    } else {
        class_counts_global<<<sm_count() * 8, 256, 0, st>>>(
            d_residues, count, (unsigned long long *)d_counts, ncls, (unsigned int *)bad.ptr);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    unsigned int h = 0;
    SHB_TRY_CUDA(cudaMemcpyAsync(&h, bad.ptr, sizeof h, cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    if (h) return set_error(SHB_ERANGE, "a residue is >= ncls=%llu", (unsigned long long)ncls);
    return SHB_OK;
}
