// FP32 fast path of the QFT on the 5th-generation tensor cores (tcgen05 +
// TMEM): the uniform comb (the collapsed Shor register), precision SHB_FP32,
// tiles == 1.  Same sum and the same GEMM factorisation as the mma.sync
// kernels of dft.cu (qft.dense_dft, qft.py:95-112 / _kernels.py:16-30):
//
//   a_j = a0 + j*stride,  j = (sb*NB + jj)*BK + k   (super-block sb, row-block jj, k < BK)
//   V_c = scale*amp * sum_sb sum_jj e^{+2 pi i (a0 + (sb*NB + jj)*BK*stride) c / q} * T[c, jj]
//   T[c, jj] = sum_k G[c, k] * 1,   G[c, k] = e^{+2 pi i k stride c / q}
//
// One tcgen05.mma (M = 128 outputs, N = NB row-blocks, K = 16) multiplies the
// generated phase matrix G (A operand, shared memory, K-major) by ones (B
// operand, shared memory) into an FP32 accumulator in TMEM: each row-block's
// T for 128 outputs at once.  G is split into two bf16 terms, G = G_hi + G_lo
// (|G - G_hi - G_lo| <= 2^-18 |G|): 4 MMAs per k-step (Re/Im x hi/lo), the
// same 4 bf16 multiply-adds per phase term as dft_tc32_uniform_kernel.
//
// Roles (one persistent CTA per SM, 9 warps):
//  * warp 8, one elected thread: issues the MMAs of a super-block into one of
//    two TMEM accumulator buffers and commits them to that buffer's `full`
//    mbarrier;
//  * warps 0-7 (two workers per TMEM lane = output): build G for the tile, then per
//    super-block load the accumulators (tcgen05.ld 32x32b), release the
//    buffer (`empty` mbarrier) and fold the NB row-blocks by an FP32 Horner
//    with w^{-BK}, rotate by the exact-index seed of the last row-block
//    (sincospif of the exact integer phase index) and add into an FP64 total.
// The last super-block of a tile runs with N rounded up to a multiple of 32
// row-blocks and a ones mask that zeroes amplitudes past the progression.
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include "shb_internal.cuh"

namespace shb {

namespace tc05 {

constexpr int TILE = 128;            // outputs per tile (MMA M, TMEM lanes)
constexpr int NB = 128;              // row-blocks per super-block (MMA N: 128 reaches the full
                                     // 4096 MAC/clk/SM, 64 only ~2800, scripts/tc05_rate_probe.cu)
#ifndef SHB_TC05_BK
#define SHB_TC05_BK 128
#endif
constexpr int BK = SHB_TC05_BK;      // k per row-block (MMA K total)
#ifndef SHB_TC05_CHAINS
#define SHB_TC05_CHAINS 1
#endif
constexpr int HORNER_CHAINS = SHB_TC05_CHAINS;  // fold: 1 chain of 64, or 4 of 16
constexpr int KSTEPS = BK / 16;      // tcgen05.mma K = 16 for bf16
constexpr int SB_AMPS = NB * BK;     // amplitudes per super-block (8192)
constexpr int A_BYTES = TILE * BK * 2;   // one bf16 variant of G
constexpr int G_BYTES = 4 * A_BYTES;     // one tile's G (Re hi, Re lo, Im hi, Im lo)
constexpr int B_BYTES = NB * BK * 2;     // ones / mask
// two G buffers when they fit (BK = 64: the next tile's G is built while this
// tile's MMAs run); at BK = 128 one buffer, rebuilt between tiles
constexpr int G_BUFS = (2 * 4 * TILE * BK * 2 + 2 * NB * BK * 2 + 1024 <= 227 * 1024) ? 2 : 1;
constexpr int SMEM_BYTES = G_BUFS * G_BYTES + 2 * B_BYTES + 1024;  // + alignment slack
constexpr int TMEM_COLS = 512;       // 2 accumulator buffers x (Re NB | Im NB)
constexpr int WORKERS = 256;         // 8 warps: G builders + folders (2 per TMEM lane quarter)
constexpr int MMA_WARP = WORKERS / 32;
constexpr int THREADS = WORKERS + 32;  // + 1 MMA warp
constexpr uint32_t CORE_ROW_BYTES = 16;
constexpr uint32_t LBO = 128;                    // next 8-wide k group
constexpr uint32_t SBO = (BK / 8) * 128;         // next 8-row group

// byte offset of (row, k) in a K-major no-swizzle operand: 8 x 16 B core
// matrices, k groups adjacent (LBO), 8-row groups every SBO (validated by
// scripts/tc05_probe.cu against a host GEMM)
__device__ __forceinline__ uint32_t kmajor(int row, int k)
{
    return (uint32_t)(row >> 3) * SBO + (uint32_t)(k >> 3) * LBO + (uint32_t)(row & 7) * CORE_ROW_BYTES +
           (uint32_t)(k & 7) * 2;
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr)
{
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(LBO >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) |
           ((uint64_t)1 << 46);  // sm_100 descriptor version; no swizzle
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, both K-major
__device__ __forceinline__ uint32_t idesc(int n)
{
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(TILE >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_addr(bar))
                 : "memory");
}

// mbarrier wait that traps instead of hanging if the pipeline ever stalls
__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t phase)
{
    uint32_t ok = 0;
    for (uint64_t spin = 0; !ok; spin++) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
        if (spin > (1ull << 28)) asm volatile("trap;");
    }
}

__device__ __forceinline__ void ld32(uint32_t taddr, float *v)
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void phase_f32(uint64_t idx, uint64_t q, double two_over_q, float &c, float &s)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    sincospif((float)((double)sidx * two_over_q), &s, &c);
}

struct Args {
    uint64_t length, a0, stride, q;
    double two_over_q;
    uint64_t c_begin, c_count, ntiles;
    double out_re, out_im;
    double2 *out;
    double *prob;
    double *tile_sums;  // per tile sum of |V|^2 (nullable)
};

__global__ void __launch_bounds__(THREADS, 1) dft_tc05_uniform_kernel(const Args p)
{
    extern __shared__ unsigned char smem_raw[];
    // 1024-B aligned operand region: two tiles' G (A operand: Re hi, Re lo, Im hi,
    // Im lo), ones, last-block mask
    unsigned char *base = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;
    unsigned char *sOnes = base + G_BUFS * G_BYTES;
    unsigned char *sMask = sOnes + B_BYTES;
    __shared__ __align__(8) uint64_t full_bar[2], empty_bar[2], a_ready;
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t q = p.q, qmask = q - 1;
    const uint64_t nsb = (p.length + SB_AMPS - 1) / SB_AMPS;
    // the last super-block: valid row-blocks and the MMA N it runs with
    const uint64_t last_amps = p.length - (nsb - 1) * SB_AMPS;  // in (0, SB_AMPS]
    const int last_rb = (int)((last_amps + BK - 1) / BK);
    const int last_n = ((last_rb + 31) / 32) * 32;  // halves of whole 16-column TMEM loads

    // ones and the last-super-block mask (B operands: row = row-block jj, K-major)
    for (int i = tid; i < NB * BK; i += THREADS) {
        const int jj = i / BK, k = i % BK;
        const __nv_bfloat16 one = __float2bfloat16_rn(1.f), zero = __float2bfloat16_rn(0.f);
        *reinterpret_cast<__nv_bfloat16 *>(sOnes + kmajor(jj, k)) = one;
        *reinterpret_cast<__nv_bfloat16 *>(sMask + kmajor(jj, k)) =
            ((uint64_t)jj * BK + k < last_amps) ? one : zero;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr(&tmem_base_sh)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&full_bar[0], 1);
        mbar_init(&full_bar[1], 1);
        mbar_init(&empty_bar[0], WORKERS);
        mbar_init(&empty_bar[1], WORKERS);
        mbar_init(&a_ready, WORKERS);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_sh;

    if (warp == MMA_WARP) {
        // ---------------------------------------------------------- MMA issuer
        if (lane == 0) {
            const uint32_t aaddr = smem_addr(sA), onesaddr = smem_addr(sOnes), maskaddr = smem_addr(sMask);
            uint64_t g = 0;  // super-blocks issued so far (buffer g & 1)
            uint32_t it = 0;
            for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, it++) {
                wait_bar(&a_ready, it & 1u);  // G of this tile is in shared memory
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t ga = aaddr + (G_BUFS == 2 ? (it & 1u) * G_BYTES : 0u);
                for (uint64_t sb = 0; sb < nsb; sb++, g++) {
                    const uint32_t b = (uint32_t)(g & 1);
                    if (g >= 2) wait_bar(&empty_bar[b], (uint32_t)((g >> 1) - 1) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const bool last = sb + 1 == nsb;
                    const int n = last ? last_n : NB;
                    const uint32_t id = idesc(n);
                    const uint32_t bsrc = last ? maskaddr : onesaddr;
                    const uint32_t d_re = tmem + b * (2 * NB), d_im = d_re + NB;
#pragma unroll
                    for (int s = 0; s < KSTEPS; s++) {
                        const uint64_t db = smem_desc(bsrc + s * 2 * LBO);
                        const uint32_t koff = s * 2 * LBO;
                        mma(d_re, smem_desc(ga + 0 * A_BYTES + koff), db, id, s > 0);
                        mma(d_re, smem_desc(ga + 1 * A_BYTES + koff), db, id, 1);
                        mma(d_im, smem_desc(ga + 2 * A_BYTES + koff), db, id, s > 0);
                        mma(d_im, smem_desc(ga + 3 * A_BYTES + koff), db, id, 1);
                    }
                    commit(&full_bar[b]);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------- G builders + folders (row = TMEM lane = output)
        // worker w: row = w % 128 (warp w/32 reads TMEM lane quarter (w/32) % 4),
        // half = w / 128 builds G columns [64 half, 64 half + 64) and folds
        // row-blocks [n/2 half, n/2 (half + 1)) of every super-block
        const int row = tid & (TILE - 1), half = tid >> 7;
        const uint32_t lane_addr = (uint32_t)(32 * (warp & 3)) << 16;
        __shared__ double vpart[2][TILE];
        __shared__ double wsum[8];
        uint64_t g = 0;
        uint32_t it = 0;
        // G[c, k] = e^{+2 pi i k stride c / q} for this worker's row and k half
        // into G buffer `buf` (A operand in shared memory): exact sincospif every
        // 8 k, FP32 rotation in between, split into bf16 hi + lo
        auto build_g = [&](uint64_t tt, uint32_t buf) {
            const uint64_t cg = p.c_begin + tt * TILE + row;
            unsigned char *gA = sA + buf * G_BYTES;
            {
                float wr, wi;
                phase_f32((p.stride * cg) & qmask, q, p.two_over_q, wr, wi);
#pragma unroll 2
                for (int k0 = half * (BK / 2); k0 < (half + 1) * (BK / 2); k0 += 8) {
                    float gr, gi;
                    phase_f32(((uint64_t)k0 * p.stride * cg) & qmask, q, p.two_over_q, gr, gi);
                    uint32_t pk[4][4];
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        float v[2][2];  // [elem][re, im]
#pragma unroll
                        for (int u = 0; u < 2; u++) {
                            v[u][0] = gr;
                            v[u][1] = gi;
                            const float nr = fmaf(gr, wr, -gi * wi), ni = fmaf(gr, wi, gi * wr);
                            gr = nr;
                            gi = ni;
                        }
                        const __nv_bfloat162 rh = __floats2bfloat162_rn(v[0][0], v[1][0]);
                        const __nv_bfloat162 ih = __floats2bfloat162_rn(v[0][1], v[1][1]);
                        const __nv_bfloat162 rl = __floats2bfloat162_rn(v[0][0] - __low2float(rh),
                                                                         v[1][0] - __high2float(rh));
                        const __nv_bfloat162 il = __floats2bfloat162_rn(v[0][1] - __low2float(ih),
                                                                         v[1][1] - __high2float(ih));
                        pk[0][e / 2] = *reinterpret_cast<const uint32_t *>(&rh);
                        pk[1][e / 2] = *reinterpret_cast<const uint32_t *>(&rl);
                        pk[2][e / 2] = *reinterpret_cast<const uint32_t *>(&ih);
                        pk[3][e / 2] = *reinterpret_cast<const uint32_t *>(&il);
                    }
                    const uint32_t off = kmajor(row, k0);
#pragma unroll
                    for (int v4 = 0; v4 < 4; v4++)
                        *reinterpret_cast<uint4 *>(gA + v4 * A_BYTES + off) =
                            make_uint4(pk[v4][0], pk[v4][1], pk[v4][2], pk[v4][3]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&a_ready);
        };
        if (G_BUFS == 2 && (uint64_t)blockIdx.x < p.ntiles) build_g(blockIdx.x, 0);
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, it++) {
            const uint64_t c = p.c_begin + t * TILE + row;
            // one buffer: the MMAs reading the previous tile's G are complete
            // (this worker waited on the commit of that tile's last super-block)
            if (G_BUFS == 1) build_g(t, 0);

            // fold this worker's half of every super-block: h = h * W + T[jj] (FP32), W = w^{-BK}
            float Wr, Wi, W16r, W16i;
            {
                float co, si;
                phase_f32(((uint64_t)BK * p.stride * c) & qmask, q, p.two_over_q, co, si);
                Wr = co;
                Wi = -si;
                phase_f32(((uint64_t)16 * BK * p.stride * c) & qmask, q, p.two_over_q, co, si);
                W16r = co;
                W16i = -si;
            }
            double vr = 0.0, vi = 0.0;
            for (uint64_t sb = 0; sb < nsb; sb++, g++) {
                const uint32_t b = (uint32_t)(g & 1);
                wait_bar(&full_bar[b], (uint32_t)(g >> 1) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int n = (sb + 1 == nsb) ? last_n : NB;
                const int j_lo = half * (n / 2), j_hi = j_lo + n / 2;
                const uint32_t d_re = tmem + lane_addr + b * (2 * NB), d_im = d_re + NB;
                // all of this worker's accumulators in one burst of TMEM loads, then
                // the buffer goes straight back to the MMA warp; the Horner runs
                // from registers (columns past j_hi are loaded and ignored)
                float tr[NB / 2], ti[NB / 2];
                ld32(d_re + j_lo, tr);
                ld32(d_re + j_lo + 32, tr + 32);
                ld32(d_im + j_lo, ti);
                ld32(d_im + j_lo + 32, ti + 32);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&empty_bar[b]);
                float hr = 0.f, hi = 0.f;
                if (HORNER_CHAINS == 1) {
                    const int cnt = j_hi - j_lo;
#pragma unroll
                    for (int e = 0; e < NB / 2; e++) {
                        if (e < cnt) {
                            const float nr = fmaf(hr, Wr, fmaf(-hi, Wi, tr[e]));
                            const float ni = fmaf(hr, Wi, fmaf(hi, Wr, ti[e]));
                            hr = nr;
                            hi = ni;
                        }
                    }
                } else {
                    // 4 independent chains of 16 row-blocks (ILP), joined with W^16:
                    // h = ((h0 W^16 + h1) W^16 + h2) W^16 + h3
                    const int nch = (j_hi - j_lo) / 16;  // halves are whole multiples of 16
                    float cr[4] = {0.f, 0.f, 0.f, 0.f}, ci[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int e = 0; e < 16; e++)
#pragma unroll
                        for (int ch = 0; ch < 4; ch++) {
                            const float nr = fmaf(cr[ch], Wr, fmaf(-ci[ch], Wi, tr[ch * 16 + e]));
                            const float ni = fmaf(cr[ch], Wi, fmaf(ci[ch], Wr, ti[ch * 16 + e]));
                            cr[ch] = nr;
                            ci[ch] = ni;
                        }
                    hr = cr[0];
                    hi = ci[0];
#pragma unroll
                    for (int ch = 1; ch < 4; ch++) {
                        if (ch < nch) {
                            const float nr = fmaf(hr, W16r, fmaf(-hi, W16i, cr[ch]));
                            const float ni = fmaf(hr, W16i, fmaf(hi, W16r, ci[ch]));
                            hr = nr;
                            hi = ni;
                        }
                    }
                }
                // seed of the last folded row-block: a0 + (sb*NB + j_hi-1)*BK*stride
                const uint64_t a_last = p.a0 + ((sb * NB + (uint64_t)(j_hi - 1)) * BK) * p.stride;
                float sc, ss;
                phase_f32((a_last * c) & qmask, q, p.two_over_q, sc, ss);
                vr = fma((double)sc, (double)hr, fma(-(double)ss, (double)hi, vr));
                vi = fma((double)sc, (double)hi, fma((double)ss, (double)hr, vi));
                // the next tile's G, into the other buffer, while this tile's MMAs
                // run (that buffer's last readers, the previous tile's MMAs, are
                // complete: this worker waited on their commit)
                if (G_BUFS == 2 && sb == 0 && t + gridDim.x < p.ntiles) build_g(t + gridDim.x, (it + 1) & 1u);
            }
            // combine the two halves (fixed order: half 0 + half 1), then the
            // epilogue: output factor, |V|^2 (hypot^2, as np.abs(.)**2), tile sum
            if (half == 1) {
                vpart[0][row] = vr;
                vpart[1][row] = vi;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(WORKERS) : "memory");
            double pr = 0.0;
            if (half == 0) {
                vr += vpart[0][row];
                vi += vpart[1][row];
                const uint64_t ci = t * TILE + row;
                if (ci < p.c_count) {
                    const double o_re = vr * p.out_re - vi * p.out_im;
                    const double o_im = vr * p.out_im + vi * p.out_re;
                    p.out[ci] = make_double2(o_re, o_im);
                    const double hh = hypot(o_re, o_im);
                    pr = hh * hh;
                    if (p.prob) p.prob[ci] = pr;
                }
            }
            if (p.tile_sums) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) pr += __shfl_down_sync(0xffffffffu, pr, o);
                if (lane == 0) wsum[warp] = pr;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(WORKERS) : "memory");
            if (p.tile_sums && tid == 0) p.tile_sums[t] = (wsum[0] + wsum[1]) + (wsum[2] + wsum[3]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

__global__ void tile_group_sums_kernel(const double *__restrict__ part, uint64_t nparts, int group,
                                       double *__restrict__ out, uint64_t nout)
{
    const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nout) return;
    double s = 0.0;
    for (int i = 0; i < group; i++) {
        const uint64_t j = g * group + i;
        if (j < nparts) s += part[j];
    }
    out[g] = s;
}

}  // namespace tc05

// Caller contract as shb_dft_uniform (validated there); block sums in the
// caller's shb_dft_num_blocks(c_count, SHB_FP32) layout (slot_outputs per slot).
int tc05_dft_uniform(uint64_t length, uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin,
                     uint64_t c_count, double out_re, double out_im, double *d_out, double *d_prob,
                     double *d_block_sums, uint64_t slot_outputs, cudaStream_t st)
{
    using namespace tc05;
    if (length == 0 || c_count == 0) return set_error(SHB_EINVAL, "tc05 path needs a non-empty support and output");
    Args a{};
    a.length = length;
    a.a0 = a0;
    a.stride = stride;
    a.q = q;
    a.two_over_q = 2.0 / (double)q;
    a.c_begin = c_begin;
    a.c_count = c_count;
    a.ntiles = (c_count + TILE - 1) / TILE;
    a.out_re = out_re;
    a.out_im = out_im;
    a.out = (double2 *)d_out;
    a.prob = d_prob;
    Scratch part;
    if (d_block_sums) {
        SHB_TRY(scratch_alloc(part, sizeof(double) * a.ntiles, st));
        a.tile_sums = (double *)part.ptr;
    }
    SHB_TRY_CUDA(cudaFuncSetAttribute(dft_tc05_uniform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    const uint64_t grid = a.ntiles < (uint64_t)sm_count() ? a.ntiles : (uint64_t)sm_count();
    dft_tc05_uniform_kernel<<<(unsigned)grid, THREADS, SMEM_BYTES, st>>>(a);
    SHB_LAUNCHED();
    if (d_block_sums) {
        const int group = (int)(slot_outputs / TILE);
        const uint64_t nout = (c_count + slot_outputs - 1) / slot_outputs;
        tile_group_sums_kernel<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>((const double *)part.ptr,
                                                                               a.ntiles, group, d_block_sums,
                                                                               nout);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

}  // namespace shb
