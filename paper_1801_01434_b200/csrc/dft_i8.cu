// FP64-accurate QFT of the uniform comb (the collapsed Shor register) on the
// 5th-generation INTEGER tensor cores (tcgen05.mma kind::i8, TMEM int32
// accumulators): precision SHB_FP64, tiles == 1.  Same sum and the same GEMM
// factorisation as dft_tc05.cu / the DMMA engine of dft.cu (qft.dense_dft,
// qft.py:95-112 / _kernels.py:16-30):
//
//   a_j = a0 + j*stride,  j = (sb*NB + jj)*BK + k   (super-block sb, row-block jj, k < BK)
//   V_c = scale*amp * sum_sb sum_jj e^{+2 pi i (a0 + (sb*NB + jj)*BK*stride) c / q} * T[c, jj]
//   T[c, jj] = sum_k G[c, k] * 1,   G[c, k] = e^{+2 pi i k stride c / q}
//
// Exact fixed-point split of the phase matrix (the integer-slice scheme of
// FP64-by-integer-GEMM emulation): each FP64 G value is rounded once to
// X = rint(G * 2^55) (|error| <= 2^-56, below half an FP64 ulp of 1) and
// written as 8 base-128 digits
//
//   X = d0*2^49 + u1*2^42 + u2*2^35 + ... + u7,   d0 in [-64, 64] (s8), u_s in [0, 127] (u8)
//
// Every int8 x int8 product and every int32 accumulation in the tensor core
// is EXACT, so T is exact up to the one rounding of G.  Digits are paired in
// one accumulator by the B operand: digit 2p against 128*mask (u8), digit
// 2p+1 against 1*mask, so accumulator p holds D_p = sum_k (128 d_2p + d_2p+1)
// (|D_p| < 2^21 for BK <= 96) and
//
//   2^55 T = D_0 2^42 + D_1 2^28 + D_2 2^14 + D_3     (one FP64 rounding)
//
// 2 components (Re, Im) x 4 accumulators x NB row-blocks of int32 = 512 TMEM
// columns at NB = 64.  The fold over row-blocks (Horner with w^{-BK}), the
// exact sincospi seeds and the totals are FP64, as in the DMMA engine.
//
// Roles (one persistent CTA per SM, 9 warps):
//  * warp 8, one elected thread: per super-block 2 x 4 x (BK/32) x 2 MMAs
//    (M = 128 outputs, N = NB row-blocks, K = 32), committed to `full`;
//  * warps 0-7 (two workers per TMEM lane = output): build the 16 digit
//    matrices of G for the tile (FP64 phases, exact sincospi every 16 k),
//    then per super-block load the accumulators (tcgen05.ld 32x32b.x8),
//    combine the 4 digit pairs to FP64, fold, seed, add to the FP64 total.
#include <math.h>
#include <stdlib.h>

#include "shb_internal.cuh"

namespace shb {

namespace i8 {

constexpr int TILE = 128;  // outputs per tile (MMA M, TMEM lanes)
#ifndef SHB_I8_NB
#define SHB_I8_NB 64
#endif
#ifndef SHB_I8_BK
#define SHB_I8_BK 96
#endif
#ifndef SHB_I8_ICOMB
#define SHB_I8_ICOMB 1  // combine digit pairs as int64 before the FP64 conversion
#endif
constexpr int NB = SHB_I8_NB;         // row-blocks per super-block (MMA N)
constexpr int BK = SHB_I8_BK;         // k per row-block (MMA K total)
static_assert(BK % 32 == 0 && BK <= 96, "BK: whole K = 32 steps, |D_p| < 2^21");
static_assert(NB % 16 == 0 && NB >= 16 && NB <= 64, "NB");
constexpr int NPAIR = 4;              // accumulators per component
constexpr int NDIG = 8;               // base-128 digits of G * 2^55
constexpr int KCH = BK / 32;          // MMA K = 32 for 8-bit operands
constexpr int SB_AMPS = NB * BK;      // amplitudes per super-block
constexpr int ACC_COLS = 2 * NPAIR * NB;    // TMEM columns of one accumulator buffer
constexpr int NBUF = 512 / ACC_COLS;        // 1 at NB = 64, 2 at NB = 32
constexpr int TMEM_COLS = 512;
constexpr int A_BYTES = TILE * BK;          // one digit matrix of one component
constexpr int G_BYTES = 2 * NDIG * A_BYTES; // [comp][digit]
constexpr int B_BYTES = NB * BK;            // one weight matrix
constexpr int SMEM_BYTES = G_BYTES + 4 * B_BYTES + 1024;  // G, (128|1) x (ones|mask), alignment slack
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
constexpr int WORKERS = 256;
constexpr int MMA_WARP = WORKERS / 32;
constexpr int THREADS = WORKERS + 32;
constexpr int CH = 8;                 // row-blocks per TMEM load burst
constexpr uint32_t LBO = 128;                 // next 16-byte k group
constexpr uint32_t SBO = (BK / 16) * 128;     // next 8-row group

// byte offset of (row, k) in a K-major no-swizzle 8-bit operand: 8 x 16 B
// core matrices (16 k each), k groups adjacent (LBO), 8-row groups every SBO
__device__ __forceinline__ uint32_t kmajor(int row, int k)
{
    return (uint32_t)(row >> 3) * SBO + (uint32_t)(k >> 4) * LBO + (uint32_t)(row & 7) * 16u + (uint32_t)(k & 15);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr)
{
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(LBO >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) |
           ((uint64_t)1 << 46);  // sm_100 descriptor version; no swizzle
}

// kind::i8 instruction descriptor: A s8 (a_signed) or u8, B u8 -> S32, both K-major
__device__ __forceinline__ uint32_t idesc(int n, bool a_signed)
{
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(TILE >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
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

__device__ __forceinline__ void ld8(uint32_t taddr, int *v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
}

__device__ __forceinline__ void phase64(uint64_t idx, uint64_t q, double two_over_q, double &c, double &s)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    sincospi((double)sidx * two_over_q, &s, &c);
}

// 2^55 T from the 4 pair accumulators: exact up to the last add
__device__ __forceinline__ double combine(int d0, int d1, int d2, int d3)
{
#if SHB_I8_ICOMB
    const long long hi = (long long)d0 * 16384 + d1;  // < 2^35, exact
    const long long lo = (long long)d2 * 16384 + d3;
    return fma((double)hi, 0x1p28, (double)lo);
#else
    const double t = fma(fma((double)d0, 0x1p14, (double)d1), 0x1p14, (double)d2);  // exact (< 2^50)
    return fma(t, 0x1p14, (double)d3);
#endif
}

struct Args {
    uint64_t length, a0, stride, q;
    double two_over_q;
    uint64_t c_begin, c_count, ntiles;
    double out_re, out_im;  // output factor (scale * amp), times 2^-55 here
    double2 *out;
    double *prob;
    double *tile_sums;  // per tile sum of |V|^2 (nullable)
};

__global__ void __launch_bounds__(THREADS, 1) dft_i8_uniform_kernel(const Args p)
{
    extern __shared__ unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;                  // [comp][digit] A operands
    unsigned char *sB = base + G_BYTES;        // [ones128, ones1, mask128, mask1]
    __shared__ __align__(8) uint64_t full_bar[NBUF], empty_bar[NBUF], a_ready;
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t q = p.q, qmask = q - 1;
    const uint64_t nsb = (p.length + SB_AMPS - 1) / SB_AMPS;
    const uint64_t last_amps = p.length - (nsb - 1) * SB_AMPS;  // in (0, SB_AMPS]
    const int last_rb = (int)((last_amps + BK - 1) / BK);
    const int last_n = ((last_rb + 15) / 16) * 16;  // MMA N multiple of 16; halves of whole 8-column loads

    // weights (B operands: row = row-block jj, K-major, u8): 128 / 1 times ones / last mask
    for (int i = tid; i < NB * BK; i += THREADS) {
        const int jj = i / BK, k = i % BK;
        const uint32_t off = kmajor(jj, k);
        const bool live = (uint64_t)jj * BK + k < last_amps;
        sB[0 * B_BYTES + off] = 128;
        sB[1 * B_BYTES + off] = 1;
        sB[2 * B_BYTES + off] = live ? 128 : 0;
        sB[3 * B_BYTES + off] = live ? 1 : 0;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr(&tmem_base_sh)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int b = 0; b < NBUF; b++) {
            mbar_init(&full_bar[b], 1);
            mbar_init(&empty_bar[b], WORKERS);
        }
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
            const uint32_t aaddr = smem_addr(sA), baddr = smem_addr(sB);
            uint64_t g = 0;  // super-blocks issued so far (buffer g % NBUF)
            uint32_t it = 0;
            for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, it++) {
                wait_bar(&a_ready, it & 1u);  // G of this tile is in shared memory
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (uint64_t sb = 0; sb < nsb; sb++, g++) {
                    const uint32_t b = (uint32_t)(g % NBUF);
                    const uint64_t use = g / NBUF;
                    if (use >= 1) wait_bar(&empty_bar[b], (uint32_t)(use - 1) & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const bool last = sb + 1 == nsb;
                    const int n = last ? last_n : NB;
                    const uint32_t id_s = idesc(n, true), id_u = idesc(n, false);
                    const uint32_t w128 = baddr + (last ? 2 : 0) * B_BYTES, w1 = w128 + B_BYTES;
#pragma unroll
                    for (int comp = 0; comp < 2; comp++)
#pragma unroll
                        for (int pr = 0; pr < NPAIR; pr++) {
                            const uint32_t d = tmem + b * ACC_COLS + (comp * NPAIR + pr) * NB;
                            const uint32_t ahi = aaddr + (comp * NDIG + 2 * pr) * A_BYTES, alo = ahi + A_BYTES;
#pragma unroll
                            for (int s = 0; s < KCH; s++) {
                                const uint32_t koff = s * 2 * LBO;
                                mma(d, smem_desc(ahi + koff), smem_desc(w128 + koff), pr == 0 ? id_s : id_u, s > 0);
                                mma(d, smem_desc(alo + koff), smem_desc(w1 + koff), id_u, 1);
                            }
                        }
                    commit(&full_bar[b]);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------- G builders + folders (row = TMEM lane = output)
        // worker w: row = w % 128 (warp w/32 reads TMEM lane quarter (w/32) % 4),
        // half = w / 128 builds G columns [BK/2 half, BK/2 (half+1)) and folds
        // row-blocks [n/2 half, n/2 (half+1)) of every super-block
        const int row = tid & (TILE - 1), half = tid >> 7;
        const uint32_t lane_addr = (uint32_t)(32 * (warp & 3)) << 16;
        __shared__ double vpart[2][TILE];
        __shared__ double wsum[8];
        uint64_t g = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
            const uint64_t c = p.c_begin + t * TILE + row;
            // G[c, k] = e^{+2 pi i k stride c / q}: exact sincospi every 16 k, FP64
            // rotation in between (<= ~15 ulp, as the DMMA engine's G), rounded to
            // X = rint(G 2^55) and split into 8 digits per component.  The MMAs
            // reading the previous tile's G are complete: this worker waited on
            // the commit of that tile's last super-block.
            {
                double wr, wi;
                phase64((p.stride * c) & qmask, q, p.two_over_q, wr, wi);
                for (int k0 = half * (BK / 2); k0 < (half + 1) * (BK / 2); k0 += 16) {
                    double gr, gi;
                    phase64(((uint64_t)k0 * p.stride * c) & qmask, q, p.two_over_q, gr, gi);
                    uint32_t pk[2][NDIG][4];
#pragma unroll
                    for (int e = 0; e < 16; e++) {
#pragma unroll
                        for (int comp = 0; comp < 2; comp++) {
                            const long long X = __double2ll_rn((comp ? gi : gr) * 0x1p55);
                            const int d0 = (int)(X >> 49);
                            const unsigned long long R = (unsigned long long)(X - ((long long)d0 << 49));
                            const uint32_t hi28 = (uint32_t)(R >> 21), lo21 = (uint32_t)R & 0x1FFFFFu;
                            const uint32_t dig[NDIG] = {(uint32_t)d0 & 0xFFu, hi28 >> 21, (hi28 >> 14) & 127u,
                                                        (hi28 >> 7) & 127u, hi28 & 127u, lo21 >> 14,
                                                        (lo21 >> 7) & 127u, lo21 & 127u};
#pragma unroll
                            for (int dd = 0; dd < NDIG; dd++) {
                                if ((e & 3) == 0)
                                    pk[comp][dd][e >> 2] = dig[dd];
                                else
                                    pk[comp][dd][e >> 2] |= dig[dd] << (8 * (e & 3));
                            }
                        }
                        const double nr = fma(gr, wr, -gi * wi), ni = fma(gr, wi, gi * wr);
                        gr = nr;
                        gi = ni;
                    }
                    const uint32_t off = kmajor(row, k0);
#pragma unroll
                    for (int comp = 0; comp < 2; comp++)
#pragma unroll
                        for (int dd = 0; dd < NDIG; dd++)
                            *reinterpret_cast<uint4 *>(sA + (comp * NDIG + dd) * A_BYTES + off) =
                                make_uint4(pk[comp][dd][0], pk[comp][dd][1], pk[comp][dd][2], pk[comp][dd][3]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&a_ready);

            // fold this worker's half of every super-block: h = h * W + 2^55 T[jj] (FP64), W = w^{-BK}
            double Wr, Wi;
            {
                double co, si;
                phase64(((uint64_t)BK * p.stride * c) & qmask, q, p.two_over_q, co, si);
                Wr = co;
                Wi = -si;
            }
            double vr = 0.0, vi = 0.0;
            for (uint64_t sb = 0; sb < nsb; sb++, g++) {
                const uint32_t b = (uint32_t)(g % NBUF);
                wait_bar(&full_bar[b], (uint32_t)(g / NBUF) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const int n = (sb + 1 == nsb) ? last_n : NB;
                const int j_lo = half * (n / 2), j_hi = j_lo + n / 2;
                const uint32_t dbase = tmem + lane_addr + b * ACC_COLS;
                double hr = 0.0, hi = 0.0;
                for (int j0 = j_lo; j0 < j_hi; j0 += CH) {
                    int acc[2][NPAIR][CH];
#pragma unroll
                    for (int comp = 0; comp < 2; comp++)
#pragma unroll
                        for (int pr = 0; pr < NPAIR; pr++)
                            ld8(dbase + (comp * NPAIR + pr) * NB + j0, acc[comp][pr]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int e = 0; e < CH; e++) {
                        const double tr = combine(acc[0][0][e], acc[0][1][e], acc[0][2][e], acc[0][3][e]);
                        const double ti = combine(acc[1][0][e], acc[1][1][e], acc[1][2][e], acc[1][3][e]);
                        const double nr = fma(hr, Wr, fma(-hi, Wi, tr));
                        const double ni = fma(hr, Wi, fma(hi, Wr, ti));
                        hr = nr;
                        hi = ni;
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&empty_bar[b]);
                // seed of the last folded row-block: a0 + (sb*NB + j_hi-1)*BK*stride
                const uint64_t a_last = p.a0 + ((sb * NB + (uint64_t)(j_hi - 1)) * BK) * p.stride;
                double sc, ss;
                phase64((a_last * c) & qmask, q, p.two_over_q, sc, ss);
                vr = fma(sc, hr, fma(-ss, hi, vr));
                vi = fma(sc, hi, fma(ss, hr, vi));
            }
            // combine the two halves (fixed order: half 0 + half 1), then the
            // epilogue: output factor (with 2^-55), |V|^2 (hypot^2, as
            // np.abs(.)**2), tile sum
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

}  // namespace i8

// Caller contract as shb_dft_uniform (validated there); block sums in the
// caller's shb_dft_num_blocks(c_count, SHB_FP64) layout (slot_outputs per slot).
int i8_dft_uniform(uint64_t length, uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin, uint64_t c_count,
                   double out_re, double out_im, double *d_out, double *d_prob, double *d_block_sums,
                   uint64_t slot_outputs, cudaStream_t st)
{
    using namespace i8;
    if (length == 0 || c_count == 0) return set_error(SHB_EINVAL, "i8 path needs a non-empty support and output");
    Args a{};
    a.length = length;
    a.a0 = a0;
    a.stride = stride;
    a.q = q;
    a.two_over_q = 2.0 / (double)q;
    a.c_begin = c_begin;
    a.c_count = c_count;
    a.ntiles = (c_count + TILE - 1) / TILE;
    a.out_re = out_re * 0x1p-55;
    a.out_im = out_im * 0x1p-55;
    a.out = (double2 *)d_out;
    a.prob = d_prob;
    Scratch part;
    if (d_block_sums) {
        SHB_TRY(scratch_alloc(part, sizeof(double) * a.ntiles, st));
        a.tile_sums = (double *)part.ptr;
    }
    SHB_TRY_CUDA(cudaFuncSetAttribute(dft_i8_uniform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    const uint64_t grid = a.ntiles < (uint64_t)sm_count() ? a.ntiles : (uint64_t)sm_count();
    dft_i8_uniform_kernel<<<(unsigned)grid, THREADS, SMEM_BYTES, st>>>(a);
    SHB_LAUNCHED();
    if (d_block_sums) {
        const int group = (int)(slot_outputs / TILE);
        const uint64_t nout = (c_count + slot_outputs - 1) / slot_outputs;
        tile_group_sums_kernel<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>((const double *)part.ptr, a.ntiles,
                                                                               group, d_block_sums, nout);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

}  // namespace shb
