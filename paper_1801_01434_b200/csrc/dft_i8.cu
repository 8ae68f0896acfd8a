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
// Roles (one persistent CTA per SM, 4 SPLIT + 1 warps):
//  * the last warp, one elected thread: per super-block and component
//    4 x (BK/32) x 2 MMAs (M = 128 outputs, N = NB row-blocks, K = 32) into
//    that component's half of TMEM, committed to the component's `full`;
//  * the other warps (SPLIT workers per TMEM lane = output): build the 16
//    digit matrices of G for the tile (FP64 phases, exact sincospi every 16
//    k), then per super-block: load the Re accumulators of their row-blocks
//    (tcgen05.ld 32x32b.x8), combine the digit pairs to FP64, release the Re
//    half (the MMAs of the next super-block's Re start under the rest), then
//    the same for Im with the Horner fold, the exact seed and the FP64 total.
#include <math.h>
#include <stdlib.h>

#include "shb_internal.cuh"

#ifndef SHB_I8_DIGITS
#define SHB_I8_DIGITS 8
#endif
// build.py compiles this file twice: the FP64-grade 8-digit engine (namespace i8,
// i8_dft_uniform) and the 6-digit one (namespace i8d6, i8d6_dft_uniform)
#if SHB_I8_DIGITS == 6
#define SHB_I8_NS i8d6
#define SHB_I8_ENTRY i8d6_dft_uniform
#else
#define SHB_I8_NS i8
#define SHB_I8_ENTRY i8_dft_uniform
#endif

namespace shb {

namespace SHB_I8_NS {

constexpr int TILE = 128;  // outputs per tile (MMA M, TMEM lanes)
// SHB_I8_DIGITS: base-128 digits of G (8: X = rint(G 2^55), FP64-grade; 6: rint(G 2^41))
#ifndef SHB_I8_NB
#define SHB_I8_NB 64
#endif
#ifndef SHB_I8_BK
#define SHB_I8_BK (SHB_I8_DIGITS == 8 ? 96 : 128)
#endif
#ifndef SHB_I8_CONV
#define SHB_I8_CONV 8  // accumulators -> FP64 (measured, DESIGN 3.1.0): 8 = 5 with D_3 truncated (one ALU
                       // op less); 5 = one IMAD.WIDE bit pattern + DADD + one I2F + one DFMA per
                       // component; 0-4, 6, 7 = earlier / slower forms
#endif
#ifndef SHB_I8_CHAINS
#define SHB_I8_CHAINS 1  // interleaved Horner chains in the fold
#endif
#ifndef SHB_I8_SEED_EVERY
#define SHB_I8_SEED_EVERY 16  // exact sincospi seed every this many super-blocks (rotation between)
#endif
#ifndef SHB_I8_PHASES
#define SHB_I8_PHASES 1  // 1: one hand-over per super-block; 2: Re and Im halves handed over separately
#endif
#ifndef SHB_I8_SPLIT
#define SHB_I8_SPLIT 2  // workers per output (TMEM lane)
#endif
constexpr int NB = SHB_I8_NB;         // row-blocks per super-block (MMA N)
constexpr int BK = SHB_I8_BK;         // k per row-block (MMA K total)
constexpr int NDIG = SHB_I8_DIGITS;   // base-128 digits of G * 2^(7 NDIG - 1)
constexpr int NPAIR = NDIG / 2;       // accumulators per component
static_assert(NDIG == 8 || NDIG == 6, "digits");
static_assert(BK % 32 == 0 && BK <= 128, "BK: whole K = 32 steps, |D_p| < 2^21");
static_assert(NB % 16 == 0 && NB >= 16 && 2 * NPAIR * NB <= 512, "NB: 2 x NPAIR x NB int32 columns <= 512");
constexpr int KCH = BK / 32;          // MMA K = 32 for 8-bit operands
constexpr int SB_AMPS = NB * BK;      // amplitudes per super-block
constexpr int COMP_COLS = NPAIR * NB;       // TMEM columns of one component's accumulators
constexpr int TMEM_COLS = 512;
constexpr int A_BYTES = TILE * BK;          // one digit matrix of one component
constexpr int G_BYTES = 2 * NDIG * A_BYTES; // [comp][digit]
constexpr int B_BYTES = NB * BK;            // one weight matrix
// the all-128 / all-1 weights of full super-blocks: whole matrices, or (6 digits, to
// fit 12 digit matrices of BK = 128) 1 KB read through the zero-stride descriptor
constexpr int ONES_BYTES = NDIG == 8 ? B_BYTES : 1024;
constexpr int SMEM_BYTES = G_BYTES + 2 * ONES_BYTES + 2 * B_BYTES + 1024;  // G, ones x (128|1), mask x (128|1), slack
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
constexpr int SPLIT = SHB_I8_SPLIT;
constexpr int WORKERS = TILE * SPLIT;
constexpr int MMA_WARP = WORKERS / 32;
constexpr int THREADS = WORKERS + 32;
#ifndef SHB_I8_CH
#define SHB_I8_CH 8
#endif
// row-blocks per TMEM load burst (two bursts in flight).  9 warps put 3 on
// one SMSP, whose 64 KB register file caps every thread at 168 registers.
constexpr int CH = SHB_I8_CH;
constexpr int RBW = NB / SPLIT;       // row-blocks per worker in a full super-block
static_assert(RBW % CH == 0, "whole load bursts per worker");
constexpr int NCH = RBW / CH;
constexpr int CHAINS = SHB_I8_CHAINS;
constexpr double T_SCALE = NDIG == 6 ? 0x1p-41 : ((SHB_I8_CONV >= 4 && SHB_I8_CONV <= 6) || SHB_I8_CONV == 8) ? 0x1p-47 : 0x1p-55;  // units of combine()
static_assert(NDIG == 8 || SHB_I8_PHASES == 1, "6 digits: one hand-over per super-block only");
constexpr int PHASES = SHB_I8_PHASES;
#ifndef SHB_I8_PREFETCH
#define SHB_I8_PREFETCH 0  // PHASES == 1: next burst in flight while this one is folded
#endif
constexpr bool PREFETCH = SHB_I8_PREFETCH;
#ifndef SHB_I8_BDEDUP
#define SHB_I8_BDEDUP 0
#endif
constexpr bool BDEDUP = SHB_I8_BDEDUP;
#ifndef SHB_I8_GSPLIT
#define SHB_I8_GSPLIT 0  // 1: build G's Re digits, release them to the MMAs, then Im
#endif
constexpr bool GSPLIT = SHB_I8_GSPLIT;
#ifndef SHB_I8_GPACK
#define SHB_I8_GPACK 0  // 1: 8-digit G bytes by in-word spreading + PRMT transposes
#endif
constexpr bool GPACK = SHB_I8_GPACK;
#ifndef SHB_I8_MMA_ORDER
#define SHB_I8_MMA_ORDER 0
#endif
constexpr int MMA_ORDER = SHB_I8_MMA_ORDER;
static_assert(CH % CHAINS == 0, "chains interleave within a burst");
constexpr uint64_t SEED_EVERY = SHB_I8_SEED_EVERY;
constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
constexpr int LAST_ALIGN = CH * SPLIT / gcd_c(CH * SPLIT, 16) * 16;  // last super-block N granule: lcm(CH SPLIT, 16)
static_assert(NB % LAST_ALIGN == 0, "the last super-block's N rounds up to at most NB");
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

__device__ __forceinline__ bool elect_one()
{
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
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

__device__ __forceinline__ void ld4(uint32_t taddr, int *v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}

__device__ __forceinline__ void ld16(uint32_t taddr, int *v)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

template <int N>
__device__ __forceinline__ void ldn(uint32_t taddr, int *v)
{
    static_assert(N == 4 || N == 8 || N == 16, "burst");
    if (N == 16)
        ld16(taddr, v);
    else if (N == 8)
        ld8(taddr, v);
    else
        ld4(taddr, v);
}

__device__ __forceinline__ void phase64(uint64_t idx, uint64_t q, double two_over_q, double &c, double &s)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    sincospi((double)sidx * two_over_q, &s, &c);
}

// exact FP64 value of an int64 |x| < 2^51: 1.5*2^52 + x has the same
// exponent, so the bit pattern is the integer sum (INT pipe) and one DADD
// removes the bias (FP64 pipe) -- no XU conversion
__device__ __forceinline__ double i64_to_f64_exact(long long x)
{
    return __longlong_as_double(0x4338000000000000LL + x) - 0x1.8p52;
}

__constant__ uint32_t c_pow2[2] = {1u << 14, 1u << 28};  // CONV 7 multipliers

// 6 digits: 2^41 T = D_0 2^28 + D_1 2^14 + D_2 (D_1, D_2 >= 0, < 2^21): the 2^52 bit
// pattern of D_1 2^14 + D_2 (exact), D_0 through one I2F, one DFMA
__device__ __forceinline__ double combine3(int d0, int d1, int d2)
{
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 16384, a;\n\t}"
        : "=l"(hb)
        : "r"((uint32_t)d2), "r"(0x43300000u), "r"((uint32_t)d1));
    return fma((double)d0, 0x1p28, __longlong_as_double((long long)hb) - 0x1p52);
}

// T in units of T_SCALE from the 4 pair accumulators (one final rounding)
__device__ __forceinline__ double combine(int d0, int d1, int d2, int d3)
{
    const long long hi = (long long)d0 * 16384 + d1;  // |.| < 2^35, exact
    const long long lo = (long long)d2 * 16384 + d3;
#if SHB_I8_CONV == 7
    // exact at full width: 2^55 T = D_0 2^42 + H',  H' = D_1 2^28 + D_2 2^14 + D_3 < 2^49
    // (D_1..D_3 >= 0): two IMAD.WIDE.U32 build the bit pattern of 2^52 + H' (bias in the
    // first addend's high word), one DADD removes it (exact), D_0 through one I2F, one DFMA
    (void)hi;
    (void)lo;
    // (the multipliers come from constant memory so that ptxas keeps one IMAD.WIDE.U32
    // each instead of expanding a power-of-two multiply into shift/add pairs)
    unsigned long long t, hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, %4, a;\n\t}"
        : "=l"(t)
        : "r"((uint32_t)d3), "r"(0x43300000u), "r"((uint32_t)d2), "r"(c_pow2[0]));
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(hb) : "r"((uint32_t)d1), "r"(c_pow2[1]), "l"(t));
    return fma((double)d0, 0x1p42, __longlong_as_double((long long)hb) - 0x1p52);
#elif SHB_I8_CONV == 6
    // as 5, but D_0 (signed) enters through the 1.5*2^52 bit pattern (one signed
    // IMAD.WIDE, INT pipe) instead of an I2F (XU pipe): one DFMA gives
    // D_0 2^34 - 2^52 exactly (|D_0| < 2^21), one DADD adds the 2^52 + H pattern
    (void)hi;
    (void)lo;
    const uint32_t l = ((uint32_t)d2 << 6) + (((uint32_t)d3 + 128u) >> 8);
    unsigned long long hb;
    long long b0;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    asm("mad.wide.s32 %0, %1, 1, %2;" : "=l"(b0) : "r"(d0), "l"(0x4338000000000000LL));
    const double t0 = fma(__longlong_as_double(b0), 0x1p34, -(0x1.8p86 + 0x1p52));
    return t0 + __longlong_as_double((long long)hb);
#elif SHB_I8_CONV == 8
    // as 5 with D_3 / 2^8 truncated instead of rounded (one ALU op less; the
    // extra 2^-48 absolute on T is below the FP64 rounding of T itself for |T| > 4)
    (void)hi;
    (void)lo;
    const uint32_t l = ((uint32_t)d2 << 6) + ((uint32_t)d3 >> 8);
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    return fma((double)d0, 0x1p34, __longlong_as_double((long long)hb) - 0x1p52);
#elif SHB_I8_CONV == 5
    // 2^47 T = D_0 2^34 + H,  H = D_1 2^20 + lo (< 2^42), lo = D_2 2^6 + round(D_3 / 2^8):
    // one IMAD.WIDE.U32 forms the bit pattern of 2^52 + H (bias in the addend's high
    // word), one DADD removes it (exact), D_0 (signed) through one I2F, one DFMA
    (void)hi;
    (void)lo;
    const uint32_t l = ((uint32_t)d2 << 6) + (((uint32_t)d3 + 128u) >> 8);
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    return fma((double)d0, 0x1p34, __longlong_as_double((long long)hb) - 0x1p52);
#elif SHB_I8_CONV == 4
    // 2^47 T = D_0 2^34 + D_1 2^20 + lo,  lo = D_2 2^6 + round(D_3 / 2^8) (< 2^28, int32):
    // D_1 and lo enter through the 2^52 bit pattern (exact, FP64 pipe), D_0 (signed)
    // through one I2F; the 2^-8 rounding of D_3 is <= 2^-48 absolute on T (below the
    // FP64 rounding of T itself)
    (void)hi;
    (void)lo;
    const uint32_t l = ((uint32_t)d2 << 6) + (((uint32_t)d3 + 128u) >> 8);
    const double m1 = __hiloint2double(0x43300000, d1) - 0x1p52;
    const double u = fma(m1, 0x1p20, __hiloint2double(0x43300000, (int)l)) - 0x1p52;  // exact, < 2^42
    return fma((double)d0, 0x1p34, u);
#elif SHB_I8_CONV == 3
    // D_1, D_2, D_3 >= 0 (unsigned digits, non-negative weights): the bias
    // 1.5*2^52 rides in the high word of the IMAD.WIDE addend
    (void)hi;
    (void)lo;
    const long long hb = (long long)d0 * 16384LL + (long long)(0x4338000000000000ULL | (uint32_t)d1);
    const unsigned long long lb = (unsigned long long)(uint32_t)d2 * 16384ULL + (0x4338000000000000ULL | (uint32_t)d3);
    return fma(__longlong_as_double(hb) - 0x1.8p52, 0x1p28, __longlong_as_double((long long)lb) - 0x1.8p52);
#elif SHB_I8_CONV == 0
    return fma((double)hi, 0x1p28, (double)lo);
#elif SHB_I8_CONV == 1
    return fma((double)hi, 0x1p28, i64_to_f64_exact(lo));
#else
    return fma(i64_to_f64_exact(hi), 0x1p28, i64_to_f64_exact(lo));
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
    unsigned long long *trace;  // SHB_I8_TRACE builds: clock64 stamps of CTA 0 (exploration)
};

#ifdef SHB_I8_TRACE
#define I8_TR(cond, slot)                                                                  \
    do {                                                                                   \
        if (p.trace && blockIdx.x == 0 && (cond)) p.trace[(slot)] = clock64();             \
    } while (0)
#else
#define I8_TR(cond, slot) \
    do {                  \
    } while (0)
#endif

__global__ void __launch_bounds__(THREADS, 1) dft_i8_uniform_kernel(const Args p)
{
    extern __shared__ unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;                  // [comp][digit] A operands
    unsigned char *sB = base + G_BYTES;        // [ones128, ones1, mask128, mask1]
    // per component c: full_bar[c] (MMA -> workers), empty_bar[c] (workers -> MMA)
    __shared__ __align__(8) uint64_t full_bar[2], empty_bar[2], a_ready[2];
    __shared__ uint32_t tmem_base_sh;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t q = p.q, qmask = q - 1;
    const uint64_t nsb = (p.length + SB_AMPS - 1) / SB_AMPS;
    const uint64_t last_amps = p.length - (nsb - 1) * SB_AMPS;  // in (0, SB_AMPS]
    const int last_rb = (int)((last_amps + BK - 1) / BK);
    // MMA N of the last super-block: a multiple of 16 and of whole load bursts per worker
    const int last_n = ((last_rb + LAST_ALIGN - 1) / LAST_ALIGN) * LAST_ALIGN;

    // weights (B operands: row = row-block jj, K-major, u8): 128 / 1 times ones / last mask
    for (int i = tid; i < NB * BK; i += THREADS) {
        const int jj = i / BK, k = i % BK;
        const uint32_t off = kmajor(jj, k);
        const bool live = (uint64_t)jj * BK + k < last_amps;
        if (off < (uint32_t)ONES_BYTES) {
            sB[off] = 128;
            sB[ONES_BYTES + off] = 1;
        }
        sB[2 * ONES_BYTES + off] = live ? 128 : 0;
        sB[2 * ONES_BYTES + B_BYTES + off] = live ? 1 : 0;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr(&tmem_base_sh)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int c2 = 0; c2 < 2; c2++) {
            mbar_init(&full_bar[c2], 1);
            mbar_init(&empty_bar[c2], WORKERS);
        }
        mbar_init(&a_ready[0], WORKERS);
        mbar_init(&a_ready[1], WORKERS);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_sh;

    if (warp == MMA_WARP) {
        // ---------------------------------------------------------- MMA issuer
        // The whole warp walks the loop (barrier waits, uniform descriptor
        // arithmetic: base descriptor + compile-time offset >> 4); one elected
        // lane issues.  At N = 64 an int8 MMA is 32 tensor cycles, so the issue
        // path has to stay short.
        const uint64_t adesc = smem_desc(smem_addr(sA)), bdesc = smem_desc(smem_addr(sB));
        const uint64_t bdesc_dedup = bdesc & ~((0x3FFFull << 16) | (0x3FFFull << 32));
#ifdef SHB_I8_ADEDUP_PROBE
        // timing probe only (WRONG results): every A operand reads one core matrix,
        // to separate the shared-memory operand reads from the tensor/TMEM cost
        const uint64_t adesc_probe = adesc & ~((0x3FFFull << 16) | (0x3FFFull << 32));
#define SHB_I8_ADESC adesc_probe
#else
#define SHB_I8_ADESC adesc
#endif
        uint64_t g = 0;  // super-blocks issued so far
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, it++) {
            wait_bar(&a_ready[0], it & 1u);  // G of this tile (GSPLIT: its Re half) is in shared memory
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            I8_TR(lane == 0 && it < 4, 10000 + it * 1000);
            for (uint64_t sb = 0; sb < nsb; sb++, g++) {
                const bool last = sb + 1 == nsb;
                const int n = last ? last_n : NB;
                const uint32_t id_s = idesc(n, true), id_u = idesc(n, false);
                // SHB_I8_BDEDUP: the all-128 / all-1 weights of a full super-block read
                // one 8 x 16 B core matrix for every row group and k group (LBO = SBO = 0)
                const uint64_t bd = ((BDEDUP || NDIG != 8) && !last) ? bdesc_dedup : bdesc;
                const uint64_t w128 = bd + (uint64_t)((last ? 2 * ONES_BYTES : 0) >> 4);
                const uint64_t w1 = w128 + (uint64_t)((last ? B_BYTES : ONES_BYTES) >> 4);
#pragma unroll
                for (int comp = 0; comp < 2; comp++) {
                    // this component's accumulators were drained for super-block g - 1
                    I8_TR(lane == 0 && it < 4 && sb < 100, 10000 + it * 1000 + 1 + 8 * sb + 3 * comp);
                    if (g >= 1 && (PHASES == 2 || comp == 0)) wait_bar(&empty_bar[comp], (uint32_t)(g - 1) & 1u);
                    if (GSPLIT && comp == 1 && sb == 0) wait_bar(&a_ready[1], it & 1u);  // Im half of G
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    I8_TR(lane == 0 && it < 4 && sb < 100, 10000 + it * 1000 + 2 + 8 * sb + 3 * comp);
                    if (elect_one()) {
#pragma unroll
                        // MMA_ORDER 0: pair-major (each accumulator's 2 KCH MMAs back to back);
                        // 1: K-chunk-major (consecutive MMAs rotate over the NPAIR accumulators)
#pragma unroll
                        for (int o = 0; o < NPAIR * KCH; o++) {
                            const int pr = MMA_ORDER ? o % NPAIR : o / KCH, s = MMA_ORDER ? o / NPAIR : o % KCH;
                            const uint32_t d = tmem + (comp * NPAIR + pr) * NB;
                            const uint64_t ahi = SHB_I8_ADESC + (uint64_t)((comp * NDIG + 2 * pr) * A_BYTES >> 4);
                            const uint64_t alo = ahi + (A_BYTES >> 4);
                            const uint64_t koff = (uint64_t)(s * 2 * LBO >> 4);
                            mma(d, ahi + koff, w128 + koff, pr == 0 ? id_s : id_u, s > 0);
                            mma(d, alo + koff, w1 + koff, id_u, 1);
                        }
                        if (PHASES == 2 || comp == 1) commit(&full_bar[PHASES == 2 ? comp : 0]);
                    }
                    __syncwarp();
                    I8_TR(lane == 0 && it < 4 && sb < 100, 10000 + it * 1000 + 3 + 8 * sb + 3 * comp);
                }
            }
        }
    } else {
        // ------------------------------------- G builders + folders (row = TMEM lane = output)
        // worker w: row = w % 128 (warp w/32 reads TMEM lane quarter (w/32) % 4),
        // part = w / 128 builds the 16-k groups part, part + SPLIT, ... of G and
        // folds row-blocks [part n/SPLIT, (part+1) n/SPLIT) of every super-block
        const int row = tid & (TILE - 1), part = tid >> 7;
        const uint32_t lane_addr = (uint32_t)(32 * (warp & 3)) << 16;
        __shared__ double vpart[SPLIT][2][TILE];
        __shared__ double wsum[WORKERS / 32];
        uint64_t g = 0;
        uint32_t itw = 0;
        const bool trw = (tid == 0 || tid == 160);
        const int trb = tid == 0 ? 0 : 5000;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, itw++) {
            const uint64_t c = p.c_begin + t * TILE + row;
            I8_TR(trw && itw < 4, trb + itw * 1000);
            // G[c, k] = e^{+2 pi i k stride c / q}: exact sincospi every 16 k, FP64
            // rotation in between (<= ~15 ulp, as the DMMA engine's G), rounded to
            // X = rint(G 2^55) and split into 8 digits per component.  The MMAs
            // reading the previous tile's G are complete: this worker waited on
            // the commit of that tile's last super-block.
#pragma unroll
            for (int cpass = 0; cpass < (GSPLIT ? 2 : 1); cpass++) {
                // GSPLIT: Re digits first, released to the MMAs (comp 0 of the first
                // super-block runs under the Im build), then Im
                const int c_lo = GSPLIT ? cpass : 0, c_hi = GSPLIT ? cpass + 1 : 2;
                double wr, wi;
                phase64((p.stride * c) & qmask, q, p.two_over_q, wr, wi);
                for (int k0 = part * 16; k0 < BK; k0 += 16 * SPLIT) {
                    double gr, gi;
                    phase64(((uint64_t)k0 * p.stride * c) & qmask, q, p.two_over_q, gr, gi);
                    uint32_t pk[2][NDIG][4];
                    if constexpr (GPACK && NDIG == 8) {
                        // per value: X = rint(G 2^55) = d0 2^49 + R (R = X mod 2^49), digit
                        // bytes spread within a word (S_hi = u1..u4, S_lo = d0, u5..u7), then a
                        // 4 x 4 byte transpose (PRMT) across 4 consecutive k per digit
                        uint32_t sh[2][4], sl[2][4];
#pragma unroll
                        for (int e = 0; e < 16; e++) {
#pragma unroll
                            for (int comp = c_lo; comp < c_hi; comp++) {
                                const long long X = __double2ll_rn((comp ? gi : gr) * 0x1p55);
                                const uint32_t lo = (uint32_t)X, hi = (uint32_t)((unsigned long long)X >> 32);
                                const uint32_t d0 = (uint32_t)((int)hi >> 17);
                                const uint32_t h28 = __funnelshift_r(lo, hi & 0x1FFFFu, 21);
                                sh[comp][e & 3] = (h28 & 0x7Fu) | ((h28 << 1) & 0x7F00u) | ((h28 << 2) & 0x7F0000u) |
                                                  ((h28 << 3) & 0x7F000000u);
                                sl[comp][e & 3] = (lo & 0x7Fu) | ((lo << 1) & 0x7F00u) | ((lo << 2) & 0x7F0000u) | (d0 << 24);
                                if ((e & 3) == 3) {
                                    const int m = e >> 2;
                                    // S bytes b0..b3 -> digits: S_hi (4, 3, 2, 1), S_lo (7, 6, 5, 0)
                                    const uint32_t ah = __byte_perm(sh[comp][0], sh[comp][1], 0x5140),
                                                   bh = __byte_perm(sh[comp][2], sh[comp][3], 0x5140),
                                                   ch = __byte_perm(sh[comp][0], sh[comp][1], 0x7362),
                                                   dh = __byte_perm(sh[comp][2], sh[comp][3], 0x7362);
                                    pk[comp][4][m] = __byte_perm(ah, bh, 0x5410);
                                    pk[comp][3][m] = __byte_perm(ah, bh, 0x7632);
                                    pk[comp][2][m] = __byte_perm(ch, dh, 0x5410);
                                    pk[comp][1][m] = __byte_perm(ch, dh, 0x7632);
                                    const uint32_t al = __byte_perm(sl[comp][0], sl[comp][1], 0x5140),
                                                   bl = __byte_perm(sl[comp][2], sl[comp][3], 0x5140),
                                                   cl = __byte_perm(sl[comp][0], sl[comp][1], 0x7362),
                                                   dl = __byte_perm(sl[comp][2], sl[comp][3], 0x7362);
                                    pk[comp][7][m] = __byte_perm(al, bl, 0x5410);
                                    pk[comp][6][m] = __byte_perm(al, bl, 0x7632);
                                    pk[comp][5][m] = __byte_perm(cl, dl, 0x5410);
                                    pk[comp][0][m] = __byte_perm(cl, dl, 0x7632);
                                }
                            }
                            const double nr = fma(gr, wr, -gi * wi), ni = fma(gr, wi, gi * wr);
                            gr = nr;
                            gi = ni;
                        }
                    } else {
#pragma unroll
                    for (int e = 0; e < 16; e++) {
#pragma unroll
                        for (int comp = c_lo; comp < c_hi; comp++) {
                            uint32_t dig[NDIG];
                            if constexpr (NDIG == 8) {
                                const long long X = __double2ll_rn((comp ? gi : gr) * 0x1p55);
                                const int d0 = (int)(X >> 49);
                                const unsigned long long R = (unsigned long long)(X - ((long long)d0 << 49));
                                const uint32_t hi28 = (uint32_t)(R >> 21), lo21 = (uint32_t)R & 0x1FFFFFu;
                                const uint32_t dd8[8] = {(uint32_t)d0 & 0xFFu, hi28 >> 21, (hi28 >> 14) & 127u,
                                                         (hi28 >> 7) & 127u, hi28 & 127u, lo21 >> 14,
                                                         (lo21 >> 7) & 127u, lo21 & 127u};
#pragma unroll
                                for (int dd = 0; dd < NDIG; dd++) dig[dd] = dd8[dd % 8];
                            } else {
                                // X = rint(G 2^41) = d0 2^35 + u1 2^28 + ... + u5
                                const long long X = __double2ll_rn((comp ? gi : gr) * 0x1p41);
                                const int d0 = (int)(X >> 35);
                                const unsigned long long R = (unsigned long long)(X - ((long long)d0 << 35));
                                const uint32_t hi21 = (uint32_t)(R >> 14), lo14 = (uint32_t)R & 0x3FFFu;
                                const uint32_t dd6[6] = {(uint32_t)d0 & 0xFFu, hi21 >> 14, (hi21 >> 7) & 127u,
                                                         hi21 & 127u, lo14 >> 7, lo14 & 127u};
#pragma unroll
                                for (int dd = 0; dd < NDIG; dd++) dig[dd] = dd6[dd % 6];
                            }
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
                    }
                    const uint32_t off = kmajor(row, k0);
#pragma unroll
                    for (int comp = c_lo; comp < c_hi; comp++)
#pragma unroll
                        for (int dd = 0; dd < NDIG; dd++)
                            *reinterpret_cast<uint4 *>(sA + (comp * NDIG + dd) * A_BYTES + off) =
                                make_uint4(pk[comp][dd][0], pk[comp][dd][1], pk[comp][dd][2], pk[comp][dd][3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&a_ready[GSPLIT ? cpass : 0]);
            }
            I8_TR(trw && itw < 4, trb + itw * 1000 + 1);

            // fold this worker's part of every super-block: h = h * W + 2^55 T[jj] (FP64), W = w^{-BK},
            // as CHAINS interleaved Horner chains with W^CHAINS, joined at the end of the part
            double Wr, Wi, W2r, W2i, Sr, Si;
            {
                double co, si;
                phase64(((uint64_t)BK * p.stride * c) & qmask, q, p.two_over_q, co, si);
                Wr = co;
                Wi = -si;
                phase64(((uint64_t)CHAINS * BK * p.stride * c) & qmask, q, p.two_over_q, co, si);
                W2r = co;
                W2i = -si;
                // seed step between full super-blocks: e^{+2 pi i NB BK stride c / q}
                phase64(((uint64_t)NB * BK * p.stride * c) & qmask, q, p.two_over_q, Sr, Si);
            }
            double vr = 0.0, vi = 0.0, sdr = 0.0, sdi = 0.0;
#ifdef SHB_I8_DRAIN_PROBE
            int probe_x = 0;
#endif
            for (uint64_t sb = 0; sb < nsb; sb++, g++) {
                const bool last = sb + 1 == nsb;
                const int n = last ? last_n : NB;
                const int rbw = n / SPLIT;  // whole load bursts
                const int j_lo = part * rbw;
                const uint32_t dre = tmem + lane_addr + j_lo, dim = dre + COMP_COLS;
                double hr[CHAINS], hi[CHAINS];
#pragma unroll
                for (int k2 = 0; k2 < CHAINS; k2++) hr[k2] = hi[k2] = 0.0;
#if SHB_I8_PHASES == 1
                // one hand-over: per burst both components (Re then Im columns)
                {
                    int acc[2][2 * NPAIR][CH];
                    I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 2 + 8 * sb);
                    wait_bar(&full_bar[0], (uint32_t)g & 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 3 + 8 * sb);
#pragma unroll
                    for (int pr = 0; pr < 2 * NPAIR; pr++) ldn<CH>(dre + pr * NB, acc[0][pr]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int ch = 0; ch < NCH; ch++) {
                        if (ch * CH < rbw) {
                            if (PREFETCH && (ch + 1) * CH < rbw) {
#pragma unroll
                                for (int pr = 0; pr < 2 * NPAIR; pr++)
                                    ldn<CH>(dre + pr * NB + (ch + 1) * CH, acc[(ch + 1) & 1][pr]);
                            }
                            const int bi = PREFETCH ? (ch & 1) : 0;
#ifdef SHB_I8_DRAIN_PROBE
                            // timing probe only (WRONG results): the loads without the FP64 work
#pragma unroll
                            for (int e = 0; e < CH; e++)
#pragma unroll
                                for (int pr = 0; pr < 2 * NPAIR; pr++) probe_x ^= acc[bi][pr][e];
                            if (false)
#endif
#pragma unroll
                            for (int e = 0; e < CH; e++) {
                                double tr, ti;
                                if constexpr (NDIG == 8) {
                                    tr = combine(acc[bi][0][e], acc[bi][1][e], acc[bi][2][e], acc[bi][3][e]);
                                    ti = combine(acc[bi][4][e], acc[bi][5][e], acc[bi][6][e], acc[bi][7][e]);
                                } else {
                                    tr = combine3(acc[bi][0][e], acc[bi][1][e], acc[bi][2][e]);
                                    ti = combine3(acc[bi][NPAIR][e], acc[bi][NPAIR + 1][e], acc[bi][NPAIR + 2][e]);
                                }
                                const int k2 = e % CHAINS;
                                const double nr = fma(hr[k2], W2r, fma(-hi[k2], W2i, tr));
                                const double ni = fma(hr[k2], W2i, fma(hi[k2], W2r, ti));
                                hr[k2] = nr;
                                hi[k2] = ni;
                            }
                            if (!PREFETCH && (ch + 1) * CH < rbw) {
#pragma unroll
                                for (int pr = 0; pr < 2 * NPAIR; pr++)
                                    ldn<CH>(dre + pr * NB + (ch + 1) * CH, acc[0][pr]);
                            }
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        }
                    }
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(&empty_bar[0]);
                    I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 6 + 8 * sb);
                }
#else
                // Re: convert this worker's row-blocks, then hand the Re half back.
                // Loads run one burst ahead (wait::ld covers the burst issued
                // before the previous conversions).
                double tre[RBW];
                int acc[2][NPAIR][CH];
                I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 2 + 8 * sb);
                wait_bar(&full_bar[0], (uint32_t)g & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 3 + 8 * sb);
#pragma unroll
                for (int pr = 0; pr < NPAIR; pr++) ldn<CH>(dre + pr * NB, acc[0][pr]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int ch = 0; ch < NCH; ch++) {
                    if (ch * CH < rbw) {
                        if ((ch + 1) * CH < rbw) {
#pragma unroll
                            for (int pr = 0; pr < NPAIR; pr++) ldn<CH>(dre + pr * NB + (ch + 1) * CH, acc[(ch + 1) & 1][pr]);
                        }
#pragma unroll
                        for (int e = 0; e < CH; e++)
                            tre[ch * CH + e] = combine(acc[ch & 1][0][e], acc[ch & 1][1][e], acc[ch & 1][2][e],
                                                       acc[ch & 1][3][e]);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&empty_bar[0]);
                I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 4 + 8 * sb);
                // Im + the Horner over the row-blocks
                wait_bar(&full_bar[1], (uint32_t)g & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 5 + 8 * sb);
#pragma unroll
                for (int pr = 0; pr < NPAIR; pr++) ldn<CH>(dim + pr * NB, acc[0][pr]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int ch = 0; ch < NCH; ch++) {
                    if (ch * CH < rbw) {
                        if ((ch + 1) * CH < rbw) {
#pragma unroll
                            for (int pr = 0; pr < NPAIR; pr++) ldn<CH>(dim + pr * NB + (ch + 1) * CH, acc[(ch + 1) & 1][pr]);
                        }
#pragma unroll
                        for (int e = 0; e < CH; e++) {
                            const double ti = combine(acc[ch & 1][0][e], acc[ch & 1][1][e], acc[ch & 1][2][e],
                                                      acc[ch & 1][3][e]);
                            const double tr = tre[ch * CH + e];
                            const int k2 = e % CHAINS;  // CH % CHAINS == 0: chain of position ch*CH + e
                            const double nr = fma(hr[k2], W2r, fma(-hi[k2], W2i, tr));
                            const double ni = fma(hr[k2], W2i, fma(hi[k2], W2r, ti));
                            hr[k2] = nr;
                            hi[k2] = ni;
                        }
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&empty_bar[1]);
                I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 6 + 8 * sb);
#endif
                // join the chains: h = (..(h_0 W + h_1) W + ..) W + h_{CHAINS-1}
                double fr = hr[0], fi = hi[0];
#pragma unroll
                for (int k2 = 1; k2 < CHAINS; k2++) {
                    const double nr = fma(fr, Wr, fma(-fi, Wi, hr[k2]));
                    const double ni = fma(fr, Wi, fma(fi, Wr, hi[k2]));
                    fr = nr;
                    fi = ni;
                }
                // seed of the last folded row-block, e^{+2 pi i a_last c / q} with
                // a_last = a0 + (sb*NB + j_lo + rbw - 1)*BK*stride: exact sincospi
                // for the last super-block and every SEED_EVERY-th, else the
                // previous seed times S (same full-super-block offset)
                double sc, ss;
                if (last || sb % SEED_EVERY == 0) {
                    const uint64_t a_last = p.a0 + ((sb * NB + (uint64_t)(j_lo + rbw - 1)) * BK) * p.stride;
                    phase64((a_last * c) & qmask, q, p.two_over_q, sc, ss);
                } else {
                    sc = fma(sdr, Sr, -sdi * Si);
                    ss = fma(sdr, Si, sdi * Sr);
                }
                sdr = sc;
                sdi = ss;
                I8_TR(trw && itw < 4 && sb < 100, trb + itw * 1000 + 7 + 8 * sb);
                vr = fma(sc, fr, fma(-ss, fi, vr));
                vi = fma(sc, fi, fma(ss, fr, vi));
            }
#ifdef SHB_I8_DRAIN_PROBE
            vr += (double)probe_x;
#endif
            // combine the parts (fixed order 0, 1, ..., SPLIT-1), then the
            // epilogue: output factor (with 2^-55), |V|^2 (hypot^2, as
            // np.abs(.)**2), tile sum
            if (part > 0) {
                vpart[part][0][row] = vr;
                vpart[part][1][row] = vi;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(WORKERS) : "memory");
            double pr = 0.0;
            if (part == 0) {
#pragma unroll
                for (int k2 = 1; k2 < SPLIT; k2++) {
                    vr += vpart[k2][0][row];
                    vi += vpart[k2][1][row];
                }
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

}  // namespace SHB_I8_NS

#ifdef SHB_I8_TRACE
static unsigned long long *&i8_trace_ptr()
{
    static unsigned long long *p = nullptr;
    return p;
}
#endif

// Caller contract as shb_dft_uniform (validated there); block sums in the
// caller's shb_dft_num_blocks(c_count, SHB_FP64) layout (slot_outputs per slot).
int SHB_I8_ENTRY(uint64_t length, uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin, uint64_t c_count,
                   double out_re, double out_im, double *d_out, double *d_prob, double *d_block_sums,
                   uint64_t slot_outputs, cudaStream_t st)
{
    using namespace SHB_I8_NS;
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
    a.out_re = out_re * T_SCALE;
    a.out_im = out_im * T_SCALE;
    a.out = (double2 *)d_out;
    a.prob = d_prob;
    Scratch part;
    if (d_block_sums) {
        SHB_TRY(scratch_alloc(part, sizeof(double) * a.ntiles, st));
        a.tile_sums = (double *)part.ptr;
    }
#ifdef SHB_I8_TRACE
    static unsigned long long *trace_buf = nullptr;
    if (!trace_buf) SHB_TRY_CUDA(cudaMalloc(&trace_buf, 20000 * sizeof(unsigned long long)));
    SHB_TRY_CUDA(cudaMemsetAsync(trace_buf, 0, 20000 * sizeof(unsigned long long), st));
    a.trace = trace_buf;
    i8_trace_ptr() = trace_buf;
#endif
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

#ifdef SHB_I8_TRACE
// exploration builds only: copy the 20000 clock64 stamps of the last launch
extern "C" int shb_i8_trace(unsigned long long *host)
{
    cudaDeviceSynchronize();
    if (!shb::i8_trace_ptr()) return -1;
    return (int)cudaMemcpy(host, shb::i8_trace_ptr(), 20000 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif
