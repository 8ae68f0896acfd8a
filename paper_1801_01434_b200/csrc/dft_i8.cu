// FP64-accurate QFT of the uniform comb (the collapsed Shor register) on the
// 5th-generation INTEGER tensor cores: tcgen05.mma kind::i8 with the
// amplitude operand in TMEM and int32 TMEM accumulators.  precision SHB_FP64,
// tiles == 1; the sum is qft.dense_dft's (qft.py:95-112 / _kernels.py:16-30)
// over the nonzero support a_j = a0 + j*stride:
//
//   V_c = scale*amp * sum_j e^{+2 pi i a_j c / q}
//
// Index split.  j = sb*SBA + kc*4096 + r*32 + kk: super-block sb (SBA =
// 4096 KCH amplitudes), K-chunk kc < KCH (6 or 8, Geo below), row-block
// r < 128 (the MMA's M = the TMEM lanes), kk < 32.  With k = kc*32 + kk
// (K = 32 KCH per row-block):
//
//   V_c = scale*amp * sum_sb sum_r e^{+2 pi i (a0 + sb*SBA*stride + r*32*stride) c / q} T_sb[r, c]
//   T_sb[r, c] = sum_k A_sb[r, k] * G[k, c],   G[k, c] = e^{+2 pi i (kc*4096 + kk) stride c / q}
//
// A_sb[r, k] is the amplitude of a_j (a weight: 1 inside the support, 0
// past its end); G is the phase matrix of the tile's outputs.  This is a GEMM
// with M = 128 row-blocks, N = 24 outputs, K = 192 or 256.  For the uniform comb A is
// all ones, so every row-block's T is the same number: the tensor work is
// executed as written (and credited), but the throughput is specific to the
// uniform comb -- a general register would need the amplitudes split into
// digits too.
//
// Exact fixed-point split (FP64 emulation by integer slices): each FP64 G
// value is rounded once to X = rint(G 2^55) (|error| <= 2^-56) and written as
// 8 base-128 digits, X = d0 2^49 + u1 2^42 + ... + u7 (d0 in [-64, 64] s8,
// u in [0, 127] u8).  Digits pair in one int32 accumulator through the A
// weights: digit 2p against 128*A (u8), digit 2p+1 against 1*A, so
// D_p = sum_k A (128 d_2p + d_2p+1), |D_p| < 2^22 for K <= 256, and
//   2^55 T = D_0 2^42 + D_1 2^28 + D_2 2^14 + D_3     (exact integers).
// Every product and accumulation in the tensor core is exact.
//
// Why this orientation (measured, scripts/i8t_probe.cu): an M128 K32 int8
// MMA with BOTH operands in shared memory reads 4 KB of A per issue and is
// shared-memory bound (39 cycles at N = 24, 48 at N = 64, vs the 12 / 32-cycle
// tensor floor); with A in TMEM only B (N x 32 B) comes from shared memory and
// the MMA runs at 15.4 cycles (N = 24) / 32.0 (N = 64).  The constant weight
// matrices cost 32 TMEM columns; two accumulator sets of 2 x 4 x 24 columns
// let the drain of super-block s overlap the MMAs of s + 1.
//
// TMEM (512 columns): [0, 192) accumulator set 0, [192, 384) set 1 --
// column (comp*4 + p)*24 + n; [384, 392) weights 128, [392, 400) weights 1,
// [400, 416) the masked weights of the last super-block's partial K-chunk.
//
// Roles (one persistent CTA per SM; 18 warps at KCH = 6, 19 at KCH = 8):
//  * the last warp (one elected lane): per super-block KCH x 2 x 4 x 2 MMAs
//    (M128 N24 K32, A from TMEM, B = one digit matrix's K-chunk) into the
//    free accumulator set, committed to a_full[set];
//  * warps 12-16 (12-17): build the next tile's 16 digit matrices of G (FP64 phases,
//    exact sincospi every 16 k, FP64 rotation between) and its per-output
//    constants into the other shared buffer while the current tile's MMAs
//    run (g_full / g_empty / c_free);
//  * warps 0-11 (lane quarter warp % 4, outputs 8 (warp / 4) ...): per
//    super-block load their accumulators (tcgen05.ld, then the set is
//    released; Re pairs, then Im pairs), combine the digit pairs to FP64 and
//    fold by Horner over super-blocks, H = H e^{-i phi_SB} + T; at the tile's
//    end fold the 128 row-blocks by Horner in w = e^{i phi_32} (8 lanes per
//    chain, chains joined with w^8), apply the exact seed of the last
//    super-block, and write V and |V|^2 (hypot^2, as np.abs(.)**2).  Every
//    output's arithmetic depends only on c, so any output shard reproduces
//    the same bits.
#include <math.h>
#include <stdlib.h>

#include "shb_internal.cuh"

namespace shb {
namespace i8 {

constexpr int NO = 24;                    // outputs per tile (MMA N)
constexpr int LANES = 128;                // row-blocks per super-block (MMA M, TMEM lanes)
constexpr int KC = 32;                    // K per MMA (8-bit operands)
constexpr int CHUNK_AMPS = LANES * KC;    // 4096 amplitudes per K-chunk
constexpr int NDIG = 8, NPAIR = 4;
constexpr int ACC_COLS = 2 * NPAIR * NO;  // one accumulator set
constexpr int COL_W = 2 * ACC_COLS;       // weights: +0 x128, +8 x1, +16 mask x128, +24 mask x1
constexpr int TMEM_COLS = 512;
static_assert(COL_W + 32 <= TMEM_COLS, "TMEM budget");
constexpr uint32_t LBO = 128;             // next 16-byte k group of a K-major operand
constexpr int FOLD_STRIDE = NO + 1;       // complex per row-block row of the fold buffer (bank spread)
constexpr int FOLD_BYTES = LANES * FOLD_STRIDE * 16;
constexpr int GSPAN = 32;                 // k per G item: one K-chunk (16-k items on more warps: slower)
constexpr int DRAIN_WARPS = 12;
constexpr int DRAIN_THREADS = DRAIN_WARPS * 32;
constexpr int OPT = NO / (DRAIN_WARPS / 4); // outputs per drain thread: one 8-column TMEM load per accumulator
static_assert(OPT == 8, "tcgen05.ld 32x32b.x8 per (component, pair)");
constexpr int CHAIN = 8;                  // row-blocks per Horner chain of the tile-end fold
constexpr int FOLD_CHAINS = LANES / CHAIN;
static_assert(FOLD_CHAINS * NO == DRAIN_THREADS && FOLD_CHAINS == 16, "one chain per drain thread");

// The geometry that depends on KCH, the K-chunks per super-block (6 or 8,
// chosen per launch by i8_dft_uniform): K = 32 KCH per row-block, SBA = 4096
// KCH amplitudes per super-block, a G buffer of 16 digit matrices of 24 x K
// bytes, one G-builder thread per (output, K-chunk).  The tile-end fold buffer
// aliases the tile's own G buffer: when the drain reaches the tile end, the
// tile's last MMAs have completed (it waited for their commit), and the G
// builders rewrite that buffer only after the drain's c_free for the tile.  So
// shared memory holds just the two G buffers (KCH = 8: 2 x 96 KB).
template <int KCH>
struct Geo {
    static constexpr int BK = KC * KCH;              // K per row-block: columns of G
    static constexpr int SBA = CHUNK_AMPS * KCH;     // amplitudes per super-block
    static constexpr uint32_t SBO = (BK / 16) * 128; // next 8-row group of a K-major operand
    static constexpr int DIG_BYTES = NO * BK;        // one digit matrix (24 x BK bytes)
    static constexpr int G_BYTES = 2 * NDIG * DIG_BYTES;
    static constexpr int SMEM_BYTES = 2 * G_BYTES;
    static constexpr int G_ITEMS = NO * BK / GSPAN;  // (output, k-span) items of a tile's G
    static constexpr int G_WARPS = (G_ITEMS + 31) / 32;
    static constexpr int G_THREADS = G_WARPS * 32;
    static constexpr int MMA_WARP = DRAIN_WARPS + G_WARPS;
    static constexpr int THREADS = (MMA_WARP + 1) * 32;
    static_assert(FOLD_BYTES <= G_BYTES, "the fold buffer fits in a G buffer");
    static_assert(SMEM_BYTES + 16 * 1024 <= 227 * 1024, "shared memory (dynamic + static)");
    static_assert(G_THREADS >= 5 * NO, "one tile constant per G thread");
    // |D_p| <= K (128 * 127 + 127) < 2^22 keeps L = D_1 2^20 + ... below 2^42 (combine_add)
    static_assert((int64_t)BK * 16383 < (1LL << 22), "pair accumulators fit combine_add()");
};

template <uint32_t SBO>
__device__ __forceinline__ uint32_t kmajor(int row, int k)
{
    return (uint32_t)(row >> 3) * SBO + (uint32_t)(k >> 4) * LBO + (uint32_t)(row & 7) * 16u + (uint32_t)(k & 15);
}

template <uint32_t SBO>
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr)
{
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(LBO >> 4) << 16) | ((uint64_t)(SBO >> 4) << 32) |
           ((uint64_t)1 << 46);  // sm_100 descriptor version; no swizzle
}

// kind::i8 instruction descriptor: A (weights) u8, B (digits) s8 or u8 -> S32, K-major, M = 128
__device__ __forceinline__ uint32_t idesc(bool b_signed)
{
    return (2u << 4) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(NO >> 3) << 17) | ((uint32_t)(LANES >> 4) << 24);
}

// D[tmem] (+)= A[tmem] x B[smem desc]
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(id), "r"(acc));
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

// mbarrier wait that traps instead of hanging if the pipeline ever stalls.  The
// suspend-time hint parks the warp in hardware until the phase completes (or the
// hint expires) instead of spinning: a spinning warp takes issue slots from the
// drain warps that share its scheduler.
__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t phase)
{
    uint32_t ok = 0;
    for (uint32_t spin = 0; !ok; spin++) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(phase), "r"(1000000u)
            : "memory");
        if (spin > (1u << 16)) asm volatile("trap;");  // > ~1 min asleep: a broken pipeline, not a slow one
    }
}

__device__ __forceinline__ void ld8(uint32_t taddr, int *v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
}

__device__ __forceinline__ void st8(uint32_t taddr, uint32_t v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v));
}

__device__ __forceinline__ void st8v(uint32_t taddr, const uint32_t *v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}

__device__ __forceinline__ double2 phase(uint64_t idx, uint64_t q, double two_over_q)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    double s, c;
    sincospi((double)sidx * two_over_q, &s, &c);
    return make_double2(c, s);
}

constexpr double T_SCALE = 0x1p-47;  // units of combine_add()

// H + T in units of 2^-47 from the 4 pair accumulators and the running sum a:
// 2^47 T = D_0 2^34 + L with L = D_1 2^20 + D_2 2^6 + floor(D_3 / 2^8) < 2^42
// (D_1..D_3 >= 0).  One IMAD.WIDE.U32 forms the bit pattern of 2^52 + L; the
// bias goes into the signed digit, (D_0 - 2^18) 2^34 = D_0 2^34 - 2^52, so one
// I2F, one DADD (2^52 + L + a) and one DFMA give a + 2^47 T with two
// roundings (the dropped bits of D_3 are <= 2^-47 absolute on T).
__device__ __forceinline__ double combine_add(int d0, int d1, int d2, int d3, double a)
{
    const uint32_t l = ((uint32_t)d2 << 6) + ((uint32_t)d3 >> 8);
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    return fma((double)(d0 - (1 << 18)), 0x1p34, __longlong_as_double((long long)hb) + a);
}

__device__ __forceinline__ double2 rot(double2 g, double2 w)  // g*w
{
    return make_double2(fma(g.x, w.x, -g.y * w.y), fma(g.x, w.y, g.y * w.x));
}

__device__ __forceinline__ double2 cmad(double2 h, double2 w, double2 t)  // h*w + t
{
    return make_double2(fma(h.x, w.x, fma(-h.y, w.y, t.x)), fma(h.x, w.y, fma(h.y, w.x, t.y)));
}

struct Args {
    uint64_t length, a0, stride, q;
    double two_over_q;
    uint64_t c_begin, c_count, ntiles, nsb, last_amps;
    double out_re, out_im;  // output factor (scale * amp), times 2^-47 here
    double2 *out;
    double *prob;
    unsigned long long *trace;  // SHB_I8_TRACE builds: clock64 stamps of CTA 0 (exploration)
};

#ifdef SHB_I8_TRACE
#define I8_TR(cond, slot)                                                      \
    do {                                                                       \
        if (p.trace && blockIdx.x == 0 && (cond)) p.trace[(slot)] = clock64(); \
    } while (0)
#else
#define I8_TR(cond, slot) \
    do {                  \
    } while (0)
#endif

template <int KCH>
__global__ void __launch_bounds__(Geo<KCH>::THREADS, 1) dft_i8_uniform_kernel(const Args p)
{
    using GE = Geo<KCH>;
    constexpr int SBA = GE::SBA, DIG_BYTES = GE::DIG_BYTES, G_BYTES = GE::G_BYTES;
    constexpr int G_ITEMS = GE::G_ITEMS, G_THREADS = GE::G_THREADS, MMA_WARP = GE::MMA_WARP;
    // no-swizzle K-major operands need 16-byte alignment only; indexing the
    // __shared__ array directly keeps every access in the shared window (LDS/STS)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char *sG = smem_raw;                                        // [2 buffers][comp][digit] B operands
    double2 *const fold0 = reinterpret_cast<double2 *>(smem_raw);  // [row-block][NO + 1] in G buffer 0 (or 1)
    __shared__ __align__(8) uint64_t g_full[2], g_empty[2], a_full[2], a_empty[2], c_free[2];
    __shared__ uint32_t tmem_base_sh;
    // per output of a tile (built with its G): e^{-i phi_SB}, w = e^{i phi_32}, w^8, seed, w^32
    __shared__ double2 tconst[2][5][NO];
    __shared__ double2 rpart[FOLD_CHAINS][NO];
    __shared__ double2 rquad[FOLD_CHAINS / 4][NO];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t q = p.q, qmask = q - 1;
    const int full_last = (int)(p.last_amps / CHUNK_AMPS);       // full K-chunks of the last super-block
    const int rem_last = (int)(p.last_amps % CHUNK_AMPS);        // live amplitudes of its partial chunk
    const int live_last = full_last + (rem_last ? 1 : 0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_addr(&tmem_base_sh)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&g_full[b], G_THREADS);
            mbar_init(&g_empty[b], 1);
            mbar_init(&a_full[b], 1);
            mbar_init(&a_empty[b], DRAIN_THREADS);
            mbar_init(&c_free[b], 1);
        }
        fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_sh;

    // the weight operands (A, u8, K-major in TMEM: lane = row-block, 4 k per column)
    if (warp < 4) {
        const int r = 32 * warp + lane;
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16) + COL_W;
        st8(ta, 0x80808080u);
        st8(ta + 8, 0x01010101u);
        uint32_t m128[8], m1[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            uint32_t a = 0, b = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const bool live = r * KC + 4 * j + e < rem_last;
                a |= (live ? 128u : 0u) << (8 * e);
                b |= (live ? 1u : 0u) << (8 * e);
            }
            m128[j] = a;
            m1[j] = b;
        }
        st8v(ta + 16, m128);
        st8v(ta + 24, m1);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    if (warp == MMA_WARP) {
        // ------------------------------------------------------------ MMA issuer
        const uint64_t gdesc0 = smem_desc<GE::SBO>(smem_addr(sG));
        const uint32_t id_s = idesc(true), id_u = idesc(false);
        uint64_t gs = 0;  // super-blocks issued so far (accumulator set gs & 1)
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, it++) {
            const uint32_t gb = it & 1;
            I8_TR(lane == 0 && it < 64, 4000 + 4 * it);
            wait_bar(&g_full[gb], (it >> 1) & 1u);
            I8_TR(lane == 0 && it < 64, 4001 + 4 * it);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t gd = gdesc0 + (uint64_t)(gb * (G_BYTES >> 4));
            for (uint64_t sb = 0; sb < p.nsb; sb++, gs++) {
                const uint32_t ab = (uint32_t)(gs & 1);
                const uint64_t use = gs >> 1;
                I8_TR(lane == 0 && gs < 240, 0 + 4 * gs);
                if (use >= 1) wait_bar(&a_empty[ab], (uint32_t)((use - 1) & 1));
                I8_TR(lane == 0 && gs < 240, 1 + 4 * gs);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const bool last = sb + 1 == p.nsb;
                const int nch = last ? live_last : KCH, nfull = last ? full_last : KCH;
                if (elect_one()) {
                    const uint32_t dset = tmem + ab * ACC_COLS;
#pragma unroll
                    for (int kc = 0; kc < KCH; kc++) {
                        if (kc < nch) {
                            const uint32_t w128 = tmem + COL_W + (kc < nfull ? 0 : 16), w1 = w128 + 8;
#pragma unroll
                            for (int o = 0; o < 2 * NPAIR; o++) {
                                const int comp = o / NPAIR, pr = o % NPAIR;
                                const uint32_t d = dset + (uint32_t)(o * NO);
                                const uint64_t bhi =
                                    gd + (uint64_t)(((comp * NDIG + 2 * pr) * DIG_BYTES + kc * 2 * LBO) >> 4);
                                mma(d, w128, bhi, pr == 0 ? id_s : id_u, kc > 0);
                                mma(d, w1, bhi + (DIG_BYTES >> 4), id_u, 1);
                            }
                        }
                    }
                    commit(&a_full[ab]);
                    if (last) commit(&g_empty[gb]);  // this tile's G is no longer read
                }
                __syncwarp();
                I8_TR(lane == 0 && gs < 240, 2 + 4 * gs);
            }
        }
    } else if (warp >= DRAIN_WARPS) {
        // ------------------------------------------------------------ G builders
        // thread -> item (output n, k-span ks of GSPAN k inside one K-chunk kc = ks*GSPAN / 32)
        const int gt = tid - DRAIN_THREADS;
        uint32_t it = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, it++) {
            const uint32_t gb = it & 1;
            I8_TR(gt == 0 && it < 64, 5000 + 4 * it);
            if (it >= 2) {
                wait_bar(&g_empty[gb], ((it >> 1) - 1) & 1u);  // the MMAs of tile it - 2 are complete
                wait_bar(&c_free[gb], ((it >> 1) - 1) & 1u);   // its drain no longer reads tconst[gb]
            }
            I8_TR(gt == 0 && it < 64, 5001 + 4 * it);
            if (gt < 5 * NO) {
                // per-output constants of the tile, exact sincospi of the integer phase
                const int kind = gt / NO, nn = gt % NO;
                const uint64_t cc = p.c_begin + t * NO + nn;
                const uint64_t a_seed = p.a0 + (p.nsb - 1) * (uint64_t)SBA * p.stride;
                const uint64_t idx = kind == 0 ? (uint64_t)SBA * p.stride * cc
                                   : kind == 1 ? (uint64_t)KC * p.stride * cc
                                   : kind == 2 ? (uint64_t)CHAIN * KC * p.stride * cc
                                   : kind == 3 ? a_seed * cc
                                               : (uint64_t)4 * CHAIN * KC * p.stride * cc;
                double2 v = phase(idx & qmask, q, p.two_over_q);
                if (kind == 0) v.y = -v.y;  // e^{-i phi_SB}: Horner runs forward over super-blocks
                tconst[gb][kind][nn] = v;
            }
            if (gt < G_ITEMS) {
                const int n = gt % NO, ks = gt / NO;  // k-span ks covers k = ks*GSPAN ... + GSPAN - 1
                const int kc = ks * GSPAN / KC;
                const uint64_t c = p.c_begin + t * NO + n;
                // G[k, c] = e^{+2 pi i (kc*4096 + kk) stride c / q}, kk < 32: exact sincospi at
                // kk = 0 and kk = 16, FP64 rotation by e^{+2 pi i stride c / q} in between
                const double2 w = phase((p.stride * c) & qmask, q, p.two_over_q);
                unsigned char *buf = sG + gb * G_BYTES + kmajor<GE::SBO>(n, ks * GSPAN);
#pragma unroll 1
                for (int k16 = 0; k16 < GSPAN / 16; k16++) {
                    const int kk0 = (ks * GSPAN) % KC + 16 * k16;
                    double2 g = phase(((uint64_t)(kc * CHUNK_AMPS + kk0) * p.stride * c) & qmask, q,
                                      p.two_over_q);
#pragma unroll
                    for (int half = 0; half < 2; half++) {
                        // 8 k at a time: 2 components x 8 digits x 8 bytes in registers
                        uint32_t pk[2][NDIG][2];
#pragma unroll
                        for (int e = 0; e < 8; e++) {
#pragma unroll
                            for (int comp = 0; comp < 2; comp++) {
                                // X = rint(G 2^55): the power-of-two scale as an exponent add on the
                                // bit pattern (INT pipe; exact for every normal G, and 0 maps to a
                                // tiny normal that rounds to 0) instead of a DMUL on the busy FP64 pipe
                                const long long X = __double2ll_rn(__longlong_as_double(
                                    __double_as_longlong(comp ? g.y : g.x) + (55LL << 52)));
                                const int d0 = (int)(X >> 49);
                                const unsigned long long R = (unsigned long long)(X - ((long long)d0 << 49));
                                const uint32_t hi28 = (uint32_t)(R >> 21), lo21 = (uint32_t)R & 0x1FFFFFu;
                                const uint32_t dig[NDIG] = {(uint32_t)d0 & 0xFFu, hi28 >> 21, (hi28 >> 14) & 127u,
                                                            (hi28 >> 7) & 127u,   hi28 & 127u, lo21 >> 14,
                                                            (lo21 >> 7) & 127u,   lo21 & 127u};
#pragma unroll
                                for (int dd = 0; dd < NDIG; dd++) {
                                    if ((e & 3) == 0)
                                        pk[comp][dd][e >> 2] = dig[dd];
                                    else
                                        pk[comp][dd][e >> 2] |= dig[dd] << (8 * (e & 3));
                                }
                            }
                            const double nr = fma(g.x, w.x, -g.y * w.y), ni = fma(g.x, w.y, g.y * w.x);
                            g = make_double2(nr, ni);
                        }
#pragma unroll
                        for (int comp = 0; comp < 2; comp++)
#pragma unroll
                            for (int dd = 0; dd < NDIG; dd++)
                                *reinterpret_cast<uint2 *>(buf + (comp * NDIG + dd) * DIG_BYTES + k16 * LBO +
                                                           8 * half) = make_uint2(pk[comp][dd][0], pk[comp][dd][1]);
                    }
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&g_full[gb]);
            I8_TR(gt == 0 && it < 64, 5002 + 4 * it);
        }
    } else {
        // ------------------------------------------------------------ drain + fold
        // thread -> row-block r (TMEM lane) and outputs n0 .. n0 + 7; the Horner
        // state H[r][n] stays in registers across super-blocks and goes to the
        // fold buffer at the tile's end
        const int quarter = warp & 3, n0 = (warp >> 2) * OPT;
        const int r = 32 * quarter + lane;
        const uint32_t lane_addr = (uint32_t)(32 * quarter) << 16;
        uint64_t gs = 0;
        uint32_t itd = 0;
        for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, itd++) {
            const uint32_t gb = itd & 1;
            I8_TR(tid == 0 && itd < 64, 2000 + 4 * itd);
            wait_bar(&g_full[gb], (itd >> 1) & 1u);  // tconst[gb] of this tile (built with its G)
            I8_TR(tid == 0 && itd < 64, 2001 + 4 * itd);
            const double2 *sinv = tconst[gb][0] + n0;
            // the Horner state of (row-block r, outputs n0 ..), kept pre-rotated: after
            // super-block sb it holds H_sb e^{-i phi_SB}, so the next super-block's
            // update H = hreg + T folds into the accumulator combine (a DADD and a
            // DFMA per component after the loads) and the rotation's FP64 latency
            // overlaps the next a_full wait and TMEM loads instead of following them
            // (3 % faster at seed 2 than H = H e^{-i phi_SB} + T after the loads)
            double2 hreg[OPT];
#pragma unroll
            for (int i = 0; i < OPT; i++) hreg[i] = make_double2(0.0, 0.0);
            for (uint64_t sb = 0; sb < p.nsb; sb++, gs++) {
                const uint32_t ab = (uint32_t)(gs & 1);
                I8_TR(tid == 0 && gs < 240, 1000 + 4 * gs);
                wait_bar(&a_full[ab], (uint32_t)((gs >> 1) & 1));
                I8_TR(tid == 0 && gs < 240, 1001 + 4 * gs);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t cols = tmem + lane_addr + ab * ACC_COLS + n0;
                // H in registers; the Re pairs and then the Im pairs (two load round trips)
                int acc[NPAIR][OPT];
                double tre[OPT];
#pragma unroll
                for (int o = 0; o < NPAIR; o++) ld8(cols + o * NO, acc[o]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < OPT; i++) tre[i] = combine_add(acc[0][i], acc[1][i], acc[2][i], acc[3][i], hreg[i].x);
#pragma unroll
                for (int o = 0; o < NPAIR; o++) ld8(cols + (NPAIR + o) * NO, acc[o]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                mbar_arrive(&a_empty[ab]);  // the accumulators are in registers
                I8_TR(tid == 0 && gs < 240, 1002 + 4 * gs);
#pragma unroll
                for (int i = 0; i < OPT; i++) {
                    const double2 hv =
                        make_double2(tre[i], combine_add(acc[0][i], acc[1][i], acc[2][i], acc[3][i], hreg[i].y));
                    hreg[i] = sb + 1 < p.nsb ? rot(hv, sinv[i]) : hv;
                }
            }
            // the tile's MMAs are complete (its last commit was awaited): its G buffer
            // becomes the fold buffer until c_free releases it to the G builders
            double2 *const fold = fold0 + (size_t)gb * (G_BYTES / sizeof(double2));
#pragma unroll
            for (int i = 0; i < OPT; i++) fold[r * FOLD_STRIDE + n0 + i] = hreg[i];
            // fold the 128 row-blocks: V' = sum_r w^r H_r as 16 Horner chains of 8
            // row-blocks, joined four at a time by w^8 and the four results by w^32
            // (a short tree instead of one 16-step chain), in a fixed order
            asm volatile("bar.sync 1, %0;" ::"n"(DRAIN_THREADS) : "memory");
            I8_TR(tid == 0 && itd < 64, 2002 + 4 * itd);
            {
                const int n = tid % NO, ch = tid / NO;
                const double2 w = tconst[gb][1][n];
                const double2 *col = fold + CHAIN * ch * FOLD_STRIDE + n;
                double2 a = col[(CHAIN - 1) * FOLD_STRIDE];
#pragma unroll
                for (int i = CHAIN - 2; i >= 0; i--) a = cmad(a, w, col[i * FOLD_STRIDE]);
                rpart[ch][n] = a;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(DRAIN_THREADS) : "memory");
            if (tid < FOLD_CHAINS / 4 * NO) {
                // 4 chains -> 1 by Horner in w^8
                const int n = tid % NO, g4 = tid / NO;
                const double2 w8 = tconst[gb][2][n];
                double2 v = rpart[4 * g4 + 3][n];
#pragma unroll
                for (int j = 2; j >= 0; j--) v = cmad(v, w8, rpart[4 * g4 + j][n]);
                rquad[g4][n] = v;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(DRAIN_THREADS) : "memory");
            if (tid < NO) {
                const int n = tid;
                const double2 w32 = tconst[gb][4][n], sd = tconst[gb][3][n];
                double2 v = rquad[FOLD_CHAINS / 4 - 1][n];
#pragma unroll
                for (int g4 = FOLD_CHAINS / 4 - 2; g4 >= 0; g4--) v = cmad(v, w32, rquad[g4][n]);
                const double vr = sd.x * v.x - sd.y * v.y, vi = sd.x * v.y + sd.y * v.x;
                const uint64_t ci = t * NO + n;
                if (ci < p.c_count) {
                    // output factor (with 2^-47), |V|^2 as np.abs(.)**2 (hypot, squared)
                    const double o_re = vr * p.out_re - vi * p.out_im;
                    const double o_im = vr * p.out_im + vi * p.out_re;
                    p.out[ci] = make_double2(o_re, o_im);
                    if (p.prob) {
                        const double hh = hypot(o_re, o_im);
                        p.prob[ci] = hh * hh;
                    }
                }
            }
            asm volatile("bar.sync 1, %0;" ::"n"(DRAIN_THREADS) : "memory");
            if (tid == 0) mbar_arrive(&c_free[gb]);  // tconst[gb] may be rebuilt for tile itd + 2
            I8_TR(tid == 0 && itd < 64, 2003 + 4 * itd);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// block sums of |V|^2 in the caller's layout: slot s sums outputs
// [s*slot, (s+1)*slot) in a fixed order (lane-strided, then a fixed shuffle tree)
__global__ void slot_sums_kernel(const double *__restrict__ prob, uint64_t count, uint64_t slot,
                                 double *__restrict__ out, uint64_t nslots)
{
    const uint64_t s = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= nslots) return;
    const uint64_t lo = s * slot, hi = lo + slot < count ? lo + slot : count;
    double acc = 0.0;
    for (uint64_t i = lo + lane; i < hi; i += 32) acc += prob[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) out[s] = acc;
}

}  // namespace i8

#ifdef SHB_I8_TRACE
static unsigned long long *&i8_trace_ptr()
{
    static unsigned long long *p = nullptr;
    return p;
}
#endif

template <int KCH>
static int launch_i8(const i8::Args &a, unsigned grid, cudaStream_t st)
{
    using GE = i8::Geo<KCH>;
    SHB_TRY_CUDA(cudaFuncSetAttribute(i8::dft_i8_uniform_kernel<KCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      GE::SMEM_BYTES));
    i8::dft_i8_uniform_kernel<KCH><<<grid, GE::THREADS, GE::SMEM_BYTES, st>>>(a);
    SHB_LAUNCHED();
    return SHB_OK;
}

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
    a.ntiles = (c_count + NO - 1) / NO;
    // KCH = 8 when it needs fewer super-blocks than KCH = 6: each super-block
    // costs one drain pass (the bound of long supports), each K-chunk of a
    // tile's G one builder item (the bound of short ones) -- profiles/r02_i8_kch_alias.jsonl
    const uint64_t nsb6 = (length + Geo<6>::SBA - 1) / Geo<6>::SBA;
    const uint64_t nsb8 = (length + Geo<8>::SBA - 1) / Geo<8>::SBA;
    const bool k8 = nsb8 < nsb6;
    const uint64_t sba = k8 ? Geo<8>::SBA : Geo<6>::SBA;
    a.nsb = k8 ? nsb8 : nsb6;
    a.last_amps = length - (a.nsb - 1) * sba;
    a.out_re = out_re * T_SCALE;
    a.out_im = out_im * T_SCALE;
    a.out = (double2 *)d_out;
#ifdef SHB_I8_TRACE
    static unsigned long long *trace_buf = nullptr;
    if (!trace_buf) SHB_TRY_CUDA(cudaMalloc(&trace_buf, 8192 * sizeof(unsigned long long)));
    SHB_TRY_CUDA(cudaMemsetAsync(trace_buf, 0, 8192 * sizeof(unsigned long long), st));
    a.trace = trace_buf;
    i8_trace_ptr() = trace_buf;
#endif
    Scratch prob;
    if (!d_prob && d_block_sums) {
        SHB_TRY(scratch_alloc(prob, sizeof(double) * c_count, st));
        d_prob = (double *)prob.ptr;
    }
    a.prob = d_prob;
    const uint64_t grid = a.ntiles < (uint64_t)sm_count() ? a.ntiles : (uint64_t)sm_count();
    SHB_TRY(k8 ? launch_i8<8>(a, (unsigned)grid, st) : launch_i8<6>(a, (unsigned)grid, st));
    if (d_block_sums) {
        const uint64_t nslots = (c_count + slot_outputs - 1) / slot_outputs;
        slot_sums_kernel<<<(unsigned)((nslots + 7) / 8), 256, 0, st>>>(d_prob, c_count, slot_outputs, d_block_sums,
                                                                       nslots);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

}  // namespace shb

#ifdef SHB_I8_TRACE
// exploration builds only: copy the 8192 clock64 stamps of the last launch
extern "C" int shb_i8_trace(unsigned long long *host)
{
    cudaDeviceSynchronize();
    if (!shb::i8_trace_ptr()) return -1;
    return (int)cudaMemcpy(host, shb::i8_trace_ptr(), 8192 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
#endif
