// Stage 3 of the hot path: the QFT as a direct DFT over the collapsed support
// (qft.dense_dft / qft.tiled_dft, qft.py:95-142; inner loop
// _kernels.partial_row_sums, _kernels.py:16-30).
//
//   V_c = scale * sum_j amp_j * e^{+2 pi i (a0 + j*stride) c / q}
//
// Only the support progression a_j = a0 + j*stride is visited, so one
// transform is q*M phase terms (the reference also walks the q-M zeros).
//
// Per output c the phase advances by a constant rotation between successive
// support elements, w_c = e^{-2 pi i stride c / q} (exact integer index ->
// sincospi), so a segment of the sum is a polynomial in w_c evaluated by
// Horner's rule in ascending j:
//
//   acc <- acc * w_c + amp_j          (one complex multiply-add per phase term)
//   segment value = e^{2 pi i a_last c / q} * acc   (exact sincospi re-seed)
//
// Segments are re-seeded every SEG terms (rounding growth <= SEG*eps) and
// tile partials (reference tiles, qft.py:131-141) are added in ascending
// tile order.  Each thread owns K outputs (K independent FMA chains).
//
// Two instantiations, selected from the data by the caller:
//  * generic (UNIF=false): any complex amplitudes.  The amplitude stream is
//    shared by the whole CTA and staged into shared memory by TMA bulk copies
//    (cp.async.bulk + mbarrier ring); inner loop = LDS.128 broadcast + 4 DFMA
//    per output and phase term, with pairs of Horner steps fused as
//    acc*W^2 + (a_j*W + a_{j+1}) so half of the FMAs read broadcast operands.
//  * uniform comb (UNIF=true): every amplitude equals `amp` (the collapsed
//    Shor register).  amp is factored out of the sum, the Horner
//    step becomes acc*w + 1 (3 DFMA + 1 DMUL, the constant from the constant
//    bank), which keeps every FP64 instruction at <= 2 register-file operand
//    reads -- the generic step needs 3 and is register-bandwidth bound.
//
// The epilogue fuses |V|^2 (hypot^2, as np.abs(.)**2, qstate.py:111) and a
// deterministic per-CTA sum of it (norm check, qstate.py:50-53).
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>
#include <vector>

#include "shb_internal.cuh"

namespace shb {

enum : uint32_t { CH_SEG_END = 1u, CH_TILE_END = 2u };

struct ChunkDesc {
    uint64_t j0;
    uint32_t cnt;
    uint32_t flags;
};

#ifndef SHB_DFT_THREADS
#define SHB_DFT_THREADS 256
#endif
#ifndef SHB_DFT_K64
#define SHB_DFT_K64 4
#endif
constexpr int DFT_THREADS = SHB_DFT_THREADS;        // consumer threads (own the outputs)
constexpr int DFT_CONSUMER_WARPS = DFT_THREADS / 32;
constexpr int DFT_PRODUCER_THREADS = 32;            // generic path: one TMA producer warp
constexpr int DFT_STAGES = 4;
constexpr int DFT_CHUNK = 1024;  // amplitudes per stage (16 KB)

template <typename R>
struct Prec;
template <>
struct Prec<double> {
    static constexpr int K = SHB_DFT_K64;  // outputs per thread
    static constexpr uint64_t SEG = 8192;  // terms between exact re-seeds
};
template <>
#ifndef SHB_DFT_K32
#define SHB_DFT_K32 4
#endif
struct Prec<float> {
    static constexpr int K = SHB_DFT_K32;
    static constexpr uint64_t SEG = 256;
};

// e^{+2 pi i idx / q} for an exact integer phase index (idx < q); the index
// is folded to (-q/2, q/2] so sincospi's argument is in (-1, 1] and exact.
__device__ __forceinline__ void phase(uint64_t idx, uint64_t q, double two_over_q, double &c, double &s)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    sincospi((double)sidx * two_over_q, &s, &c);
}

struct DftArgs {
    const double2 *amps;
    const ChunkDesc *sched;
    uint32_t nchunks;
    uint64_t a0, stride, q;
    double two_over_q;
    uint64_t c_begin, c_count;
    double out_re, out_im;  // output factor: scale (generic) or scale*amp (uniform)
    double2 *out;
    double *prob;
    double *block_sums;
};

template <typename R, bool UNIF, bool TILED>
__global__ void __launch_bounds__(UNIF ? DFT_THREADS : DFT_THREADS + DFT_PRODUCER_THREADS,
                                  (UNIF || !TILED) ? 2 : 1)
    dft_kernel(const DftArgs p)
{
    constexpr int K = Prec<R>::K;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    __shared__ __align__(8) uint64_t full_bar[DFT_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[DFT_STAGES];
    __shared__ double red_tmp[DFT_THREADS / 32];

    const int tid = threadIdx.x;
    const uint64_t q = p.q, qmask = q - 1;
    const uint64_t cblk = (uint64_t)blockIdx.x * DFT_THREADS * K;

    // per-output state: step rotation (cos, sin) of phi = 2 pi stride c / q,
    // Horner acc (h), tile partial (t, only when tiles > 1), running total (v)
    constexpr int KT = TILED ? K : 1;
    constexpr int K2 = UNIF ? 1 : K;  // W^2 only on the generic path
    // FP32 path: segment seeds advance by the exact FP64 rotation U = e^{i phi SEG}
    // between full consecutive segments, re-seeded by sincospi every SEED_EXACT
    constexpr bool F32 = sizeof(R) == 4 && UNIF;  // the generic path keeps exact seeds (register budget)
    constexpr int KS = F32 ? K : 1;
    constexpr uint32_t SEED_EXACT = 32;
    double sdr[KS], sdi[KS], ur[KS], ui[KS];
    uint32_t segs_done = 0;
    R wr[K], wi[K], hr[K], hi[K], w2r[K2], w2i[K2];
    double tr[KT], ti[KT], vr[K], vi[K];
    uint64_t cval[K];
#pragma unroll
    for (int i = 0; i < K; i++) {
        cval[i] = p.c_begin + cblk + (uint64_t)i * DFT_THREADS + tid;
        double co, si;
        phase((p.stride * cval[i]) & qmask, q, p.two_over_q, co, si);
        wr[i] = (R)co;
        wi[i] = (R)si;
        if (!UNIF) {
            phase((2 * p.stride * cval[i]) & qmask, q, p.two_over_q, co, si);
            w2r[i % K2] = (R)co;
            w2i[i % K2] = (R)si;
        }
        hr[i] = hi[i] = (R)0;
        vr[i] = vi[i] = 0.0;
        if (F32) {
            phase((Prec<R>::SEG * p.stride * cval[i]) & qmask, q, p.two_over_q, co, si);
            ur[i % KS] = co;
            ui[i % KS] = si;
            sdr[i % KS] = sdi[i % KS] = 0.0;
        }
    }
#pragma unroll
    for (int i = 0; i < KT; i++) tr[i] = ti[i] = 0.0;

    // generic path: warp-specialised pipeline.  The warp after the 8 consumer
    // warps is the TMA producer; full_bar[s] completes when stage s holds its
    // chunk (tx bytes), empty_bar[s] when all consumer warps are done with it,
    // so consumer warps never wait on each other.
    if (!UNIF) {
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < DFT_STAGES; s++) {
                mbar_init(&full_bar[s], 1);
                mbar_init(&empty_bar[s], DFT_CONSUMER_WARPS);
            }
            fence_mbar_init();
        }
        __syncthreads();
        if (tid == DFT_THREADS) {
            for (uint32_t ch = 0; ch < p.nchunks; ch++) {
                const int s = ch % DFT_STAGES;
                if (ch >= DFT_STAGES) mbar_wait(&empty_bar[s], ((ch / DFT_STAGES) - 1) & 1u);
                const ChunkDesc d = p.sched[ch];
                const uint32_t bytes = d.cnt * 16u;
                mbar_arrive_expect_tx(&full_bar[s], bytes);
                tma_bulk_g2s(buf + (size_t)s * DFT_CHUNK, p.amps + d.j0, bytes, &full_bar[s]);
            }
        }
    }
    const bool consumer = UNIF || tid < DFT_THREADS;  // the producer warp owns no outputs

    for (uint32_t ch = 0; consumer && ch < p.nchunks; ch++) {
        const ChunkDesc d = p.sched[ch];
        const int cnt = (int)d.cnt;
        if (UNIF) {
            // acc * conj(e^{i phi}) + 1:
            //   re = acc_re cos + acc_im sin + 1 ; im = acc_im cos - acc_re sin
#pragma unroll 4
            for (int e = 0; e < cnt; e++) {
#pragma unroll
                for (int i = 0; i < K; i++) {
                    const R t_re = fma(hi[i], wi[i], (R)1);
                    const R t_im = hi[i] * wr[i];
                    const R n_re = fma(hr[i], wr[i], t_re);
                    const R n_im = fma(-hr[i], wi[i], t_im);
                    hr[i] = n_re;
                    hi[i] = n_im;
                }
            }
        } else {
            const int s = ch % DFT_STAGES;
            mbar_wait(&full_bar[s], (ch / DFT_STAGES) & 1u);
            const double2 *sb = buf + (size_t)s * DFT_CHUNK;
            // two Horner steps fused: acc'' = acc*W^2 + (a_j*W + a_{j+1}),
            // W = conj(e^{i phi}).  Still 4 FMA per phase term; the
            // b = a_j*W + a_{j+1} half reads two broadcast amplitude operands
            // that the K outputs reuse (2.6 register reads per DFMA overall,
            // vs 3.0 for the plain step -- the path stays register-file bound).
            int e = 0;
#pragma unroll 2
            for (; e + 2 <= cnt; e += 2) {
                const double2 av0 = sb[e], av1 = sb[e + 1];
                const R a0r = (R)av0.x, a0i = (R)av0.y, a1r = (R)av1.x, a1i = (R)av1.y;
#pragma unroll
                for (int i = 0; i < K; i++) {
                    const R b_re = fma(a0r, wr[i], fma(a0i, wi[i], a1r));
                    const R b_im = fma(a0i, wr[i], fma(-a0r, wi[i], a1i));
                    const R n_re = fma(hr[i], w2r[i], fma(hi[i], w2i[i], b_re));
                    const R n_im = fma(hi[i], w2r[i], fma(-hr[i], w2i[i], b_im));
                    hr[i] = n_re;
                    hi[i] = n_im;
                }
            }
            if (e < cnt) {  // odd tail: one plain Horner step
                const double2 av = sb[e];
                const R a_re = (R)av.x, a_im = (R)av.y;
#pragma unroll
                for (int i = 0; i < K; i++) {
                    const R t_re = fma(hi[i], wi[i], a_re);
                    const R t_im = fma(hi[i], wr[i], a_im);
                    const R n_re = fma(hr[i], wr[i], t_re);
                    const R n_im = fma(-hr[i], wi[i], t_im);
                    hr[i] = n_re;
                    hi[i] = n_im;
                }
            }
        }
        if (d.flags & CH_SEG_END) {
            // seed = e^{+2 pi i a_last c / q}; t += seed * acc; acc = 0
            const uint64_t a_last = p.a0 + (d.j0 + d.cnt - 1) * p.stride;
            // a full segment right after another one ends SEG*stride later: its
            // seed is the previous seed times U (FP32 path; FP64 re-seeds exactly)
            const bool exact = !F32 || segs_done % SEED_EXACT == 0 || d.cnt != Prec<R>::SEG;
            segs_done++;
#pragma unroll
            for (int i = 0; i < K; i++) {
                double sc, ss;
                if (exact) {
                    phase((a_last * cval[i]) & qmask, q, p.two_over_q, sc, ss);
                } else {
                    sc = fma(sdr[i % KS], ur[i % KS], -sdi[i % KS] * ui[i % KS]);
                    ss = fma(sdr[i % KS], ui[i % KS], sdi[i % KS] * ur[i % KS]);
                }
                if (F32) {
                    sdr[i % KS] = sc;
                    sdi[i % KS] = ss;
                }
                const double xr = (double)hr[i], xi = (double)hi[i];
                if (TILED) {
                    tr[i % KT] = fma(sc, xr, fma(-ss, xi, tr[i % KT]));
                    ti[i % KT] = fma(sc, xi, fma(ss, xr, ti[i % KT]));
                } else {
                    vr[i] = fma(sc, xr, fma(-ss, xi, vr[i]));
                    vi[i] = fma(sc, xi, fma(ss, xr, vi[i]));
                }
                hr[i] = hi[i] = (R)0;
            }
        }
        if (TILED && (d.flags & CH_TILE_END)) {
#pragma unroll
            for (int i = 0; i < K; i++) {
                vr[i] += tr[i % KT];
                vi[i] += ti[i % KT];
                tr[i % KT] = ti[i % KT] = 0.0;
            }
        }
        if (!UNIF) {
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&empty_bar[ch % DFT_STAGES]);  // warp done with the stage
        }
    }

    // epilogue: output factor (1/sqrt(q), times amp on the uniform path), |V|^2, block sum
    double psum = 0.0;
#pragma unroll
    for (int i = 0; i < K; i++) {
        const uint64_t ci = cblk + (uint64_t)i * DFT_THREADS + tid;
        if (consumer && ci < p.c_count) {
            const double o_re = vr[i] * p.out_re - vi[i] * p.out_im;
            const double o_im = vr[i] * p.out_im + vi[i] * p.out_re;
            p.out[ci] = make_double2(o_re, o_im);
            const double h = hypot(o_re, o_im);
            const double pr = h * h;
            if (p.prob) p.prob[ci] = pr;
            psum += pr;
        }
    }
    if (p.block_sums) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) psum += __shfl_down_sync(0xffffffffu, psum, o);
        if ((tid & 31) == 0 && consumer) red_tmp[tid >> 5] = psum;
        __syncthreads();
        if (tid == 0) {
            double b = 0.0;
#pragma unroll
            for (int w = 0; w < DFT_THREADS / 32; w++) b += red_tmp[w];
            p.block_sums[blockIdx.x] = b;
        }
    }
}

template <typename R, bool UNIF, bool TILED>
static int launch_dft_t(DftArgs a, uint64_t length, uint32_t tiles, cudaStream_t st)
{
    constexpr int K = Prec<R>::K;
    const uint64_t SEG = Prec<R>::SEG;
    const uint64_t q = a.q, a0 = a.a0, stride = a.stride;
    // ---- chunk schedule: tiles -> re-seed segments -> smem chunks
    std::vector<ChunkDesc> sched;
    sched.reserve(length / DFT_CHUNK + tiles + length / SEG + 4);
    const uint64_t tile_span = q / tiles;
    for (uint32_t t = 0; t < tiles && length; t++) {
        const uint64_t lo_a = (uint64_t)t * tile_span, hi_a = lo_a + tile_span;
        auto first_j_at_or_above = [&](uint64_t x) -> uint64_t {
            if (x <= a0) return 0;
            const uint64_t j = (x - a0 + stride - 1) / stride;
            return j < length ? j : length;
        };
        const uint64_t jlo = first_j_at_or_above(lo_a), jhi = first_j_at_or_above(hi_a);
        if (jhi <= jlo) continue;
        for (uint64_t s0 = jlo; s0 < jhi; s0 += SEG) {
            const uint64_t s1 = (s0 + SEG < jhi) ? s0 + SEG : jhi;
            for (uint64_t c0 = s0; c0 < s1; c0 += DFT_CHUNK) {
                const uint64_t c1 = (c0 + DFT_CHUNK < s1) ? c0 + DFT_CHUNK : s1;
                ChunkDesc d{c0, (uint32_t)(c1 - c0), 0u};
                if (c1 == s1) d.flags |= CH_SEG_END;
                if (c1 == s1 && s1 == jhi) d.flags |= CH_TILE_END;
                sched.push_back(d);
            }
        }
    }
    a.nchunks = (uint32_t)sched.size();
    Scratch d_sched;
    SHB_TRY(scratch_alloc(d_sched, sizeof(ChunkDesc) * (a.nchunks ? a.nchunks : 1), st));
    if (a.nchunks)
        SHB_TRY_CUDA(cudaMemcpyAsync(d_sched.ptr, sched.data(), sizeof(ChunkDesc) * a.nchunks,
                                     cudaMemcpyHostToDevice, st));
    a.sched = (const ChunkDesc *)d_sched.ptr;
    const size_t smem = UNIF ? 0 : (size_t)DFT_STAGES * DFT_CHUNK * sizeof(double2);
    if (smem)  // per device and cheap: set on every launch (one process may drive several GPUs)
        SHB_TRY_CUDA(cudaFuncSetAttribute(dft_kernel<R, UNIF, TILED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    const uint64_t per_blk = (uint64_t)DFT_THREADS * K;
    const uint64_t nblk = (a.c_count + per_blk - 1) / per_blk;
    if (nblk > 0x7FFFFFFFull) return set_error(SHB_EINVAL, "too many outputs for one launch");
    const unsigned nthreads = UNIF ? DFT_THREADS : DFT_THREADS + DFT_PRODUCER_THREADS;
    dft_kernel<R, UNIF, TILED><<<(unsigned)nblk, nthreads, smem, st>>>(a);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

template <typename R, bool UNIF>
static int launch_dft(DftArgs a, uint64_t length, uint32_t tiles, cudaStream_t st)
{
    // tile partials only exist for the reference's tiled engine (qft.py:115-142)
    return tiles > 1 ? launch_dft_t<R, UNIF, true>(a, length, tiles, st)
                     : launch_dft_t<R, UNIF, false>(a, length, tiles, st);
}


// ---------------------------------------------------------------------------
// FP64 tensor-core (DMMA) formulation of the same sum.  With j = (jb*8 + j1)*B + k
// (B = MMA_B, j1 < 8, k < B):
//   sum_j a_j w^j = sum_jb w^{8B jb} sum_j1 w^{B j1} T_jb[j1, c],
//   T_jb[j1, c] = sum_k a_{(jb*8+j1)*B+k} * w_c^k
// T_jb is an [8 x B] x [B x 8] GEMM per 8 outputs: mma.sync m8n8k4 f64, four
// real DMMAs per complex product (8 flops per phase term, as the vector
// kernels).  A = amplitudes (row j1, col k), B = G[k][c] = w_c^k (exact,
// sincospi), D[j1][c] = T.  Each lane keeps a Horner over blocks for its two
// D columns (U = w^{-8B}); every MMA_SEG_BLOCKS blocks the lane's partial is
// multiplied by the exact seed e^{i theta(a0 + (8B jb_last + B j1) stride, c)}
// and added to its total; one cross-lane reduction at the end.
// m8n8k4.f64 fragments: A[r = lane/4][k = lane%4], B[k = lane%4][n = lane/4],
// C/D[r = lane/4][n = 2*(lane%4) + {0,1}].
#ifndef SHB_MMA_B
#define SHB_MMA_B 64    // generic amplitude stream (register cap 168 with the producer warp)
#endif
#ifndef SHB_MMA_BU
#define SHB_MMA_BU 128  // uniform comb (no amplitude registers: G takes 128 of them)
#endif
#ifndef SHB_MMA_CT
#define SHB_MMA_CT 1
#endif
constexpr int MMA_CT = SHB_MMA_CT;  // 8-output tiles per warp
// CTA shapes (measured, scripts/build_mma_real_variants.sh): the uniform path
// (254 registers) runs one CTA of 8 warps per SM; the amplitude-stream path
// (168-register cap with its producer warp) runs two CTAs of 4 consumer warps
// (+7 % on real amplitudes against one CTA of 8).
#ifndef SHB_MMA_WARPS_U
#define SHB_MMA_WARPS_U 8
#endif
#ifndef SHB_MMA_WARPS_G
#define SHB_MMA_WARPS_G 4
#endif
#ifndef SHB_MMA_MINB_U
#define SHB_MMA_MINB_U 1
#endif
#ifndef SHB_MMA_MINB_G
#define SHB_MMA_MINB_G 2
#endif
template <bool UNIF>
struct MmaShape {
    static constexpr int WARPS = UNIF ? SHB_MMA_WARPS_U : SHB_MMA_WARPS_G;  // consumer warps
    static constexpr int MINB = UNIF ? SHB_MMA_MINB_U : SHB_MMA_MINB_G;
    static constexpr int THREADS = UNIF ? WARPS * 32 : WARPS * 32 + 32;    // + TMA producer warp
    static constexpr int OUT_PER_CTA = WARPS * MMA_CT * 8;
};
#ifndef SHB_MMA_NACC
#define SHB_MMA_NACC 1  // accumulator sets by k-step parity (real form)
#endif
#ifndef SHB_MMA_PIPE
#define SHB_MMA_PIPE 0  // 2-set software pipeline over blocks (amplitude-stream path)
#endif
#ifndef SHB_MMA_PIPE_U
#define SHB_MMA_PIPE_U 1  // ... on the uniform path (+1.5 % at B = 128, scripts/build_mma_real_variants.sh)
#endif
#ifndef SHB_MMA_GREC
#define SHB_MMA_GREC 1  // G fragments by recurrence from 2 exact phases
#endif
#ifndef SHB_MMA_SEG
#define SHB_MMA_SEG 32768  // amplitudes between exact per-lane re-seeds
#endif
constexpr int MMA_CHUNK = 1024;            // amplitudes per smem stage (generic path)

// volatile: on the uniform comb every block's T is the same product, and a
// non-volatile asm would let the compiler hoist it out of the block loop --
// the kernel must perform every phase term it is credited with.  Callers
// order the DMMAs so that independent ones separate dependent pairs.
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

struct MmaArgs {
    const double2 *amps;  // null on the uniform path
    uint64_t length;       // progression length (amplitudes)
    uint64_t a0, stride, q;
    double two_over_q;
    uint64_t c_begin, c_count;
    double amp_re, amp_im;  // uniform amplitude (uniform path)
    double out_re, out_im;  // output factor
    double2 *out;
    double *prob;
    double *block_sums;
};

// REALA: every amplitude is real (always so on the uniform path, where the
// amplitude is factored out and A = 1).  A real A times the complex G is two
// real GEMMs (Re T = A Gr, Im T = A Gi): 2 DMMAs per k-step instead of 4, i.e.
// 4 flops per phase term -- the multiplies by Im A = 0 are not issued.  The two
// DMMA chains alternate between two accumulator sets by k-step parity so that
// dependent DMMAs on one accumulator are 4 instructions apart.
template <bool UNIF, bool REALA>
__global__ void __launch_bounds__(MmaShape<UNIF>::THREADS, MmaShape<UNIF>::MINB)
    dft_mma_kernel(const MmaArgs p)
{
    constexpr int MMA_WARPS = MmaShape<UNIF>::WARPS;
    constexpr int MMA_OUT_PER_CTA = MmaShape<UNIF>::OUT_PER_CTA;
    constexpr int MMA_B = UNIF ? SHB_MMA_BU : SHB_MMA_B;  // k extent per block row
    constexpr int MMA_KS = MMA_B / 4;                      // k-steps of 4
    constexpr int MMA_BLOCK = 8 * MMA_B;                   // amplitudes per block
    constexpr int MMA_SEG_BLOCKS = SHB_MMA_SEG / MMA_BLOCK > 0 ? SHB_MMA_SEG / MMA_BLOCK : 1;
    constexpr int BPC = MMA_CHUNK / MMA_BLOCK > 0 ? MMA_CHUNK / MMA_BLOCK : 1;  // blocks per smem stage
    static_assert(UNIF || MMA_CHUNK % MMA_BLOCK == 0, "smem stages must hold whole blocks");
    constexpr int NACC = REALA ? SHB_MMA_NACC : 1;
    constexpr int NP = (UNIF ? SHB_MMA_PIPE_U : SHB_MMA_PIPE) ? 2 : 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    __shared__ __align__(8) uint64_t full_bar[DFT_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[DFT_STAGES];
    __shared__ double red_tmp[MMA_WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t q = p.q, qmask = q - 1;
    const uint64_t nblocks = (p.length + MMA_BLOCK - 1) / MMA_BLOCK;
    const uint64_t nchunks = (p.length + MMA_CHUNK - 1) / MMA_CHUNK;
    const uint64_t cta_c = (uint64_t)blockIdx.x * MMA_OUT_PER_CTA;
    const bool consumer = UNIF || warp < MMA_WARPS;

    if (!UNIF) {
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < DFT_STAGES; s++) {
                mbar_init(&full_bar[s], 1);
                mbar_init(&empty_bar[s], MMA_WARPS);
            }
            fence_mbar_init();
        }
        __syncthreads();
        if (tid == MMA_WARPS * 32) {  // TMA producer
            for (uint64_t ch = 0; ch < nchunks; ch++) {
                const int s = (int)(ch % DFT_STAGES);
                if (ch >= DFT_STAGES) mbar_wait(&empty_bar[s], (uint32_t)((ch / DFT_STAGES) - 1) & 1u);
                const uint64_t j0 = ch * MMA_CHUNK;
                const uint64_t cnt = (p.length - j0) < MMA_CHUNK ? (p.length - j0) : MMA_CHUNK;
                mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(cnt * 16));
                tma_bulk_g2s(buf + (size_t)s * MMA_CHUNK, p.amps + j0, (uint32_t)(cnt * 16), &full_bar[s]);
            }
        }
    }

    // this lane's outputs: B-fragment column (G) and D-fragment columns
    const int r = lane >> 2, kq = lane & 3;
    uint64_t cG[MMA_CT], cD[MMA_CT][2];
    double gr[MMA_CT][MMA_KS], gi[MMA_CT][MMA_KS];
    double ur[MMA_CT][2], ui[MMA_CT][2];       // U = w^{-8B} for the D columns
    double hr[MMA_CT][2], hi[MMA_CT][2];       // per-lane Horner over blocks (this segment)
    double vr[MMA_CT][2], vi[MMA_CT][2];       // per-lane totals
    double dr[NP][NACC][MMA_CT][2], di[NP][NACC][MMA_CT][2];  // MMA accumulators (Re T, Im T)
#pragma unroll
    for (int ct = 0; ct < MMA_CT; ct++) {
        const uint64_t tile = cta_c + (uint64_t)warp * (MMA_CT * 8) + ct * 8;
        cG[ct] = p.c_begin + tile + r;
        if (SHB_MMA_GREC) {
            // G[ks] = w^{4 ks + kq}: two exact sincospi and 15 complex products
            // (<= ~15 ulp; the same G serves every block of the transform)
            double sr, si4;
            phase((4 * p.stride * cG[ct]) & qmask, q, p.two_over_q, sr, si4);
            phase(((uint64_t)kq * p.stride * cG[ct]) & qmask, q, p.two_over_q, gr[ct][0], gi[ct][0]);
#pragma unroll
            for (int ks = 1; ks < MMA_KS; ks++) {
                gr[ct][ks] = fma(gr[ct][ks - 1], sr, -gi[ct][ks - 1] * si4);
                gi[ct][ks] = fma(gr[ct][ks - 1], si4, gi[ct][ks - 1] * sr);
            }
        } else {
#pragma unroll
            for (int ks = 0; ks < MMA_KS; ks++) {
                const uint64_t k = (uint64_t)ks * 4 + kq;
                double co, si;
                phase((k * p.stride * cG[ct]) & qmask, q, p.two_over_q, co, si);
                gr[ct][ks] = co;
                gi[ct][ks] = si;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            cD[ct][h] = p.c_begin + tile + 2 * kq + h;
            double co, si;
            phase(((uint64_t)MMA_BLOCK * p.stride * cD[ct][h]) & qmask, q, p.two_over_q, co, si);
            ur[ct][h] = co;
            ui[ct][h] = -si;  // w^{-8B}
            hr[ct][h] = hi[ct][h] = vr[ct][h] = vi[ct][h] = 0.0;
#pragma unroll
            for (int s = 0; s < NP * NACC; s++) dr[s / NACC][s % NACC][ct][h] = di[s / NACC][s % NACC][ct][h] = 0.0;
        }
    }

    const double amp_r = p.amp_re, amp_i = p.amp_im;
    // Software pipeline over blocks (NP = 2 accumulator sets): iteration jb
    // issues block jb's DMMAs into set jb&1, then folds block jb-1 from the
    // other set, so the fold (which waits on the last DMMA of its block) sits
    // behind a block of independent DMMAs instead of draining the tensor pipe.
    // Warps of a CTA run in lockstep, so without this every warp drained at
    // the same time (ncu: DADD of the fold = 21% of stall samples).
    for (uint64_t i = 0; consumer && i <= nblocks; i += NP) {
#pragma unroll
        for (int P = 0; P < NP; P++) {
            const uint64_t jb = i + P;
            if (jb < nblocks) {
                const uint64_t ch = jb / BPC;
                const int s = (int)(ch % DFT_STAGES);
                const int boff = (int)(jb % BPC) * MMA_BLOCK;
                if (!UNIF && boff == 0) mbar_wait(&full_bar[s], (uint32_t)(ch / DFT_STAGES) & 1u);
                const double2 *sb = buf + (size_t)s * MMA_CHUNK + boff;
                const uint64_t jblk = jb * MMA_BLOCK;
                // T = A * G (complex): Re += ar*gr - ai*gi ; Im += ar*gi + ai*gr, issued
                // so that independent DMMAs separate the updates of each accumulator
                auto mma_step = [&](int ks, double ar, double ai) {
                    if (REALA) {
                        const int sa = ks % NACC;
#pragma unroll
                        for (int ct = 0; ct < MMA_CT; ct++) {
                            dmma_8x8x4(dr[P][sa][ct][0], dr[P][sa][ct][1], ar, gr[ct][ks]);
                            dmma_8x8x4(di[P][sa][ct][0], di[P][sa][ct][1], ar, gi[ct][ks]);
                        }
                        return;
                    }
#pragma unroll
                    for (int ct = 0; ct < MMA_CT; ct++) {
                        dmma_8x8x4(dr[P][0][ct][0], dr[P][0][ct][1], ar, gr[ct][ks]);
                        dmma_8x8x4(di[P][0][ct][0], di[P][0][ct][1], ar, gi[ct][ks]);
                    }
#pragma unroll
                    for (int ct = 0; ct < MMA_CT; ct++) {
                        dmma_8x8x4(dr[P][0][ct][0], dr[P][0][ct][1], -ai, gi[ct][ks]);
                        dmma_8x8x4(di[P][0][ct][0], di[P][0][ct][1], ai, gr[ct][ks]);
                    }
                };
                // A fragment: row j1 = r, col k of the block.  Only the last block can
                // be ragged; full blocks take the operands without a bounds select (a
                // per-step select rewrites the A register the previous DMMAs read).
                if (jblk + MMA_BLOCK <= p.length) {
#pragma unroll
                    for (int ks = 0; ks < MMA_KS; ks++) {
                        if (UNIF) {
                            mma_step(ks, amp_r, amp_i);
                        } else if (REALA) {
                            mma_step(ks, sb[r * MMA_B + ks * 4 + kq].x, 0.0);
                        } else {
                            const double2 av = sb[r * MMA_B + ks * 4 + kq];
                            mma_step(ks, av.x, av.y);
                        }
                    }
                } else {
#pragma unroll
                    for (int ks = 0; ks < MMA_KS; ks++) {
                        const int jl = r * MMA_B + ks * 4 + kq;
                        double ar = 0.0, ai = 0.0;  // ragged tail: zero rows
                        if (jblk + jl < p.length) {
                            if (UNIF) {
                                ar = amp_r;
                                ai = amp_i;
                            } else {
                                const double2 av = sb[jl];
                                ar = av.x;
                                ai = av.y;
                            }
                        }
                        mma_step(ks, ar, ai);
                    }
                }
                if (!UNIF && (boff + MMA_BLOCK == MMA_CHUNK || jb + 1 == nblocks)) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[s]);
                }
            }
            // fold block jf = jb - (NP - 1) from set Q
            const int Q = (P + 1) % NP;  // constant after unrolling
            if (jb + 1 >= (uint64_t)NP && jb + 1 - NP < nblocks) {
                const uint64_t jf = jb + 1 - NP;
                // Horner over blocks: h = h * w^{-8B} + T ; T reset
#pragma unroll
                for (int ct = 0; ct < MMA_CT; ct++)
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        const double tr_ = NACC > 1 ? dr[Q][0][ct][h] + dr[Q][NACC - 1][ct][h] : dr[Q][0][ct][h];
                        const double ti_ = NACC > 1 ? di[Q][0][ct][h] + di[Q][NACC - 1][ct][h] : di[Q][0][ct][h];
                        const double nr = fma(hr[ct][h], ur[ct][h], fma(-hi[ct][h], ui[ct][h], tr_));
                        const double ni = fma(hr[ct][h], ui[ct][h], fma(hi[ct][h], ur[ct][h], ti_));
                        hr[ct][h] = nr;
                        hi[ct][h] = ni;
#pragma unroll
                        for (int s2 = 0; s2 < NACC; s2++) dr[Q][s2][ct][h] = di[Q][s2][ct][h] = 0.0;
                    }
                if ((jf + 1) % MMA_SEG_BLOCKS == 0 || jf + 1 == nblocks) {
                    // exact seed of this lane's last row: a0 + (8B jf + B r) * stride
                    const uint64_t a_lane = p.a0 + (jf * MMA_BLOCK + (uint64_t)r * MMA_B) * p.stride;
#pragma unroll
                    for (int ct = 0; ct < MMA_CT; ct++)
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            double sc, ss;
                            phase((a_lane * cD[ct][h]) & qmask, q, p.two_over_q, sc, ss);
                            vr[ct][h] = fma(sc, hr[ct][h], fma(-ss, hi[ct][h], vr[ct][h]));
                            vi[ct][h] = fma(sc, hi[ct][h], fma(ss, hr[ct][h], vi[ct][h]));
                            hr[ct][h] = hi[ct][h] = 0.0;
                        }
                }
            }
        }
    }

    // cross-lane sum over the 8 rows (lanes with equal lane%4), then lanes 0..3 write
    double psum = 0.0;
    if (consumer) {
#pragma unroll
        for (int ct = 0; ct < MMA_CT; ct++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    vr[ct][h] += __shfl_xor_sync(0xffffffffu, vr[ct][h], o);
                    vi[ct][h] += __shfl_xor_sync(0xffffffffu, vi[ct][h], o);
                }
                const uint64_t ci = cD[ct][h] - p.c_begin;
                if (r == 0 && ci < p.c_count) {
                    const double o_re = vr[ct][h] * p.out_re - vi[ct][h] * p.out_im;
                    const double o_im = vr[ct][h] * p.out_im + vi[ct][h] * p.out_re;
                    p.out[ci] = make_double2(o_re, o_im);
                    const double hh = hypot(o_re, o_im);
                    const double pr = hh * hh;
                    if (p.prob) p.prob[ci] = pr;
                    psum += pr;
                }
            }
    }
    if (p.block_sums) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) psum += __shfl_down_sync(0xffffffffu, psum, o);
        if (lane == 0 && consumer) red_tmp[warp] = psum;
        __syncthreads();
        if (tid == 0) {
            double b = 0.0;
#pragma unroll
            for (int w = 0; w < MMA_WARPS; w++) b += red_tmp[w];
            p.block_sums[blockIdx.x] = b;
        }
    }
}

// ---------------------------------------------------------------------------
// FP32 fast path on the BF16 tensor cores (precision = SHB_FP32, uniform comb,
// tiles == 1).  Same GEMM factorisation as the DMMA engine with 16-row blocks:
// j = (jb*16 + j1)*TC_BK + k,
//   T_jb[j1, c] = sum_k 1 * G[k, c],  G[k, c] = e^{+2 pi i k stride c / q}
// as mma.sync m16n8k16 bf16 -> f32 with A = 1 (the uniform amplitude is
// factored out of the sum, exact in bf16) and G split into two bf16 terms,
// G = G_hi + G_lo (|G - G_hi - G_lo| <= 2^-18 |G|): 4 MMAs per k-step (Re/Im x
// hi/lo), FP32 accumulation.  Per lane the blocks are folded by an FP32 Horner
// (U = w^{-16 TC_BK}); every TC_SEG_BLOCKS blocks the FP32 partial is rotated
// by the exact-index seed (sincospif of the exact integer phase index) and
// added to an FP64 total.  Error budget (<= 1e-4 relative on |V|^2, SPEC
// north star): G split 2^-18, FP32 Horner over <= 16 steps, FP32 seeds
// ~2e-7 -- measured max|dp|/max p in tests/bench.
#ifndef SHB_TC_BK
#define SHB_TC_BK 64
#endif
#ifndef SHB_TC_SEG
#define SHB_TC_SEG 32768
#endif
constexpr int TC_BK = SHB_TC_BK;          // k extent per block row
constexpr int TC_KS = TC_BK / 16;         // k-steps of 16
constexpr int TC_BLOCK = 16 * TC_BK;      // amplitudes per block
constexpr int TC_SEG_BLOCKS = SHB_TC_SEG / TC_BLOCK > 0 ? SHB_TC_SEG / TC_BLOCK : 1;
constexpr int TC_WARPS = 8;
constexpr int TC_OUT_PER_CTA = TC_WARPS * 8;  // 64

__device__ __forceinline__ void hmma_bf16_16816(float (&d)[4], uint32_t a, uint32_t b0, uint32_t b1)
{
    // A = all ones (every A register holds the same bf16x2 pair)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%6}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a), "r"(b0), "r"(b1));
}

// e^{+2 pi i idx / q} in FP32 from the exact integer index (folded to (-q/2, q/2])
__device__ __forceinline__ void phase_f32(uint64_t idx, uint64_t q, double two_over_q, float &c, float &s)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    sincospif((float)((double)sidx * two_over_q), &s, &c);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo_elem, float hi_elem)
{
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);  // .x -> low 16 bits
    return *reinterpret_cast<const uint32_t *>(&v);
}

#ifndef SHB_TC_MINB
#define SHB_TC_MINB 2
#endif
__global__ void __launch_bounds__(TC_WARPS * 32, SHB_TC_MINB) dft_tc32_uniform_kernel(const MmaArgs p)
{
    __shared__ double red_tmp[TC_WARPS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t q = p.q, qmask = q - 1;
    const uint64_t nblocks = (p.length + TC_BLOCK - 1) / TC_BLOCK;
    const uint64_t tile = (uint64_t)blockIdx.x * TC_OUT_PER_CTA + (uint64_t)warp * 8;
    const int g = lane >> 2, t4 = lane & 3;
    // B fragment (16 x 8, col): lane holds k = 2 t4 + {0,1} and 2 t4 + 8 + {0,1}, column n = g
    const uint64_t cB = p.c_begin + tile + g;
    uint32_t brh[TC_KS][2], brl[TC_KS][2], bih[TC_KS][2], bil[TC_KS][2];
#pragma unroll
    for (int ks = 0; ks < TC_KS; ks++)
#pragma unroll
        for (int hlf = 0; hlf < 2; hlf++) {
            float gr[2], gi[2], grl[2], gil[2];
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const uint64_t k = (uint64_t)ks * 16 + hlf * 8 + 2 * t4 + e;
                phase_f32((k * p.stride * cB) & qmask, q, p.two_over_q, gr[e], gi[e]);
                grl[e] = gr[e] - __bfloat162float(__float2bfloat16_rn(gr[e]));
                gil[e] = gi[e] - __bfloat162float(__float2bfloat16_rn(gi[e]));
            }
            brh[ks][hlf] = pack_bf16x2(gr[0], gr[1]);
            bih[ks][hlf] = pack_bf16x2(gi[0], gi[1]);
            brl[ks][hlf] = pack_bf16x2(grl[0], grl[1]);
            bil[ks][hlf] = pack_bf16x2(gil[0], gil[1]);
        }
    // D fragment (16 x 8): rows g, g+8; columns 2 t4 + {0,1}.  Per (row, col):
    // FP32 Horner h over blocks, FP64 total v.
    uint64_t cD[2];
    float ur[2], ui[2];
    float hr[2][2], hi[2][2];  // [row half][col]
    double vr[2], vi[2];       // [col] (rows merged after seeding)
#pragma unroll
    for (int e = 0; e < 2; e++) {
        cD[e] = p.c_begin + tile + 2 * t4 + e;
        float co, si;
        phase_f32(((uint64_t)TC_BLOCK * p.stride * cD[e]) & qmask, q, p.two_over_q, co, si);
        ur[e] = co;
        ui[e] = -si;  // w^{-TC_BLOCK}
        vr[e] = vi[e] = 0.0;
        hr[0][e] = hr[1][e] = hi[0][e] = hi[1][e] = 0.f;
    }
    const uint32_t ones = 0x3F803F80u;  // bf16x2 (1, 1)
    for (uint64_t jb = 0; jb < nblocks; jb++) {
        float dr[4] = {0.f, 0.f, 0.f, 0.f}, di[4] = {0.f, 0.f, 0.f, 0.f};
        float drl[4] = {0.f, 0.f, 0.f, 0.f}, dil[4] = {0.f, 0.f, 0.f, 0.f};
        const uint64_t jblk = jb * TC_BLOCK;
        if (jblk + TC_BLOCK <= p.length) {
#pragma unroll
            for (int ks = 0; ks < TC_KS; ks++) {
                hmma_bf16_16816(dr, ones, brh[ks][0], brh[ks][1]);
                hmma_bf16_16816(di, ones, bih[ks][0], bih[ks][1]);
                hmma_bf16_16816(drl, ones, brl[ks][0], brl[ks][1]);
                hmma_bf16_16816(dil, ones, bil[ks][0], bil[ks][1]);
            }
        } else {
            // ragged last block: rows j1 whose k range leaves the progression
            // take A = 0 (per row half) -- A rows are g (a0, a2 regs) and g+8
            // (a1, a3); a k-step column range is 16 wide, so mask per element
#pragma unroll
            for (int ks = 0; ks < TC_KS; ks++) {
                // A fragment elements: row g / g+8, k = ks*16 + 2 t4 + {0,1} (+8)
                uint32_t a[4];
#pragma unroll
                for (int rr = 0; rr < 2; rr++)
#pragma unroll
                    for (int hlf = 0; hlf < 2; hlf++) {
                        const uint64_t row = (uint64_t)g + 8 * rr;
                        const uint64_t j0 = jblk + row * TC_BK + (uint64_t)ks * 16 + hlf * 8 + 2 * t4;
                        const float e0 = j0 < p.length ? 1.f : 0.f, e1 = j0 + 1 < p.length ? 1.f : 0.f;
                        a[hlf * 2 + rr] = pack_bf16x2(e0, e1);
                    }
                auto mma4 = [&](float (&d)[4], uint32_t b0, uint32_t b1) {
                    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, "
                                 "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
                };
                mma4(dr, brh[ks][0], brh[ks][1]);
                mma4(di, bih[ks][0], bih[ks][1]);
                mma4(drl, brl[ks][0], brl[ks][1]);
                mma4(dil, bil[ks][0], bil[ks][1]);
            }
        }
        // FP32 Horner over blocks: h = h * U + T   (T = hi + lo products)
#pragma unroll
        for (int rr = 0; rr < 2; rr++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float tr_ = dr[rr * 2 + e] + drl[rr * 2 + e];
                const float ti_ = di[rr * 2 + e] + dil[rr * 2 + e];
                const float nr = fmaf(hr[rr][e], ur[e], fmaf(-hi[rr][e], ui[e], tr_));
                const float ni = fmaf(hr[rr][e], ui[e], fmaf(hi[rr][e], ur[e], ti_));
                hr[rr][e] = nr;
                hi[rr][e] = ni;
            }
        if ((jb + 1) % TC_SEG_BLOCKS == 0 || jb + 1 == nblocks) {
            // seed of row j1's last block: a0 + (TC_BLOCK jb + TC_BK j1) * stride
#pragma unroll
            for (int rr = 0; rr < 2; rr++) {
                const uint64_t a_row = p.a0 + (jb * TC_BLOCK + (uint64_t)(g + 8 * rr) * TC_BK) * p.stride;
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    float sc, ss;
                    phase_f32((a_row * cD[e]) & qmask, q, p.two_over_q, sc, ss);
                    const double xr = hr[rr][e], xi = hi[rr][e];
                    vr[e] = fma((double)sc, xr, fma(-(double)ss, xi, vr[e]));
                    vi[e] = fma((double)sc, xi, fma((double)ss, xr, vi[e]));
                    hr[rr][e] = hi[rr][e] = 0.f;
                }
            }
        }
    }
    // sum over the 16 rows: lanes with equal t4 (xor 4, 8, 16); lanes 0..3 write
    double psum = 0.0;
#pragma unroll
    for (int e = 0; e < 2; e++) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            vr[e] += __shfl_xor_sync(0xffffffffu, vr[e], o);
            vi[e] += __shfl_xor_sync(0xffffffffu, vi[e], o);
        }
        const uint64_t ci = cD[e] - p.c_begin;
        if (g == 0 && ci < p.c_count) {
            const double o_re = vr[e] * p.out_re - vi[e] * p.out_im;
            const double o_im = vr[e] * p.out_im + vi[e] * p.out_re;
            p.out[ci] = make_double2(o_re, o_im);
            const double hh = hypot(o_re, o_im);
            const double pr = hh * hh;
            if (p.prob) p.prob[ci] = pr;
            psum += pr;
        }
    }
    if (p.block_sums) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) psum += __shfl_down_sync(0xffffffffu, psum, o);
        if (lane == 0) red_tmp[warp] = psum;
        __syncthreads();
        if (tid == 0) {
            double b = 0.0;
#pragma unroll
            for (int w = 0; w < TC_WARPS; w++) b += red_tmp[w];
            p.block_sums[blockIdx.x] = b;
        }
    }
}

// Fold MMA per-CTA |V|^2 sums (128 outputs each) into the vector-kernel layout
// the caller allocated (shb_dft_num_blocks: DFT_THREADS*K outputs per slot), in
// a fixed order so the norm stays deterministic.
__global__ void group_sums_kernel(const double *__restrict__ part, uint64_t nparts, int group,
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

template <bool UNIF, bool REALA>
static int launch_dft_mma(MmaArgs a, cudaStream_t st)
{
    const size_t smem = UNIF ? 0 : (size_t)DFT_STAGES * MMA_CHUNK * sizeof(double2);
    if (smem)
        SHB_TRY_CUDA(cudaFuncSetAttribute(dft_mma_kernel<UNIF, REALA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    constexpr int MMA_OUT_PER_CTA = MmaShape<UNIF>::OUT_PER_CTA;
    const uint64_t nblk = (a.c_count + MMA_OUT_PER_CTA - 1) / MMA_OUT_PER_CTA;
    if (nblk > 0x7FFFFFFFull) return set_error(SHB_EINVAL, "too many outputs for one launch");
    const unsigned nthreads = MmaShape<UNIF>::THREADS;
    double *caller_sums = a.block_sums;
    Scratch part;
    if (caller_sums) {
        SHB_TRY(scratch_alloc(part, sizeof(double) * nblk, st));
        a.block_sums = (double *)part.ptr;
    }
    dft_mma_kernel<UNIF, REALA><<<(unsigned)nblk, nthreads, smem, st>>>(a);
    SHB_LAUNCHED();
    if (caller_sums) {
        constexpr int group = DFT_THREADS * Prec<double>::K / MMA_OUT_PER_CTA;
        static_assert(group * MMA_OUT_PER_CTA == DFT_THREADS * Prec<double>::K, "slot sizes must nest");
        const uint64_t nout = (a.c_count + DFT_THREADS * Prec<double>::K - 1) / (DFT_THREADS * Prec<double>::K);
        group_sums_kernel<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>((const double *)part.ptr, nblk, group,
                                                                          caller_sums, nout);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

static int launch_dft_tc32_uniform(MmaArgs a, cudaStream_t st)
{
    const uint64_t nblk = (a.c_count + TC_OUT_PER_CTA - 1) / TC_OUT_PER_CTA;
    if (nblk > 0x7FFFFFFFull) return set_error(SHB_EINVAL, "too many outputs for one launch");
    double *caller_sums = a.block_sums;
    Scratch part;
    if (caller_sums) {
        SHB_TRY(scratch_alloc(part, sizeof(double) * nblk, st));
        a.block_sums = (double *)part.ptr;
    }
    dft_tc32_uniform_kernel<<<(unsigned)nblk, TC_WARPS * 32, 0, st>>>(a);
    SHB_LAUNCHED();
    if (caller_sums) {
        // caller layout: shb_dft_num_blocks(c_count, SHB_FP32) slots of DFT_THREADS*K outputs
        constexpr int group = DFT_THREADS * Prec<float>::K / TC_OUT_PER_CTA;
        static_assert(group * TC_OUT_PER_CTA == DFT_THREADS * Prec<float>::K, "slot sizes must nest");
        const uint64_t nout = (a.c_count + DFT_THREADS * Prec<float>::K - 1) / (DFT_THREADS * Prec<float>::K);
        group_sums_kernel<<<(unsigned)((nout + 255) / 256), 256, 0, st>>>((const double *)part.ptr, nblk, group,
                                                                          caller_sums, nout);
        SHB_LAUNCHED();
    }
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

// FP32 fast path for the uniform comb (tiles == 1): the BF16 tensor-core
// forms.  Default: the tcgen05/TMEM kernel (dft_tc05.cu; 1.3-1.8e14 phase
// terms/s, scripts/tc05_check.py); SHB_FP32_ENGINE=mma selects the warp-level
// mma.sync form (4e13), =vector the FP32 Horner kernel (7e12).
enum Fp32Engine { F32_VECTOR, F32_MMA, F32_TC05 };
static Fp32Engine fp32_engine()
{
    const char *e = getenv("SHB_FP32_ENGINE");
    if (e && e[0] == 'v') return F32_VECTOR;
    if (e && e[0] == 'm') return F32_MMA;
    return F32_TC05;
}
static bool use_tc32_engine() { return fp32_engine() != F32_VECTOR; }

// Engine choice for FP64, tiles == 1 (measured, profiles/r01_mma_real.jsonl):
// * uniform comb: the int8 tensor-core engine (use_i8_engine, below);
// * real amplitudes (and the uniform comb under SHB_DFT_ENGINE=mma): the real-A DMMA form, 2 real products
//   per phase term (7.7-8.0e12 terms/s at q = 2^24 and 2^30, vs 4.3e12 for the
//   vector Horner kernel, whose complex recurrence needs 4 FP64 ops per term
//   whatever the amplitudes);
// * complex amplitudes: the complex DMMA form (30 vs 26 TF at q = 2^24; the
//   vector form is register-file bound there).
// The vector kernel serves tiles > 1 and FP32.  SHB_DFT_ENGINE=vector|mma
// overrides (tests run both).  The choice does not depend on this launch's
// output range, so every output shard of a transform uses the same kernel and
// the spectrum stays bitwise identical for any number of ranks.
static bool use_mma_engine(bool uniform, uint64_t q)
{
    (void)uniform;
    (void)q;
    const char *e = getenv("SHB_DFT_ENGINE");
    if (e && e[0]) return e[0] == 'm' || e[0] == 'i';  // i8 serves the uniform comb only
    return true;
}

// Uniform comb, FP64: the int8 tensor-core engine (dft_i8.cu) by default --
// exact integer products of an 8-digit split of G*2^55 with FP64 folds, ~2e-15
// of max|V| against the long-double closed form (tests/test_gpu_baseline_configs.py).
// SHB_DFT_ENGINE=mma|vector selects the FP64-pipe kernels.
static bool use_i8_engine()
{
    const char *e = getenv("SHB_DFT_ENGINE");
    return !(e && e[0]) || e[0] == 'i';
}

static bool use_real_form()
{
    const char *rf = getenv("SHB_MMA_REAL");
    return !(rf && rf[0] == '0');
}

static int validate(uint64_t length, uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin,
                    uint64_t c_count, uint32_t tiles, int precision, double *d_out)
{
    if (q < 2 || (q & (q - 1))) return set_error(SHB_EINVAL, "q must be a power of two >= 2");
    if (tiles < 1 || q % tiles) return set_error(SHB_EINVAL, "tiles %u does not divide q", tiles);
    if (stride == 0) return set_error(SHB_EINVAL, "stride must be >= 1");
    if (c_begin > q || c_count > q - c_begin) return set_error(SHB_EINVAL, "output rows outside [0, q)");
    if (length && (a0 >= q || (length - 1) > (q - 1 - a0) / stride))
        return set_error(SHB_EINVAL, "support progression leaves [0, q)");
    if (precision != SHB_FP64 && precision != SHB_FP32) return set_error(SHB_EINVAL, "unknown precision %d", precision);
    if (c_count && !d_out) return set_error(SHB_EINVAL, "null output buffer");
    return SHB_OK;
}

static DftArgs make_args(uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin, uint64_t c_count,
                         double *d_out, double *d_prob, double *d_block_sums)
{
    DftArgs a{};
    a.a0 = a0;
    a.stride = stride;
    a.q = q;
    a.two_over_q = 2.0 / (double)q;
    a.c_begin = c_begin;
    a.c_count = c_count;
    a.out = (double2 *)d_out;
    a.prob = d_prob;
    a.block_sums = d_block_sums;
    return a;
}

}  // namespace shb

using namespace shb;

extern "C" uint64_t shb_dft_num_blocks(uint64_t c_count, int precision)
{
    const int K = (precision == SHB_FP32) ? Prec<float>::K : Prec<double>::K;
    const uint64_t per = (uint64_t)DFT_THREADS * K;
    return (c_count + per - 1) / per;
}

extern "C" int shb_dft(const double *d_amps, uint64_t length, uint64_t a0, uint64_t stride, uint64_t q,
                       uint64_t c_begin, uint64_t c_count, uint32_t tiles, double scale, int precision,
                       double *d_out, double *d_prob, double *d_block_sums, void *stream)
{
    SHB_TRY(validate(length, a0, stride, q, c_begin, c_count, tiles, precision, d_out));
    if (c_count == 0) return SHB_OK;
    if (length && !d_amps) return set_error(SHB_EINVAL, "null amplitude buffer");
    if (length && (reinterpret_cast<uintptr_t>(d_amps) & 15))
        return set_error(SHB_EINVAL, "amplitude buffer must be 16-byte aligned");
    DftArgs a = make_args(a0, stride, q, c_begin, c_count, d_out, d_prob, d_block_sums);
    a.amps = (const double2 *)d_amps;
    a.out_re = scale;
    a.out_im = 0.0;
    cudaStream_t st = as_stream(stream);
    if (precision == SHB_FP32) return launch_dft<float, false>(a, length, tiles, st);
    if (tiles == 1 && length && use_mma_engine(false, q)) {
        MmaArgs m{(const double2 *)d_amps, length, a0, stride, q, 2.0 / (double)q, c_begin, c_count,
                  0.0, 0.0, scale, 0.0, (double2 *)d_out, d_prob, d_block_sums};
        return launch_dft_mma<false, false>(m, st);
    }
    return launch_dft<double, false>(a, length, tiles, st);
}

extern "C" int shb_dft_real(const double *d_amps, uint64_t length, uint64_t a0, uint64_t stride, uint64_t q,
                            uint64_t c_begin, uint64_t c_count, uint32_t tiles, double scale, int precision,
                            double *d_out, double *d_prob, double *d_block_sums, void *stream)
{
    SHB_TRY(validate(length, a0, stride, q, c_begin, c_count, tiles, precision, d_out));
    if (c_count == 0) return SHB_OK;
    if (precision == SHB_FP64 && tiles == 1 && length && use_real_form() && use_mma_engine(false, q)) {
        if (!d_amps) return set_error(SHB_EINVAL, "null amplitude buffer");
        if (reinterpret_cast<uintptr_t>(d_amps) & 15)
            return set_error(SHB_EINVAL, "amplitude buffer must be 16-byte aligned");
        MmaArgs m{(const double2 *)d_amps, length, a0, stride, q, 2.0 / (double)q, c_begin, c_count,
                  0.0, 0.0, scale, 0.0, (double2 *)d_out, d_prob, d_block_sums};
        return launch_dft_mma<false, true>(m, as_stream(stream));
    }
    return shb_dft(d_amps, length, a0, stride, q, c_begin, c_count, tiles, scale, precision, d_out, d_prob,
                   d_block_sums, stream);
}

extern "C" int shb_dft_uniform(double amp_re, double amp_im, uint64_t length, uint64_t a0, uint64_t stride,
                               uint64_t q, uint64_t c_begin, uint64_t c_count, uint32_t tiles, double scale,
                               int precision, double *d_out, double *d_prob, double *d_block_sums, void *stream)
{
    SHB_TRY(validate(length, a0, stride, q, c_begin, c_count, tiles, precision, d_out));
    if (c_count == 0) return SHB_OK;
    DftArgs a = make_args(a0, stride, q, c_begin, c_count, d_out, d_prob, d_block_sums);
    a.amps = nullptr;
    a.out_re = amp_re * scale;
    a.out_im = amp_im * scale;
    cudaStream_t st = as_stream(stream);
    if (precision == SHB_FP32) {
        if (tiles == 1 && length && fp32_engine() == F32_TC05)
            return tc05_dft_uniform(length, a0, stride, q, c_begin, c_count, a.out_re, a.out_im, d_out, d_prob,
                                    d_block_sums, (uint64_t)DFT_THREADS * Prec<float>::K, st);
        if (tiles == 1 && length && use_tc32_engine()) {
            MmaArgs m{nullptr, length, a0, stride, q, 2.0 / (double)q, c_begin, c_count,
                      1.0, 0.0, a.out_re, a.out_im, (double2 *)d_out, d_prob, d_block_sums};
            return launch_dft_tc32_uniform(m, st);
        }
        return launch_dft<float, true>(a, length, tiles, st);
    }
    if (tiles == 1 && length && use_i8_engine())
        return i8_dft_uniform(length, a0, stride, q, c_begin, c_count, a.out_re, a.out_im, d_out, d_prob,
                              d_block_sums, (uint64_t)DFT_THREADS * Prec<double>::K, st);
    if (tiles == 1 && length && use_mma_engine(true, q)) {
        // the amplitude is factored out (out factor = amp*scale): the MMA runs on ones
        MmaArgs m{nullptr, length, a0, stride, q, 2.0 / (double)q, c_begin, c_count,
                  1.0, 0.0, a.out_re, a.out_im, (double2 *)d_out, d_prob, d_block_sums};
        // A = 1 is real: the 2-DMMA real form (SHB_MMA_REAL=0 forces the complex form)
        return use_real_form() ? launch_dft_mma<true, true>(m, st) : launch_dft_mma<true, false>(m, st);
    }
    return launch_dft<double, true>(a, length, tiles, st);
}

// Which kernel shb_dft / shb_dft_real / shb_dft_uniform launch for these
// arguments, and the FP64/FP32 flops one phase term costs in it (8 for a
// complex multiply-add, 4 for a real amplitude times a complex phase).
extern "C" const char *shb_dft_engine(int uniform, int real, uint64_t q, int precision, uint32_t tiles,
                                      int *flops_per_term)
{
    if (precision == SHB_FP32 && uniform && tiles == 1 && use_tc32_engine()) {
        if (flops_per_term) *flops_per_term = 8;  // 4 bf16 MACs: (Re, Im) x (hi, lo)
        return fp32_engine() == F32_TC05 ? "dft_tc05_uniform_kernel" : "dft_tc32_uniform_kernel";
    }
    if (precision == SHB_FP64 && uniform && tiles == 1 && use_i8_engine()) {
        if (flops_per_term) *flops_per_term = 32;  // 16 int8 MACs: (Re, Im) x 8 digits
        return "i8::dft_i8_uniform_kernel";
    }
    const bool mma = precision == SHB_FP64 && tiles == 1 && use_mma_engine(uniform != 0, q);
    const bool realf = mma && (uniform || real) && use_real_form();
    if (flops_per_term) *flops_per_term = realf ? 4 : 8;
    if (!mma) return uniform ? "dft_kernel<uniform>" : "dft_kernel<generic>";
    if (realf) return uniform ? "dft_mma_kernel<uniform, real A>" : "dft_mma_kernel<generic, real A>";
    return uniform ? "dft_mma_kernel<uniform, complex A>" : "dft_mma_kernel<generic, complex A>";
}
