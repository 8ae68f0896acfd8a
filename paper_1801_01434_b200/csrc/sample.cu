// Stage 4 (tail of the hot path): Born-rule read of part 1
// (qstate.sample_part1 / l2_norm, qstate.py:108-118).
//
//   probs = np.abs(amp)**2 ; cum = np.cumsum(probs)
//   m = searchsorted(cum, u*cum[-1], side="right")
//
// np.cumsum is a strictly sequential chain of float64 adds, and a parallel
// scan rounds differently, which flips m near CDF boundaries.  This file
// reproduces the sequential chain EXACTLY on the GPU.  While the running sum
// S stays inside one binade [2^e, 2^(e+1)) with ulp u, the float add
// fl(S + p) equals S + u*round(p/u) (ties: round-half-even on the parity of
// S/u + floor(p/u)).  So inside a binade the chain is an exact INTEGER prefix
// sum of per-element increments, which a CTA computes with a block scan; the
// one add that leaves the binade is done in floating point, and rare ties are
// resolved in order by one thread.  The result is bit-identical to numpy for
// any input (tests/test_gpu_parity.py checks adversarial vectors).
//
// Pass 1 (one CTA, sequential over 8192-element chunks) yields cum[-1] and
// the exact running sum at every chunk start; pass 2 re-walks only the one
// chunk that contains u*cum[-1].
#include <math.h>

#include <vector>

#include "shb_internal.cuh"

namespace shb {

// ------------------------------------------------------------ probabilities
__global__ void prob_kernel(const double2 *__restrict__ v, uint64_t n, double *__restrict__ p)
{
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += step) {
        const double2 z = v[i];
        const double h = hypot(z.x, z.y);
        p[i] = h * h;
    }
}

// ------------------------------------------------- deterministic tree sum
constexpr int SUM_THREADS = 512;
constexpr int SUM_BLOCKS = 1024;

__device__ inline double block_sum(double v, double *tmp)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) tmp[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) r += tmp[w];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SUM_THREADS) sum_partial_kernel(const double *__restrict__ x, uint64_t n,
                                                                  double *__restrict__ part)
{
    __shared__ double tmp[SUM_THREADS / 32];
    // fixed assignment: block b owns a contiguous slice -> order independent of the GPU
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = per * blockIdx.x, hi = (lo + per < n) ? lo + per : n;
    double s = 0.0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += SUM_THREADS) s += x[i];
    const double b = block_sum(s, tmp);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void __launch_bounds__(SUM_THREADS) sum_final_kernel(const double *__restrict__ part, int n,
                                                                double *__restrict__ out)
{
    __shared__ double tmp[SUM_THREADS / 32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += SUM_THREADS) s += part[i];
    const double b = block_sum(s, tmp);
    if (threadIdx.x == 0) *out = b;
}

// --------------------------------------------- exact sequential cumsum walk
constexpr int SEQ_THREADS = 1024;
constexpr int SEQ_V = 8;                           // elements per thread per chunk
constexpr int SEQ_CHUNK = SEQ_THREADS * SEQ_V;     // 8192
constexpr uint64_t SAT = 1ull << 62;               // saturation for the unit scan
constexpr uint64_t TWO53 = 1ull << 53;

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b)
{
    const uint64_t s = a + b;
    return s > SAT ? SAT : s;
}

// ulp of S and the power of two where it next changes
__device__ __forceinline__ void binade(double S, double &u, double &B)
{
    if (S < 0x1p-1021) {
        u = 0x1p-1074;
        B = 0x1p-1021;
    } else {
        int e;
        frexp(S, &e);  // S in [2^(e-1), 2^e)
        u = ldexp(1.0, e - 53);
        B = ldexp(1.0, e);
    }
}

struct SeqShared {
    uint64_t warp_tmp[SEQ_THREADS / 32];
    uint32_t warp_min[SEQ_THREADS / 32];
    uint64_t P[SEQ_CHUNK];        // inclusive unit prefix of the current range
    uint64_t add[SEQ_CHUNK];      // per-element unit increments
    uint8_t tie[SEQ_CHUNK];
    uint16_t tlist[SEQ_CHUNK];    // tie positions, ascending (parallel tie resolution)
    double S;                     // exact running sum before `start`
    int start;                    // first unprocessed local index
    int done;
    uint64_t found;
};

// block-wide saturating inclusive scan over thread totals -> exclusive offset
__device__ inline uint64_t block_excl_sat(uint64_t v, uint64_t *warp_tmp)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = sat_add(x, y);
    }
    if (lane == 31) warp_tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t w = warp_tmp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w = sat_add(w, y);
        }
        warp_tmp[lane] = w;
    }
    __syncthreads();
    const uint64_t before_warp = wid ? warp_tmp[wid - 1] : 0;
    // x - v is exact unless saturated; recompute exclusive as sat(before_warp + (x excl v))
    uint64_t excl_in_warp = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) excl_in_warp = 0;
    __syncthreads();
    return sat_add(before_warp, excl_in_warp);
}

__device__ inline int block_min_int(int v, uint32_t *warp_min)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_down_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) warp_min[wid] = (uint32_t)v;
    __syncthreads();
    int r = (int)warp_min[0];
    for (int w = 1; w < SEQ_THREADS / 32; w++) r = min(r, (int)warp_min[w]);
    __syncthreads();
    return r;
}

// Per-tile record for the fast walk: integer increment of the whole tile in
// the binade predicted for its start (approximate prefix of tile sums).
struct TileRec {
    uint64_t A;     // sum over the tile of round(p / 2^uexp) (saturating)
    int32_t uexp;   // predicted ulp exponent (INT32_MIN: predicted start sum is 0)
    uint32_t flags; // TR_TIES | TR_ALLZERO
};
enum : uint32_t { TR_TIES = 1u, TR_ALLZERO = 2u };

__device__ __forceinline__ int ulp_exp(double S)
{
    if (S < 0x1p-1021) return -1074;
    int e;
    frexp(S, &e);
    return e - 53;
}

// pass 1: approximate tile sums (any order: they only predict binades)
__global__ void __launch_bounds__(256) tile_sum_kernel(const double *__restrict__ p, uint64_t L,
                                                      double *__restrict__ tsum)
{
    __shared__ double tmp[8];
    const uint64_t base = (uint64_t)blockIdx.x * SEQ_CHUNK;
    double s = 0.0;
    for (int i = threadIdx.x; i < SEQ_CHUNK; i += 256)
        if (base + i < L) s += p[base + i];
    const double b = block_sum(s, tmp);
    if (threadIdx.x == 0) tsum[blockIdx.x] = b;
}

// pass 2: exclusive prefix of the tile sums (one CTA)
__global__ void __launch_bounds__(SUM_THREADS) tile_prefix_kernel(const double *__restrict__ tsum, uint64_t nt,
                                                                 double s_in, double *__restrict__ tstart)
{
    __shared__ double part[SUM_THREADS];
    const uint64_t per = (nt + SUM_THREADS - 1) / SUM_THREADS;
    const uint64_t lo = per * threadIdx.x, hi = lo + per < nt ? lo + per : nt;
    double s = 0.0;
    for (uint64_t i = lo; i < hi; i++) s += tsum[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = s_in;  // approximate tile starts only predict binades (exactness comes from the walk)
        for (int t = 0; t < SUM_THREADS; t++) {
            const double v = part[t];
            part[t] = run;
            run += v;
        }
    }
    __syncthreads();
    double run = part[threadIdx.x];
    for (uint64_t i = lo; i < hi; i++) {
        tstart[i] = run;
        run += tsum[i];
    }
}

// pass 3: per-tile integer increment in the predicted binade
__global__ void __launch_bounds__(256) tile_rec_kernel(const double *__restrict__ p, uint64_t L,
                                                      const double *__restrict__ tstart,
                                                      TileRec *__restrict__ rec)
{
    __shared__ uint64_t tmpA[8];
    __shared__ uint32_t tmpF[8];
    const uint64_t base = (uint64_t)blockIdx.x * SEQ_CHUNK;
    const double S0 = tstart[blockIdx.x];
    const bool zero = !(S0 > 0.0);
    const int ue = zero ? -1074 : ulp_exp(S0);
    uint64_t A = 0;
    uint32_t ties = 0, nonzero = 0;
    for (int i = threadIdx.x; i < SEQ_CHUNK; i += 256) {
        if (base + i >= L) break;
        const double v = p[base + i];
        nonzero |= (v != 0.0);
        const double x = ldexp(v, -ue);  // exact power-of-two scaling
        uint64_t a;
        if (!(x < 9007199254740992.0)) {
            a = 1ull << 54;
        } else {
            const double kf = floor(x), fr = x - kf;
            a = (uint64_t)kf + (fr > 0.5 ? 1u : 0u);
            ties |= (fr == 0.5);
        }
        A = sat_add(A, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        A = sat_add(A, __shfl_down_sync(0xffffffffu, A, o));
        ties |= __shfl_down_sync(0xffffffffu, ties, o);
        nonzero |= __shfl_down_sync(0xffffffffu, nonzero, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        tmpA[wid] = A;
        tmpF[wid] = (ties ? TR_TIES : 0u) | (nonzero ? 0u : TR_ALLZERO);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t a = 0;
        uint32_t f = TR_ALLZERO;
        for (int w = 0; w < 8; w++) {
            a = sat_add(a, tmpA[w]);
            const uint32_t fw = tmpF[w];
            f = (f & fw & TR_ALLZERO) | ((f | fw) & TR_TIES);
        }
        rec[blockIdx.x] = TileRec{a, zero ? INT32_MIN : ue, f};
    }
}

// Resolve ties in index order: a tie rounds half-to-even on the parity of the
// running unit count just before it, which is the exclusive prefix of the
// unadjusted increments plus the adjustments of the earlier ties.  One block
// scan gives every prefix; one thread then visits only the tie positions (a
// handful per tile) instead of all 8192 elements.  Rare path: kept out of
// line so it does not raise the register count of the walk.
__device__ __noinline__ void resolve_ties(SeqShared &sh, uint64_t loc, uint64_t Su)
{
    const int tid = threadIdx.x;
    uint64_t ex = block_excl_sat(loc, sh.warp_tmp);
    uint64_t nt = 0;
#pragma unroll 1
    for (int k = 0; k < SEQ_V; k++) {
        const int li = tid * SEQ_V + k;
        sh.P[li] = ex;  // exclusive prefix at li (from `start`)
        ex = sat_add(ex, sh.add[li]);
        nt += sh.tie[li];
    }
    uint64_t toff = block_excl_sat(nt, sh.warp_tmp);
#pragma unroll 1
    for (int k = 0; k < SEQ_V; k++) {
        const int li = tid * SEQ_V + k;
        if (sh.tie[li]) sh.tlist[toff++] = (uint16_t)li;
    }
    uint64_t ntie = nt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ntie += __shfl_xor_sync(0xffffffffu, ntie, o);
    __syncthreads();  // block_excl_sat's last reads of warp_tmp are done
    if ((tid & 31) == 0) sh.warp_tmp[tid >> 5] = ntie;
    __syncthreads();
    if (tid == 0) {
        uint64_t total_ties = 0;
        for (int w = 0; w < SEQ_THREADS / 32; w++) total_ties += sh.warp_tmp[w];
        uint64_t adj = 0;
        for (uint64_t j = 0; j < total_ties; j++) {
            const int li = sh.tlist[j];
            const uint64_t a = sh.add[li];
            if ((Su + sh.P[li] + adj + a) & 1ull) {  // saturated prefixes lie past a crossing
                sh.add[li] = a + 1;
                adj++;
            }
        }
    }
    __syncthreads();
}

// Detailed exact walk of one tile by the whole CTA (binade crossings, ties,
// first nonzero, or the target search).  Updates sh.S / sh.found / sh.done.
__device__ void walk_tile(const double *__restrict__ p, uint64_t L, uint64_t ck, int mode, double target,
                          SeqShared &sh)
{
    const int tid = threadIdx.x;
    const uint64_t base = ck * SEQ_CHUNK;
    const int n = (int)((L - base) < (uint64_t)SEQ_CHUNK ? (L - base) : SEQ_CHUNK);
    double v[SEQ_V];
#pragma unroll
    for (int k = 0; k < SEQ_V; k++) {
        const int li = tid * SEQ_V + k;
        v[k] = (li < n) ? p[base + li] : 0.0;
    }
    if (tid == 0) sh.start = 0;
    __syncthreads();
    while (true) {
        const int start = sh.start;
        if (start >= n) break;
        const double S = sh.S;
        if (S == 0.0) {
            // running sum is still exactly zero: the first nonzero element sets it
            int first = n;
#pragma unroll
            for (int k = 0; k < SEQ_V; k++) {
                const int li = tid * SEQ_V + k;
                if (li >= start && li < n && v[k] != 0.0 && li < first) first = li;
            }
            first = block_min_int(first, sh.warp_min);
            if (first >= n) break;  // whole rest of the tile keeps S == 0
            if (tid == 0) {
                sh.S = 0.0 + p[base + first];
                if (mode == 1 && sh.S > target) {
                    sh.found = base + first;
                    sh.done = 1;
                }
                sh.start = first + 1;
            }
            __syncthreads();
            if (sh.done) break;
            continue;
        }
        double u, B;
        binade(S, u, B);
        const uint64_t Su = (uint64_t)(S / u);
        // per-element unit increments in the current binade
        uint64_t loc = 0;
        int any_tie = 0;
#pragma unroll
        for (int k = 0; k < SEQ_V; k++) {
            const int li = tid * SEQ_V + k;
            uint64_t a = 0;
            uint8_t t = 0;
            if (li >= start && li < n) {
                const double x = v[k] / u;
                if (!(x < 9007199254740992.0)) {
                    a = 1ull << 54;  // certainly leaves the binade
                } else {
                    const double kf = floor(x), fr = x - kf;
                    a = (uint64_t)kf + (fr > 0.5 ? 1u : 0u);
                    t = (fr == 0.5);
                    any_tie |= t;
                }
            }
            sh.add[li] = a;
            sh.tie[li] = t;
            loc = sat_add(loc, a);
        }
        any_tie = __syncthreads_or(any_tie);
        if (any_tie) {
            resolve_ties(sh, loc, Su);
            loc = 0;
#pragma unroll
            for (int k = 0; k < SEQ_V; k++) loc = sat_add(loc, sh.add[tid * SEQ_V + k]);
        }
        uint64_t run = block_excl_sat(loc, sh.warp_tmp);
        // inclusive prefix + first crossing (N >= 2^53) / first hit (N > floor(target/u))
        const double tu = target / u;
        const bool hit_possible = (mode == 1) && (tu < 9007199254740992.0);
        const uint64_t tfl = hit_possible ? (uint64_t)floor(tu) : 0;
        int cross = n, hit = n;
#pragma unroll
        for (int k = 0; k < SEQ_V; k++) {
            const int li = tid * SEQ_V + k;
            run = sat_add(run, sh.add[li]);
            sh.P[li] = run;
            if (li >= start && li < n) {
                const uint64_t N = sat_add(Su, run);
                if (N >= TWO53 && li < cross) cross = li;
                if (hit_possible && N > tfl && li < hit) hit = li;
            }
        }
        cross = block_min_int(cross, sh.warp_min);
        hit = block_min_int(hit, sh.warp_min);
        if (tid == 0) {
            if (hit < cross) {
                sh.found = base + hit;
                sh.done = 1;
            } else if (cross < n) {
                // exact sum just before the crossing element, then one float add
                const uint64_t Nprev = Su + (cross > start ? sh.P[cross - 1] : 0);
                const double Sprev = (double)Nprev * u;
                const double Snew = Sprev + p[base + cross];
                sh.S = Snew;
                sh.start = cross + 1;
                if (mode == 1 && Snew > target) {
                    sh.found = base + cross;
                    sh.done = 1;
                }
            } else {
                sh.S = (double)(Su + sh.P[n - 1]) * u;
                sh.start = n;
            }
        }
        __syncthreads();
        if (sh.done) break;
    }
    __syncthreads();
}

// Walk tiles [tile_lo, tile_hi) from the exact running sum S0.
// mode 0: record the exact S at every tile start (tile_S) and the total;
//         warp 0 advances over tiles whose record proves they stay inside
//         one binade without ties (S += 2^uexp * A, exact), the whole CTA
//         walks the others element by element.
// mode 1: find the first index whose running sum exceeds `target`.
__global__ void __launch_bounds__(SEQ_THREADS, 1)
    seqscan_kernel(const double *__restrict__ p, uint64_t L, uint64_t tile_lo, uint64_t tile_hi, double S0,
                   int mode, double target, const TileRec *__restrict__ recs, double *__restrict__ tile_S,
                   double *__restrict__ total, uint64_t *__restrict__ found)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SeqShared &sh = *reinterpret_cast<SeqShared *>(smem_raw);
    __shared__ uint64_t next_slow;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        sh.S = S0;
        sh.done = 0;
        sh.found = L;
    }
    __syncthreads();
    uint64_t t = tile_lo;
    while (t < tile_hi) {
        if (recs != nullptr) {
            if (tid < 32) {
                // warp 0 advances 32 tile records per step: inside one binade
                // the running sum after tile i is S + 2^uexp * (A_0 + ... + A_i),
                // a warp scan; the first tile that crosses a binade, has a tie or
                // was mispredicted stops the fast walk (ballot).
                double S = sh.S;
                uint64_t tt = t, stop = tile_hi;
                TileRec rn{0, 0, TR_ALLZERO};  // records of the next step, loaded one step ahead
                if (tt + lane < tile_hi) rn = recs[tt + lane];
                while (tt < tile_hi) {
                    const int cnt = (tile_hi - tt) < 32 ? (int)(tile_hi - tt) : 32;
                    const TileRec r = rn;
                    if (tt + 32 + lane < tile_hi) rn = recs[tt + 32 + lane];
                    int first_bad;
                    if (S == 0.0) {
                        const bool ok = lane >= cnt || (r.flags & TR_ALLZERO);
                        const uint32_t bad = ~__ballot_sync(0xffffffffu, ok);
                        first_bad = bad ? __ffs(bad) - 1 : cnt;
                        if (mode == 0 && lane < first_bad && lane < cnt) tile_S[tt + lane] = 0.0;
                    } else {
                        // S > 0 normal: S = sig * 2^(E - 1075), sig in [2^52, 2^53)
                        const uint64_t bits = (uint64_t)__double_as_longlong(S);
                        const int E = (int)(bits >> 52);
                        const uint64_t sig = (bits & ((1ull << 52) - 1)) | (1ull << 52);
                        const uint64_t a = lane < cnt ? r.A : 0;
                        uint64_t P = a;  // inclusive saturating scan of the increments
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint64_t y = __shfl_up_sync(0xffffffffu, P, o);
                            if (lane >= o) P = sat_add(P, y);
                        }
                        const bool ok = lane >= cnt ||
                                        (E > 1 && (E - 1075) == r.uexp && !(r.flags & TR_TIES) && sig + P < TWO53);
                        const uint32_t bad = ~__ballot_sync(0xffffffffu, ok);
                        first_bad = bad ? __ffs(bad) - 1 : cnt;
                        const uint64_t excl = P - a;  // exact below saturation, which only bad lanes reach
                        if (mode == 0 && lane < first_bad && lane < cnt)
                            tile_S[tt + lane] =
                                __longlong_as_double((long long)(((uint64_t)E << 52) | (sig + excl - (1ull << 52))));
                        // running sum after the last good tile
                        const uint64_t Pl = __shfl_sync(0xffffffffu, P, first_bad > 0 ? first_bad - 1 : 0);
                        if (first_bad > 0)
                            S = __longlong_as_double((long long)(((uint64_t)E << 52) | (sig + Pl - (1ull << 52))));
                    }
                    if (first_bad < cnt) {
                        stop = tt + first_bad;
                        break;
                    }
                    tt += cnt;
                }
                if (lane == 0) {
                    sh.S = S;
                    next_slow = stop;
                }
            }
            __syncthreads();
            t = next_slow;
            if (t >= tile_hi) break;
        }
        if (mode == 0 && tid == 0) tile_S[t] = sh.S;
        walk_tile(p, L, t, mode, target, sh);
        if (sh.done) break;
        t++;
    }
    __syncthreads();
    if (tid == 0) {
        if (total) *total = sh.S;
        if (found) *found = sh.found;
    }
}

static size_t seq_smem() { return sizeof(SeqShared); }

static int seq_prepare()
{
    SHB_TRY_CUDA(cudaFuncSetAttribute(seqscan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)seq_smem()));
    return SHB_OK;
}

}  // namespace shb

using namespace shb;

extern "C" int shb_probabilities(const double *d_state, uint64_t count, double *d_prob, void *stream)
{
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    uint64_t blocks = (count + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    prob_kernel<<<(unsigned)blocks, 256, 0, st>>>((const double2 *)d_state, count, d_prob);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

extern "C" int shb_sum(const double *d_x, uint64_t count, double *out, void *stream)
{
    if (!out) return set_error(SHB_EINVAL, "null output");
    *out = 0.0;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    Scratch part, res;
    SHB_TRY(scratch_alloc(part, sizeof(double) * SUM_BLOCKS, st));
    SHB_TRY(scratch_alloc(res, sizeof(double), st));
    sum_partial_kernel<<<SUM_BLOCKS, SUM_THREADS, 0, st>>>(d_x, count, (double *)part.ptr);
    SHB_LAUNCHED();
    sum_final_kernel<<<1, SUM_THREADS, 0, st>>>((const double *)part.ptr, SUM_BLOCKS, (double *)res.ptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    SHB_TRY_CUDA(cudaMemcpyAsync(out, res.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    return SHB_OK;
}

// The sequential cumsum in two parts.  (1) Records: approximate tile sums,
// their prefix from a hint of the running value entering the vector, and per
// tile the integer increment in the binade that prefix predicts -- all
// parallel, and exactness does not depend on the hint (a mispredicted tile
// is simply walked element by element).  (2) The walk: one CTA advances the
// EXACT running sum from s_in over the records (32 tiles per warp step) and
// writes the exact running value at every tile start.  A sharded read
// computes (1) on every shard at once and chains only (2) from shard to shard.
static int seq_records(const double *d_prob, uint64_t count, double s_hint, TileRec *recs, cudaStream_t st)
{
    const uint64_t nt = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch tsum, tstart;
    SHB_TRY(scratch_alloc(tsum, sizeof(double) * nt, st));
    SHB_TRY(scratch_alloc(tstart, sizeof(double) * nt, st));
    tile_sum_kernel<<<(unsigned)nt, 256, 0, st>>>(d_prob, count, (double *)tsum.ptr);
    SHB_LAUNCHED();
    tile_prefix_kernel<<<1, SUM_THREADS, 0, st>>>((const double *)tsum.ptr, nt, s_hint, (double *)tstart.ptr);
    SHB_LAUNCHED();
    tile_rec_kernel<<<(unsigned)nt, 256, 0, st>>>(d_prob, count, (const double *)tstart.ptr, recs);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

static int seq_walk(const double *d_prob, uint64_t count, const TileRec *recs, double s_in, double *tile_S,
                    double *total_host, cudaStream_t st)
{
    SHB_TRY(seq_prepare());
    const uint64_t nt = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch tot;
    SHB_TRY(scratch_alloc(tot, sizeof(double), st));
    seqscan_kernel<<<1, SEQ_THREADS, seq_smem(), st>>>(d_prob, count, 0, nt, s_in, 0, 0.0, recs, tile_S,
                                                         (double *)tot.ptr, nullptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    SHB_TRY_CUDA(cudaMemcpyAsync(total_host, tot.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    return SHB_OK;
}

// exact walk over all tiles -> (total, exact running sum at every tile start)
static int seq_total(const double *d_prob, uint64_t count, double s_in, double *tile_S, double *total_host,
                     cudaStream_t st)
{
    const uint64_t nt = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch recs;
    SHB_TRY(scratch_alloc(recs, sizeof(TileRec) * nt, st));
    SHB_TRY(seq_records(d_prob, count, s_in, (TileRec *)recs.ptr, st));
    return seq_walk(d_prob, count, (const TileRec *)recs.ptr, s_in, tile_S, total_host, st);
}

extern "C" int shb_cumsum_total(const double *d_prob, uint64_t count, double *total, void *stream)
{
    if (!total) return set_error(SHB_EINVAL, "null output");
    *total = 0.0;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    const uint64_t nch = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch cs;
    SHB_TRY(scratch_alloc(cs, sizeof(double) * nch, st));
    return seq_total(d_prob, count, 0.0, (double *)cs.ptr, total, st);
}

static int search_from_tiles(const double *d_prob, uint64_t count, const double *d_tile_S, double tot,
                             double target, uint64_t *index, cudaStream_t st)
{
    *index = count;
    if (!(tot > target)) return SHB_OK;  // no running sum exceeds target -> count
    const uint64_t nch = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    // tile c ends with running sum tile_S[c+1] (or the total for the last one)
    std::vector<double> hs(nch);
    SHB_TRY_CUDA(cudaMemcpyAsync(hs.data(), d_tile_S, sizeof(double) * nch, cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    uint64_t lo = 0, hi = nch - 1;  // first tile whose end value > target
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (hs[mid + 1] > target) hi = mid;
        else lo = mid + 1;
    }
    Scratch fnd;
    SHB_TRY(scratch_alloc(fnd, sizeof(uint64_t), st));
    seqscan_kernel<<<1, SEQ_THREADS, seq_smem(), st>>>(d_prob, count, lo, lo + 1, hs[lo], 1, target, nullptr,
                                                         nullptr, nullptr, (uint64_t *)fnd.ptr);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    SHB_TRY_CUDA(cudaMemcpyAsync(index, fnd.ptr, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SHB_TRY_CUDA(cudaStreamSynchronize(st));
    return SHB_OK;
}

extern "C" int shb_cumsum_search(const double *d_prob, uint64_t count, double target, uint64_t *index,
                                 void *stream)
{
    if (!index) return set_error(SHB_EINVAL, "null output");
    *index = count;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    const uint64_t nch = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch cs;
    SHB_TRY(scratch_alloc(cs, sizeof(double) * nch, st));
    double tot = 0.0;
    SHB_TRY(seq_total(d_prob, count, 0.0, (double *)cs.ptr, &tot, st));
    return search_from_tiles(d_prob, count, (const double *)cs.ptr, tot, target, index, st);
}

// Continuations of the sequential cumsum from a running value s_in (a shard of
// a longer vector whose earlier elements summed, left to right, to s_in): the
// sharded Born-rule read chains these rank to rank (distributed.py).
extern "C" int shb_cumsum_total_from(const double *d_prob, uint64_t count, double s_in, double *s_out,
                                     void *stream)
{
    if (!s_out) return set_error(SHB_EINVAL, "null output");
    *s_out = s_in;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    const uint64_t nch = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch cs;
    SHB_TRY(scratch_alloc(cs, sizeof(double) * nch, st));
    return seq_total(d_prob, count, s_in, (double *)cs.ptr, s_out, st);
}

extern "C" int shb_cumsum_search_from(const double *d_prob, uint64_t count, double s_in, double target,
                                      uint64_t *index, void *stream)
{
    if (!index) return set_error(SHB_EINVAL, "null output");
    *index = count;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    const uint64_t nch = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch cs;
    SHB_TRY(scratch_alloc(cs, sizeof(double) * nch, st));
    double tot = s_in;
    SHB_TRY(seq_total(d_prob, count, s_in, (double *)cs.ptr, &tot, st));
    return search_from_tiles(d_prob, count, (const double *)cs.ptr, tot, target, index, st);
}

extern "C" int shb_sample_index(const double *d_prob, uint64_t count, double u, uint64_t *index, double *total,
                                void *stream)
{
    if (!index) return set_error(SHB_EINVAL, "null output");
    *index = count;
    if (total) *total = 0.0;
    if (count == 0) return SHB_OK;
    cudaStream_t st = as_stream(stream);
    const uint64_t nch = (count + SEQ_CHUNK - 1) / SEQ_CHUNK;
    Scratch cs;
    SHB_TRY(scratch_alloc(cs, sizeof(double) * nch, st));
    double tot = 0.0;
    SHB_TRY(seq_total(d_prob, count, 0.0, (double *)cs.ptr, &tot, st));
    if (total) *total = tot;
    const double target = u * tot;  // s.uniform() * cum[-1] (qstate.py:113)
    return search_from_tiles(d_prob, count, (const double *)cs.ptr, tot, target, index, st);
}

// ------------------------------------------------ split scan (sharded reads)
extern "C" uint64_t shb_cumsum_tiles(uint64_t count) { return (count + SEQ_CHUNK - 1) / SEQ_CHUNK; }

extern "C" uint64_t shb_cumsum_record_bytes(void) { return sizeof(TileRec); }

extern "C" int shb_cumsum_records(const double *d_prob, uint64_t count, double s_hint, void *d_recs, void *stream)
{
    if (count == 0) return SHB_OK;
    if (!d_prob || !d_recs) return set_error(SHB_EINVAL, "null buffer");
    return seq_records(d_prob, count, s_hint, (TileRec *)d_recs, as_stream(stream));
}

extern "C" int shb_cumsum_walk(const double *d_prob, uint64_t count, const void *d_recs, double s_in,
                               double *d_tile_S, double *s_out, void *stream)
{
    if (!s_out) return set_error(SHB_EINVAL, "null output");
    *s_out = s_in;
    if (count == 0) return SHB_OK;
    if (!d_prob || !d_recs || !d_tile_S) return set_error(SHB_EINVAL, "null buffer");
    return seq_walk(d_prob, count, (const TileRec *)d_recs, s_in, d_tile_S, s_out, as_stream(stream));
}

extern "C" int shb_cumsum_find(const double *d_prob, uint64_t count, const double *d_tile_S, double total,
                               double target, uint64_t *index, void *stream)
{
    if (!index) return set_error(SHB_EINVAL, "null output");
    *index = count;
    if (count == 0) return SHB_OK;
    if (!d_prob || !d_tile_S) return set_error(SHB_EINVAL, "null buffer");
    return search_from_tiles(d_prob, count, d_tile_S, total, target, index, as_stream(stream));
}
