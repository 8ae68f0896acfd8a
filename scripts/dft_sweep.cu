// Exploration harness (not part of the product): time variants of the
// uniform-comb Horner DFT inner loop at q = 2^24, M = 144631 (n=3127 attempt)
// to pick K (outputs per thread), CTA size and occupancy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dft_sweep scripts/dft_sweep.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void phase(uint64_t idx, uint64_t q, double two_over_q, double &c, double &s)
{
    const int64_t sidx = (idx > (q >> 1)) ? (int64_t)(idx - q) : (int64_t)idx;
    sincospi((double)sidx * two_over_q, &s, &c);
}

template <int K, int NT, int MINB, int VAR>
__global__ void __launch_bounds__(NT, MINB) kern(uint64_t a0, uint64_t stride, uint64_t len, uint64_t q,
                                                 double two_over_q, double scale, double2 *out, double *prob)
{
    const uint64_t qmask = q - 1;
    const uint64_t cblk = (uint64_t)blockIdx.x * NT * K;
    double wr[K], wi[K], hr[K], hi[K], vr[K], vi[K];
    uint64_t cval[K];
#pragma unroll
    for (int i = 0; i < K; i++) {
        cval[i] = cblk + (uint64_t)i * NT + threadIdx.x;
        double co, si;
        phase((stride * cval[i]) & qmask, q, two_over_q, co, si);
        wr[i] = co;
        wi[i] = si;
        hr[i] = hi[i] = vr[i] = vi[i] = 0.0;
    }
    const uint64_t SEG = 8192;
    for (uint64_t s0 = 0; s0 < len; s0 += SEG) {
        const int cnt = (int)((len - s0) < SEG ? (len - s0) : SEG);
        if (VAR == 0) {
#pragma unroll 4
            for (int e = 0; e < cnt; e++) {
#pragma unroll
                for (int i = 0; i < K; i++) {
                    const double t_re = fma(hi[i], wi[i], 1.0);
                    const double t_im = hi[i] * wr[i];
                    const double n_re = fma(hr[i], wr[i], t_re);
                    const double n_im = fma(-hr[i], wi[i], t_im);
                    hr[i] = n_re;
                    hi[i] = n_im;
                }
            }
        } else {
            // variant 1: interleave so consecutive FP64 ops share an operand
#pragma unroll 4
            for (int e = 0; e < cnt; e++) {
                double t_re[K], t_im[K];
#pragma unroll
                for (int i = 0; i < K; i++) {
                    t_re[i] = fma(hi[i], wi[i], 1.0);
                    t_im[i] = hi[i] * wr[i];
                }
#pragma unroll
                for (int i = 0; i < K; i++) {
                    const double n_re = fma(hr[i], wr[i], t_re[i]);
                    const double n_im = fma(-hr[i], wi[i], t_im[i]);
                    hr[i] = n_re;
                    hi[i] = n_im;
                }
            }
        }
        const uint64_t a_last = a0 + (s0 + cnt - 1) * stride;
#pragma unroll
        for (int i = 0; i < K; i++) {
            double sc, ss;
            phase((a_last * cval[i]) & qmask, q, two_over_q, sc, ss);
            vr[i] = fma(sc, hr[i], fma(-ss, hi[i], vr[i]));
            vi[i] = fma(sc, hi[i], fma(ss, hr[i], vi[i]));
            hr[i] = hi[i] = 0.0;
        }
    }
#pragma unroll
    for (int i = 0; i < K; i++) {
        const uint64_t ci = cblk + (uint64_t)i * NT + threadIdx.x;
        if (ci < q) {
            const double o_re = vr[i] * scale, o_im = vi[i] * scale;
            out[ci] = make_double2(o_re, o_im);
            const double h = hypot(o_re, o_im);
            prob[ci] = h * h;
        }
    }
}

// FP32 Horner (SEG terms per exact FP64 re-seed), FP64 segment accumulation
template <int K, int NT, int MINB, int SEGF>
__global__ void __launch_bounds__(NT, MINB) kern32(uint64_t a0, uint64_t stride, uint64_t len, uint64_t q,
                                                   double two_over_q, double scale, double2 *out, double *prob)
{
    const uint64_t qmask = q - 1;
    const uint64_t cblk = (uint64_t)blockIdx.x * NT * K;
    float wr[K], wi[K], hr[K], hi[K];
    double vr[K], vi[K];
    uint64_t cval[K];
#pragma unroll
    for (int i = 0; i < K; i++) {
        cval[i] = cblk + (uint64_t)i * NT + threadIdx.x;
        double co, si;
        phase((stride * cval[i]) & qmask, q, two_over_q, co, si);
        wr[i] = (float)co;
        wi[i] = (float)si;
        hr[i] = hi[i] = 0.f;
        vr[i] = vi[i] = 0.0;
    }
    for (uint64_t s0 = 0; s0 < len; s0 += SEGF) {
        const int cnt = (int)((len - s0) < SEGF ? (len - s0) : SEGF);
#pragma unroll 4
        for (int e = 0; e < cnt; e++) {
#pragma unroll
            for (int i = 0; i < K; i++) {
                const float t_re = fmaf(hi[i], wi[i], 1.f);
                const float t_im = hi[i] * wr[i];
                const float n_re = fmaf(hr[i], wr[i], t_re);
                const float n_im = fmaf(-hr[i], wi[i], t_im);
                hr[i] = n_re;
                hi[i] = n_im;
            }
        }
        const uint64_t a_last = a0 + (s0 + cnt - 1) * stride;
#pragma unroll
        for (int i = 0; i < K; i++) {
            double sc, ss;
            phase((a_last * cval[i]) & qmask, q, two_over_q, sc, ss);
            vr[i] = fma(sc, (double)hr[i], fma(-ss, (double)hi[i], vr[i]));
            vi[i] = fma(sc, (double)hi[i], fma(ss, (double)hr[i], vi[i]));
            hr[i] = hi[i] = 0.f;
        }
    }
#pragma unroll
    for (int i = 0; i < K; i++) {
        const uint64_t ci = cblk + (uint64_t)i * NT + threadIdx.x;
        if (ci < q) {
            const double o_re = vr[i] * scale, o_im = vi[i] * scale;
            out[ci] = make_double2(o_re, o_im);
            const double h = hypot(o_re, o_im);
            prob[ci] = h * h;
        }
    }
}

template <int K, int NT, int MINB, int SEGF>
void run32(const char *name, uint64_t q, uint64_t a0, uint64_t stride, uint64_t len, double2 *out, double *prob,
           double *pref)
{
    const uint64_t nblk = (q + (uint64_t)NT * K - 1) / ((uint64_t)NT * K);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern32<K, NT, MINB, SEGF><<<nblk, NT>>>(a0, stride, len, q, 2.0 / q, 1.0 / sqrt((double)q), out, prob);
    cudaEventRecord(e0);
    kern32<K, NT, MINB, SEGF><<<nblk, NT>>>(a0, stride, len, q, 2.0 / q, 1.0 / sqrt((double)q), out, prob);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern32<K, NT, MINB, SEGF>);
    // max |dp| / max p against the FP64 probabilities (whole vector)
    static double hp[1 << 20], hr[1 << 20];
    double md = 0, mp = 0;
    for (uint64_t off = 0; off < q; off += (1 << 20)) {
        cudaMemcpy(hp, prob + off, sizeof hp, cudaMemcpyDeviceToHost);
        cudaMemcpy(hr, pref + off, sizeof hr, cudaMemcpyDeviceToHost);
        for (int i = 0; i < (1 << 20); i++) {
            md = fmax(md, fabs(hp[i] - hr[i]));
            mp = fmax(mp, hr[i]);
        }
    }
    printf("%-28s regs=%3d  %8.2f ms  %6.2f 'TFLOP/s'  %.3e terms/s  max|dp|/maxp=%.2e err=%s\n", name, fa.numRegs, ms,
           8.0 * (double)q * len / (ms * 1e-3) / 1e12, (double)q * len / (ms * 1e-3), md / mp,
           cudaGetErrorString(cudaGetLastError()));
}

template <int K, int NT, int MINB, int VAR>
void run(const char *name, uint64_t q, uint64_t a0, uint64_t stride, uint64_t len, double2 *out, double *prob,
         double2 *ref)
{
    const uint64_t nblk = (q + (uint64_t)NT * K - 1) / ((uint64_t)NT * K);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<K, NT, MINB, VAR><<<nblk, NT>>>(a0, stride, len, q, 2.0 / q, 1.0 / sqrt((double)q), out, prob);
    cudaEventRecord(e0);
    const int reps = 2;
    for (int r = 0; r < reps; r++)
        kern<K, NT, MINB, VAR><<<nblk, NT>>>(a0, stride, len, q, 2.0 / q, 1.0 / sqrt((double)q), out, prob);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern<K, NT, MINB, VAR>);
    double err = 0;
    if (ref) {
        static double2 h[4096], g[4096];
        cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
        cudaMemcpy(g, ref, sizeof g, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 4096; i++) err = fmax(err, fabs(h[i].x - g[i].x) + fabs(h[i].y - g[i].y));
    }
    const double tf = 8.0 * (double)q * len / (ms * 1e-3) / 1e12;
    printf("%-28s regs=%3d  %8.2f ms  %6.2f TFLOP/s  maxdiff(first 4096)=%.2e  err=%s\n", name, fa.numRegs, ms, tf, err,
           cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    const uint64_t q = 1ull << 24, a0 = 29, stride = 116, len = 144631;
    double2 *out, *ref;
    double *prob;
    cudaMalloc(&out, q * 16);
    cudaMalloc(&ref, q * 16);
    cudaMalloc(&prob, q * 8);
    run<4, 256, 2, 0>("K4 T256 B2 v0 (ref)", q, a0, stride, len, ref, prob, nullptr);
    run<4, 256, 2, 0>("K4 T256 B2 v0", q, a0, stride, len, out, prob, ref);
    run<4, 256, 2, 1>("K4 T256 B2 v1", q, a0, stride, len, out, prob, ref);
    run<2, 256, 4, 0>("K2 T256 B4 v0", q, a0, stride, len, out, prob, ref);
    run<2, 256, 4, 1>("K2 T256 B4 v1", q, a0, stride, len, out, prob, ref);
    run<4, 128, 4, 0>("K4 T128 B4 v0", q, a0, stride, len, out, prob, ref);
    run<4, 256, 3, 0>("K4 T256 B3 v0", q, a0, stride, len, out, prob, ref);
    run<6, 256, 2, 0>("K6 T256 B2 v0", q, a0, stride, len, out, prob, ref);
    run<8, 256, 1, 0>("K8 T256 B1 v0", q, a0, stride, len, out, prob, ref);
    run<8, 128, 2, 0>("K8 T128 B2 v0", q, a0, stride, len, out, prob, ref);
    run<8, 128, 2, 1>("K8 T128 B2 v1", q, a0, stride, len, out, prob, ref);
    run<3, 256, 3, 0>("K3 T256 B3 v0", q, a0, stride, len, out, prob, ref);
    run<1, 256, 8, 0>("K1 T256 B8 v0", q, a0, stride, len, out, prob, ref);
    run<2, 512, 2, 0>("K2 T512 B2 v0", q, a0, stride, len, out, prob, ref);
    double *pref;
    cudaMalloc(&pref, q * 8);
    run<4, 256, 2, 0>("fp64 reference probs", q, a0, stride, len, ref, pref, nullptr);
    run32<4, 256, 2, 256>("fp32 K4 T256 B2 SEG256", q, a0, stride, len, out, prob, pref);
    run32<8, 256, 2, 256>("fp32 K8 T256 B2 SEG256", q, a0, stride, len, out, prob, pref);
    run32<8, 256, 2, 1024>("fp32 K8 T256 B2 SEG1024", q, a0, stride, len, out, prob, pref);
    run32<8, 128, 4, 512>("fp32 K8 T128 B4 SEG512", q, a0, stride, len, out, prob, pref);
    run32<4, 256, 3, 512>("fp32 K4 T256 B3 SEG512", q, a0, stride, len, out, prob, pref);
    return 0;
}
