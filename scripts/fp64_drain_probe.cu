// Throughput of the int8 engine's drain arithmetic on one SM (exploration):
// per (component, output) one accumulator combine (I2F + DADD + DFMA) and per
// output one complex Horner step (4 DFMA), 8 outputs per thread, vs plain
// independent DFMA chains.  Prints FP64-pipe lane-ops per SM clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_drain_probe scripts/fp64_drain_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double combine(int d0, int d1, int d2, int d3)
{
    const uint32_t l = ((uint32_t)d2 << 6) + ((uint32_t)d3 >> 8);
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    return fma((double)d0, 0x1p34, __longlong_as_double((long long)hb) - 0x1p52);
}

__device__ __forceinline__ double combine_noi2f(int d0, int d1, int d2, int d3)
{
    const uint32_t l = ((uint32_t)d2 << 6) + ((uint32_t)d3 >> 8);
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    const double dd0 = __longlong_as_double(0x4338000000000000LL + (long long)d0) - 0x1.8p52;
    return fma(dd0, 0x1p34, __longlong_as_double((long long)hb) - 0x1p52);
}

__device__ __forceinline__ double combine_c64(int d0, int d1, int d2, int d3)
{
    const uint32_t l = ((uint32_t)d2 << 6) + ((uint32_t)d3 >> 8);
    const long long x = ((long long)d0 << 34) + ((long long)(uint32_t)d1 << 20) + (long long)l;
    return (double)x;
}

// one DFMA: 2^47 T ~ D_0 2^34 + (D_1 2^20 + lo) where the second term is the exact
// bit pattern of 2^52 + H minus... folded into the Horner addend (probe only)
__device__ __forceinline__ double combine_min(int d0, int d1, int d2, int d3)
{
    const uint32_t l = ((uint32_t)d2 << 6) + ((uint32_t)d3 >> 8);
    unsigned long long hb;
    asm("{\n\t.reg .b64 a;\n\tmov.b64 a, {%1, %2};\n\tmad.wide.u32 %0, %3, 1048576, a;\n\t}"
        : "=l"(hb)
        : "r"(l), "r"(0x43300000u), "r"((uint32_t)d1));
    return __longlong_as_double((long long)hb);
}

template <int MODE>
__global__ void probe(int iters, double *out, long long *cyc)
{
    int acc[8][8];
    for (int o = 0; o < 8; o++)
        for (int i = 0; i < 8; i++) acc[o][i] = (threadIdx.x * 131 + o * 17 + i * 7) & 0xFFFFF;
    double hr[8], hi[8];
    for (int i = 0; i < 8; i++) hr[i] = hi[i] = 1e-3 * i;
    const double sr = 0.6, si = 0.8;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE != 1) {
                double tr, ti;
                if (MODE == 0) {
                    tr = combine(acc[0][i], acc[1][i], acc[2][i], acc[3][i]);
                    ti = combine(acc[4][i], acc[5][i], acc[6][i], acc[7][i]);
                } else if (MODE == 2) {
                    tr = combine_noi2f(acc[0][i], acc[1][i], acc[2][i], acc[3][i]);
                    ti = combine_noi2f(acc[4][i], acc[5][i], acc[6][i], acc[7][i]);
                } else if (MODE == 3) {
                    tr = combine_c64(acc[0][i], acc[1][i], acc[2][i], acc[3][i]);
                    ti = combine_c64(acc[4][i], acc[5][i], acc[6][i], acc[7][i]);
                } else {
                    tr = combine_min(acc[0][i], acc[1][i], acc[2][i], acc[3][i]);
                    ti = combine_min(acc[4][i], acc[5][i], acc[6][i], acc[7][i]);
                }
                const double nr = fma(hr[i], sr, fma(-hi[i], si, tr));
                const double ni = fma(hr[i], si, fma(hi[i], sr, ti));
                hr[i] = nr;
                hi[i] = ni;
            } else {
                // 10 independent-ish DFMA per output (the same FP64 op count, no I2F/DADD)
                hr[i] = fma(hr[i], sr, fma(-hi[i], si, fma(hr[i], 1.0000001, 1e-9)));
                hi[i] = fma(hr[i], si, fma(hi[i], sr, fma(hi[i], 1.0000001, 1e-9)));
                hr[i] = fma(hr[i], 0.999, fma(hi[i], 1e-7, fma(hr[i], 1e-7, 1e-9)));
                hi[i] = fma(hi[i], 0.999, 1e-9);
            }
        }
#pragma unroll
        for (int o = 0; o < 8; o++)
#pragma unroll
            for (int i = 0; i < 8; i++) acc[o][i] ^= it;
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; i++) s += hr[i] + hi[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main()
{
    double *d;
    long long *c;
    cudaMalloc(&d, 1 << 20);
    cudaMalloc(&c, 8 * 148);
    const char *names[5] = {"drain", "dfma", "noi2f", "conv64", "nocvt"};
    for (int mode = 0; mode < 5; mode++)
        for (int warps : {8, 12, 16}) {
            const int iters = 2000;
            if (mode == 0) probe<0><<<148, warps * 32>>>(iters, d, c);
            if (mode == 1) probe<1><<<148, warps * 32>>>(iters, d, c);
            if (mode == 2) probe<2><<<148, warps * 32>>>(iters, d, c);
            if (mode == 3) probe<3><<<148, warps * 32>>>(iters, d, c);
            if (mode == 4) probe<4><<<148, warps * 32>>>(iters, d, c);
            cudaDeviceSynchronize();
            long long cyc;
            cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
            // FP64-pipe lane-ops per iteration per thread: mode 0: 8 x (2 x (I2F + DADD + DFMA) + 4 DFMA) = 80
            const double ops = 80.0 * iters * warps * 32;
            printf("mode %s warps %2d: %.1f cycles/iter  %.1f FP64 lane-ops/clk/SM  (%s)\n",
                   names[mode], warps, (double)cyc / iters, ops / cyc, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
