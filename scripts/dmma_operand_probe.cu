// Exploration (not product): does DMMA throughput depend on the B operand
// changing from one instruction to the next (as G[ks] does in the DFT kernel)?
// Variant 0: constant A and B (the dmma_chains_probe setting).  Variant 1: B
// cycles through KS registers, 2 accumulator chains (Re/Im) as in the real-A
// DFT kernel.  Variant 2: as 1 plus a 4-DFMA fold of each chain every KS steps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/dmma_operand_probe scripts/dmma_operand_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int VAR, int KS>
__global__ void __launch_bounds__(256, 1) probe(double *out, int iters, double a, double b0)
{
    double g[KS], h[KS];
#pragma unroll
    for (int i = 0; i < KS; i++) {
        g[i] = b0 + i * 1e-3 + threadIdx.x * 1e-9;
        h[i] = b0 - i * 1e-3;
    }
    double dr0 = 0, dr1 = 0, di0 = 0, di1 = 0, hr = 0, hi = 0;
    const double ur = 0.999, ui = 0.001;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
            if (VAR == 0) {
                dmma(dr0, dr1, a, b0);
                dmma(di0, di1, a, b0);
            } else {
                dmma(dr0, dr1, a, g[ks]);
                dmma(di0, di1, a, h[ks]);
            }
        }
        if (VAR == 2) {
            const double nr = fma(hr, ur, fma(-hi, ui, dr0 + dr1));
            const double ni = fma(hr, ui, fma(hi, ur, di0 + di1));
            hr = nr;
            hi = ni;
            dr0 = dr1 = di0 = di1 = 0;
        }
    }
    const double s = dr0 + dr1 + di0 + di1 + hr + hi;
    if (s == 1.2345) out[0] = s;
}

template <int VAR, int KS>
void run(double *sink, int sms, int ctas_per_sm)
{
    const int iters = (1 << 16) / KS;
    const int grid = sms * ctas_per_sm;
    probe<VAR, KS><<<grid, 256>>>(sink, 16, 1.0, 0.5);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<VAR, KS><<<grid, 256>>>(sink, iters, 1.0, 0.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)grid * 256 / 32 * iters * KS * 2 * 512.0;
    printf("variant %d KS %3d  %6.2f TF  (%s)\n", VAR, KS, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *sink;
    cudaMalloc(&sink, 8);
    run<0, 32>(sink, sms, 1);
    run<1, 32>(sink, sms, 1);
    run<2, 32>(sink, sms, 1);
    run<1, 16>(sink, sms, 1);
    run<2, 16>(sink, sms, 1);
    run<2, 64>(sink, sms, 1);
    return 0;
}
