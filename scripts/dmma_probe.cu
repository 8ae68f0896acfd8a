// Exploration (not product): FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput
// on sm_100a, alone and concurrently with DFMA chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/dmma_probe scripts/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>  // 0: DMMA only, 1: DFMA only, 2: both in every warp
__global__ void __launch_bounds__(256) probe(double *out, int iters, double a, double b)
{
    double d[8][2], x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { d[i][0] = d[i][1] = threadIdx.x * 1e-6 + i; x[i] = i * 1e-3; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE != 1) dmma(d[i][0], d[i][1], a, b);
            if (MODE != 0) { x[i] = fma(x[i], a, b); x[i] = fma(x[i], a, b); }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) s += d[i][0] + d[i][1] + x[i];
    if (s == 1.2345) out[0] = s;
}

template <int MODE>
void run(const char *name, double *sink, int sms)
{
    const int grid = sms * 4, iters = 1 << 14;
    probe<MODE><<<grid, 256>>>(sink, 16, 0.999, 1e-9);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<MODE><<<grid, 256>>>(sink, iters, 0.999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warps = grid * 8.0;
    const double dmma_flops = (MODE != 1) ? warps * iters * 8 * 512.0 : 0;   // 8x8x4 MACs x2 per warp-mma
    const double dfma_flops = (MODE != 0) ? grid * 256.0 * iters * 8 * 2 * 2.0 : 0;
    printf("%-18s %8.2f ms  DMMA %6.2f TF  DFMA %6.2f TF  total %6.2f TF  (%s)\n", name, ms,
           dmma_flops / ms / 1e9, dfma_flops / ms / 1e9, (dmma_flops + dfma_flops) / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *sink; cudaMalloc(&sink, 8);
    run<0>("DMMA only", sink, sms);
    run<1>("DFMA only", sink, sms);
    run<2>("DMMA + DFMA", sink, sms);
    return 0;
}
