// Exploration (not product): FP64 DMMA (mma.sync m8n8k4 f64) throughput as a
// function of independent accumulator chains per warp and warps per SM --
// how much ILP/TLP the DMMA engine needs to reach the FP64 datapath peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/dmma_chains_probe scripts/dmma_chains_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NCH>
__global__ void probe(double *out, int iters, double a, double b)
{
    double d[NCH][2];
#pragma unroll
    for (int i = 0; i < NCH; i++) d[i][0] = d[i][1] = threadIdx.x * 1e-6 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < NCH; i++) dmma(d[i][0], d[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += d[i][0] + d[i][1];
    if (s == 1.2345) out[0] = s;
}

template <int NCH>
void run(double *sink, int sms, int warps_per_sm)
{
    const int iters = (1 << 16) / NCH;
    const int wpc = 4;  // warps per CTA
    const int grid = sms * (warps_per_sm / wpc);
    probe<NCH><<<grid, 32 * wpc>>>(sink, 16, 0.999, 1e-9);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<NCH><<<grid, 32 * wpc>>>(sink, iters, 0.999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)grid * wpc * iters * NCH * 512.0;
    printf("chains/warp %2d  warps/SM %2d  chains/SMSP %3d  %7.2f TF  (%s)\n", NCH, warps_per_sm,
           NCH * warps_per_sm / 4, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *sink;
    cudaMalloc(&sink, 8);
    for (int w : {4, 8, 12, 16, 32}) {
        run<1>(sink, sms, w);
        run<2>(sink, sms, w);
        run<4>(sink, sms, w);
        run<8>(sink, sms, w);
    }
    return 0;
}
