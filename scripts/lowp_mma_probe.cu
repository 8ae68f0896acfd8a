// Exploration (not product): legacy warp-level mma.sync throughput on B200 for
// the FP32 fast-path candidates: TF32 m16n8k8 and BF16 m16n8k16 (FP32
// accumulate), vs FP64 DMMA m8n8k4.  One value per chain, NCH chains per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/lowp_mma_probe scripts/lowp_mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int KIND, int NCH>
__global__ void probe(float *out, int iters, uint32_t a, uint32_t b)
{
    float d[NCH][4];
#pragma unroll
    for (int i = 0; i < NCH; i++) d[i][0] = d[i][1] = d[i][2] = d[i][3] = threadIdx.x * 1e-6f + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < NCH; i++) {
            if (KIND == 0) mma_tf32(d[i], a, a ^ i, a, a, b, b ^ i);
            else mma_bf16(d[i], a, a ^ i, a, a, b, b ^ i);
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
    if (s == 1.2345f) out[0] = s;
}

template <int KIND, int NCH>
void run(float *sink, int sms, int warps_per_sm)
{
    const int iters = (1 << 16) / NCH;
    const int wpc = 4;
    const int grid = sms * (warps_per_sm / wpc);
    probe<KIND, NCH><<<grid, 32 * wpc>>>(sink, 16, 0x3f800000u, 0x3f800000u);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<KIND, NCH><<<grid, 32 * wpc>>>(sink, iters, 0x3f800000u, 0x3f800000u);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = KIND == 0 ? 16.0 * 8 * 8 : 16.0 * 8 * 16;
    const double flops = (double)grid * wpc * iters * NCH * macs * 2;
    printf("%s chains/warp %2d warps/SM %2d  %8.1f TFLOP/s  (%s)\n", KIND == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16",
           NCH, warps_per_sm, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *sink;
    cudaMalloc(&sink, 8);
    for (int w : {8, 16, 32}) {
        run<0, 2>(sink, sms, w);
        run<0, 4>(sink, sms, w);
        run<0, 8>(sink, sms, w);
        run<1, 2>(sink, sms, w);
        run<1, 4>(sink, sms, w);
        run<1, 8>(sink, sms, w);
    }
    return 0;
}
