// Exploration (not product): tcgen05.ld throughput of the int8 DFT drain's
// access pattern -- bursts of 8 x (32x32b.x8) loads whose columns are STRIDE
// apart (the 8 digit-pair accumulators of one row-block group), one
// wait::ld per burst -- against consecutive columns.  8 warps per CTA, one
// CTA per SM, bytes/clk/SM from clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmem_ld_burst_probe scripts/tmem_ld_burst_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t *r)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}

__global__ void probe(unsigned long long *cycles, uint32_t *sink, int iters, int stride, int inner)
{
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * (uint32_t)inner;
    uint32_t s = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; it++)
        for (int ch = 0; ch < inner; ch += 8) {
            uint32_t r[8][8];
#pragma unroll
            for (int p = 0; p < 8; p++) ld8(t + ((p * stride + ch) & 511), r[p]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int p = 0; p < 8; p++)
#pragma unroll
                for (int e = 0; e < 8; e++) s ^= r[p][e];
        }
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
    if (s == 0x12345678u) sink[0] = s;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *cyc, h[1024];
    uint32_t *sink;
    cudaMalloc(&cyc, sms * sizeof(unsigned long long));
    cudaMalloc(&sink, 4);
    const int iters = 256;
    // (stride, inner): inner = columns each warp walks per accumulator (kernel: 32 of 64 row-blocks)
    const int cases[][2] = {{64, 32}, {8, 32}, {56, 24}, {48, 24}, {72, 32}, {65, 32}, {68, 32}, {80, 32}, {96, 32}};
    for (auto &c : cases) {
        probe<<<sms, 256>>>(cyc, sink, 2, c[0], c[1]);
        probe<<<sms, 256>>>(cyc, sink, iters, c[0], c[1]);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double mean = 0;
        for (int i = 0; i < sms; i++) mean += (double)h[i] / sms;
        const double bytes = 8.0 * 32 * 8 * 4 * (c[1] / 8) * 8 * iters;  // warps x lanes x cols x B x bursts x loads
        printf("stride %3d inner %2d: %7.1f B/clk/SM  (%.0f cycles per 256 KB, %s)\n", c[0], c[1], bytes / mean,
               262144.0 / (bytes / mean), cudaGetErrorString(e));
    }
    return 0;
}
