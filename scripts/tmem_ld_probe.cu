// Exploration (not product): tcgen05.ld (TMEM -> registers) throughput per SM
// on this B200, as a function of warps per CTA and load width -- the drain
// rate that bounds dft_i8_uniform_kernel (8 int32 accumulators per output and
// row-block).  One CTA per SM, 512 TMEM columns allocated, every warp reads
// its lane quarter repeatedly; bytes/clk/SM from clock64 over the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tmem_ld_probe scripts/tmem_ld_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ uint32_t ldx(uint32_t taddr)
{
    uint32_t r[32];
    if (X == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    } else if (X == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < X; i++) s ^= r[i];
    return s;
}

template <int X>
__global__ void probe(unsigned long long *cycles, uint32_t *sink, int iters)
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
    const uint32_t t = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t s = 0;
    __syncthreads();
    const unsigned long long c0 = clock64();
    for (int it = 0; it < iters; it++)
        for (int col = 0; col < 512; col += X) s ^= ldx<X>(t + col);
    __syncthreads();
    const unsigned long long c1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
    if (s == 0x12345678u) sink[0] = s;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int X>
void run(int sms, int warps)
{
    unsigned long long *cyc;
    uint32_t *sink;
    cudaMalloc(&cyc, sms * sizeof(unsigned long long));
    cudaMalloc(&sink, 4);
    const int iters = 64;
    probe<X><<<sms, 32 * warps>>>(cyc, sink, 2);
    probe<X><<<sms, 32 * warps>>>(cyc, sink, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1024];
    cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; i++) mean += (double)h[i] / sms;
    // bytes per CTA: warps x 32 lanes x 512 columns x 4 B x iters
    const double bytes = (double)warps * 32 * 512 * 4 * iters;
    printf("x%-2d warps %2d: %8.1f B/clk/SM  (%.0f cycles, %s)\n", X, warps, bytes / mean, mean, cudaGetErrorString(e));
    cudaFree(cyc);
    cudaFree(sink);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 16}) {
        run<8>(sms, w);
        run<16>(sms, w);
        run<32>(sms, w);
    }
    return 0;
}
