// Exploration (not product): tcgen05.mma kind::f16 (bf16 -> f32) issue rate
// for M = 128 and N in {64, 128, 256}, A from shared memory or TMEM, B from
// shared memory; one issuing thread per SM, one accumulator.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tc05_rate_probe scripts/tc05_rate_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr)
{
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n)
{
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N, bool ATMEM>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long *cycles)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < 48 * 1024 / 4; i += 128) reinterpret_cast<uint32_t *>(sm)[i] = 0x3F803F80u;
    asm volatile("fence.proxy.async.shared::cta;");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t t = tbase;
    if (tid == 0) {
        const uint32_t id = idesc(128, N);
        const uint64_t da = sdesc(smem_u32(sm)), db = sdesc(smem_u32(sm + 16384));
        const uint32_t at = t + 256 + 0;
        const long long t0 = clock64();
        for (int i = 0; i < iters; i++) {
            if (ATMEM)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(t), "r"(at), "l"(db), "r"(id), "r"(1));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(t), "l"(da), "l"(db), "r"(id), "r"(1));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
        const long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}

template <int N, bool ATMEM>
void run(int sms)
{
    unsigned long long *dc, hc;
    cudaMalloc(&dc, 8);
    const int iters = 20000;
    cudaFuncSetAttribute(rate<N, ATMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    rate<N, ATMEM><<<sms, 128, 64 * 1024>>>(100, dc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate<N, ATMEM><<<sms, 128, 64 * 1024>>>(iters, dc);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&hc, dc, 8, cudaMemcpyDeviceToHost);
    const double macs = 128.0 * N * 16 * iters;
    printf("N=%3d A in %s: %6.1f cyc/MMA  %7.0f MAC/clk/SM  %7.1f TFLOP/s (%s)\n", N, ATMEM ? "TMEM" : "smem",
           (double)hc / iters, macs / hc, 2 * macs * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(e));
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, false>(sms);
    run<64, true>(sms);
    run<128, false>(sms);
    run<128, true>(sms);
    run<256, false>(sms);
    run<256, true>(sms);
    return 0;
}
