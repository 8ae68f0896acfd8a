// Exploration (not product): one tcgen05.mma kind::f16 (bf16 x bf16 -> f32),
// M=128, N=64, K=16*KS, A and B K-major in shared memory without swizzle,
// D in TMEM, read back with tcgen05.ld 32x32b -- validates the descriptor
// encodings against a host reference before they are used in a kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tc05_probe scripts/tc05_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr int M = 128, N = 64, KS = 4, K = 16 * KS;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// core matrix = 8 rows x 16 bytes, stored row after row (128 B).
// element (row, k) of a K-major operand lives at
//   (row / 8) * SBO + (k / 8) * LBO + (row % 8) * 16 + (k % 8) * 2
__device__ __forceinline__ uint32_t kmajor_off(int row, int k, int lbo, int sbo)
{
    return (row >> 3) * sbo + (k >> 3) * lbo + (row & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo & 0x3FFFF) >> 4) << 16;
    d |= (uint64_t)((sbo & 0x3FFFF) >> 4) << 32;
    d |= (uint64_t)1 << 46;  // version (sm_100)
    // base offset 0, lbo mode 0, swizzle none (bits 61-63 = 0)
    return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16_f32(int m, int n)
{
    return (1u << 4)            // D format F32
         | (1u << 7)            // A BF16
         | (1u << 10)           // B BF16
         | (0u << 15)           // A K-major
         | (0u << 16)           // B K-major
         | ((uint32_t)(n >> 3) << 17)
         | ((uint32_t)(m >> 4) << 24);
}

// physical layout: k-core matrices adjacent (pk = 128 B), 8-row groups every
// pr bytes; the descriptor gets (d_lbo, d_sbo) -- two hypotheses are tried
__global__ void __launch_bounds__(128, 1) probe(const float *A, const float *B, float *D, int pk, int pr, int d_lbo,
                                               int d_sbo, int a_in_tmem)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __nv_bfloat16 *sa = reinterpret_cast<__nv_bfloat16 *>(sm);
    __nv_bfloat16 *sb = reinterpret_cast<__nv_bfloat16 *>(sm + 64 * 1024);
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < M * K; i += 128) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<__nv_bfloat16 *>(reinterpret_cast<unsigned char *>(sa) + kmajor_off(r, k, pk, pr)) =
            __float2bfloat16_rn(A[i]);
    }
    for (int i = tid; i < N * K; i += 128) {
        const int n = i / K, k = i % K;
        *reinterpret_cast<__nv_bfloat16 *>(reinterpret_cast<unsigned char *>(sb) + kmajor_off(n, k, pk, pr)) =
            __float2bfloat16_rn(B[i]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t id = idesc_bf16_f32(M, N);
        if (a_in_tmem) {  // A -> TMEM columns [128, 128 + 8 KS): one 128x256b copy per k-step
            for (int s = 0; s < KS; s++) {
                const uint64_t da = sdesc(smem_u32(sa) + s * 2 * pk, d_lbo, d_sbo);
                asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 128 + 8 * s), "l"(da));
            }
        }
        for (int s = 0; s < KS; s++) {
            const uint64_t da = sdesc(smem_u32(sa) + s * 2 * pk, d_lbo, d_sbo);
            const uint64_t db = sdesc(smem_u32(sb) + s * 2 * pk, d_lbo, d_sbo);
            const uint32_t acc = s > 0;
            if (a_in_tmem)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                             ::"r"(tmem), "r"(tmem + 128 + 8 * s), "l"(db), "r"(id), "r"(acc));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(id), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        for (long spin = 0; !done; spin++) {
            if (spin > (1l << 26)) asm volatile("trap;");
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w reads lanes 32w..32w+31, 8 columns at a time
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; j++) D[tid * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main()
{
    std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N, 0.f);
    srand(1);
    auto rb = [] { return __bfloat162float(__float2bfloat16_rn((rand() % 2001 - 1000) / 1000.f)); };
    for (auto &x : A) x = rb();
    for (auto &x : B) x = rb();
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double s = 0;
            for (int k = 0; k < K; k++) s += (double)A[i * K + k] * B[j * K + k];
            R[i * N + j] = (float)s;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    const int pk = 128, pr = (K / 8) * 128;
    const int hyp[2][2] = {{pk, pr}, {pk, pr}};  // run 0: A from smem; run 1: A via tcgen05.cp into TMEM
    for (int h = 0; h < 2; h++) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, 96 * 1024>>>(dA, dB, dD, pk, pr, hyp[h][0], hyp[h][1], h);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int i = 0; i < M * N; i++) maxerr = fmax(maxerr, fabs(D[i] - R[i]));
        printf("a_in_tmem=%d LBO=%d SBO=%d: %s  max|D-R| = %g  D[0]=%g R[0]=%g D[77]=%g R[77]=%g\n", h, hyp[h][0], hyp[h][1],
               cudaGetErrorString(e), maxerr, D[0], R[0], D[77], R[77]);
        if (e != cudaSuccess) break;
    }
    return 0;
}
