// Internal helpers shared by the shorb200 translation units (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/shorb200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "shorb200 is written for sm_100a (B200) only"
#endif

namespace shb {

// ------------------------------------------------------------ error state
int set_error(int code, const char *fmt, ...);
int check_cuda(cudaError_t e, const char *what);

#define SHB_TRY_CUDA(expr)                                      \
    do {                                                        \
        cudaError_t _e = (expr);                                \
        if (_e != cudaSuccess) return ::shb::check_cuda(_e, #expr); \
    } while (0)

#define SHB_TRY(expr)              \
    do {                           \
        int _s = (expr);           \
        if (_s != SHB_OK) return _s; \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Count of kernels this library launched (reported by bench.py as gpu_launches).
void note_launch(unsigned n = 1);
#define SHB_LAUNCHED() ::shb::note_launch(1)

// Stream-ordered scratch allocation (cudaMallocAsync pool).
struct Scratch {
    void *ptr = nullptr;
    cudaStream_t st = nullptr;
    ~Scratch() {
        if (ptr) cudaFreeAsync(ptr, st);
    }
};
int scratch_alloc(Scratch &s, size_t bytes, cudaStream_t st);

// FP32 uniform-comb DFT on tcgen05 (dft_tc05.cu); arguments as shb_dft_uniform,
// already validated.  Block sums in slots of `slot_outputs` outputs.
int tc05_dft_uniform(uint64_t length, uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin,
                     uint64_t c_count, double out_re, double out_im, double *d_out, double *d_prob,
                     double *d_block_sums, uint64_t slot_outputs, cudaStream_t st);

// FP64-accurate uniform-comb DFT on the int8 tensor cores (dft_i8.cu);
// arguments as shb_dft_uniform, already validated.
int i8_dft_uniform(uint64_t length, uint64_t a0, uint64_t stride, uint64_t q, uint64_t c_begin, uint64_t c_count,
                   double out_re, double out_im, double *d_out, double *d_prob, double *d_block_sums,
                   uint64_t slot_outputs, cudaStream_t st);

// ------------------------------------------------------------ integer math
__host__ __device__ inline uint64_t gcd_u64(uint64_t a, uint64_t b)
{
    if (a == 0) return b;
    if (b == 0) return a;
#ifdef __CUDA_ARCH__
    const int shift = __ffsll((long long)(a | b)) - 1;
    a >>= __ffsll((long long)a) - 1;
    do {
        b >>= __ffsll((long long)b) - 1;
        if (a > b) {
            uint64_t t = a;
            a = b;
            b = t;
        }
        b -= a;
    } while (b != 0);
    return a << shift;
#else
    while (b) {
        uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
#endif
}

// ------------------------------------------------ mbarrier / TMA bulk copy
__device__ inline uint32_t smem_addr(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ inline void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ inline void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ inline void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ inline void mbar_wait(uint64_t *bar, uint32_t phase)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(phase)
        : "memory");
}

__device__ inline void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// 1-D bulk copy global -> shared through the TMA unit (UBLKCP), completion
// signalled on `bar` with complete_tx.  bytes % 16 == 0, 16-B aligned.
__device__ inline void tma_bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                   uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ------------------------------------------------------------ block scans
template <int NT>
__device__ inline uint64_t block_exclusive_scan_u64(uint64_t v, uint64_t *warp_tmp, uint64_t &total)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t w = (lane < NT / 32) ? warp_tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) warp_tmp[lane] = w;
    }
    __syncthreads();
    total = warp_tmp[NT / 32 - 1];
    const uint64_t before = (wid > 0 ? warp_tmp[wid - 1] : 0) + x - v;
    __syncthreads();
    return before;
}

}  // namespace shb
