// Gate-level QFT primitives (the reference's circuit engine, qft.py:164-231):
// a Hadamard on one qubit, a controlled phase between two qubits and the
// bit-reversal permutation.  circuit_qft (qft.py) builds the QFT from these,
// so the "circuit" engine is an independent gate-level cross-check of the
// direct-DFT kernels rather than another call into them.
//
// Every operation is elementwise on a complex128 vector (HBM-bound: 32 B
// per pair for the Hadamard, 16 B per selected element for the phase, 32 B
// per element for the permutation) and reproduces numpy's arithmetic
// bit for bit: every operation is an explicit round-to-nearest intrinsic,
// the complex multiply is numpy's fused form (verified against the reference's
// own outputs), complex-by-real products are that full complex multiply
// against (s + 0j) as numpy performs it, and the phase factor
// (cos, sin) is computed on the host by numpy exactly as qft.py:193 does.
#include "shb_internal.cuh"

namespace shb {

constexpr int GATE_THREADS = 256;

__device__ __forceinline__ double2 cmul_exact(double2 a, double br, double bi)
{
    // numpy's complex128 multiply loop (SIMD, fused): (fma(ar, br, -(ai bi)),
    // fma(ar, bi, ai br)) -- pinned bitwise by tests/golden/gates.npz
    return make_double2(__fma_rn(a.x, br, -__dmul_rn(a.y, bi)), __fma_rn(a.x, bi, __dmul_rn(a.y, br)));
}

// t with a 1 inserted at bit position p (the bits from p upwards move up one)
__device__ __forceinline__ uint64_t insert_one(uint64_t t, int p)
{
    const uint64_t low = t & ((1ull << p) - 1);
    return ((t ^ low) << 1) | (1ull << p) | low;
}

// qft.py:164-177: view (q >> (b+1), 2, 1 << b); (u, v) -> ((u+v) s, (u-v) s)
__global__ void __launch_bounds__(GATE_THREADS)
    hadamard_kernel(double2 *__restrict__ a, uint64_t half, int b, double s)
{
    const uint64_t lo_mask = (1ull << b) - 1;
    for (uint64_t t = (uint64_t)blockIdx.x * GATE_THREADS + threadIdx.x; t < half;
         t += (uint64_t)gridDim.x * GATE_THREADS) {
        const uint64_t i0 = ((t & ~lo_mask) << 1) | (t & lo_mask);
        const uint64_t i1 = i0 | (1ull << b);
        const double2 u = a[i0], v = a[i1];
        a[i0] = cmul_exact(make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y)), s, 0.0);
        a[i1] = cmul_exact(make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y)), s, 0.0);
    }
}

// qft.py:180-196: amplitudes whose index has both bits set *= e^{i angle}.
// Thread t visits the q/4 indices with both bits set (the other two bits
// of the index are spread around them).
__global__ void __launch_bounds__(GATE_THREADS)
    cphase_kernel(double2 *__restrict__ a, uint64_t quarter, int lo_bit, int hi_bit, double er, double ei)
{
    for (uint64_t t = (uint64_t)blockIdx.x * GATE_THREADS + threadIdx.x; t < quarter;
         t += (uint64_t)gridDim.x * GATE_THREADS) {
        const uint64_t i = insert_one(insert_one(t, lo_bit), hi_bit);
        a[i] = cmul_exact(a[i], er, ei);
    }
}

// qft.py:199-212: out[reverse_bits_w(i)] = in[i]
__global__ void __launch_bounds__(GATE_THREADS)
    bitrev_kernel(const double2 *__restrict__ in, double2 *__restrict__ out, uint64_t q, int w)
{
    for (uint64_t i = (uint64_t)blockIdx.x * GATE_THREADS + threadIdx.x; i < q;
         i += (uint64_t)gridDim.x * GATE_THREADS)
        out[__brevll(i) >> (64 - w)] = in[i];
}

static int width_of(uint64_t q)
{
    if (q < 2 || (q & (q - 1))) return -1;
    return 63 - __builtin_clzll(q);
}

static unsigned gate_grid(uint64_t items)
{
    const uint64_t want = (items + GATE_THREADS - 1) / GATE_THREADS;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    return (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace shb

using namespace shb;

extern "C" {

int shb_apply_hadamard(double *state, uint64_t q, int qubit, void *stream)
{
    const int w = width_of(q);
    if (!state) return set_error(SHB_EINVAL, "null state");
    if (w < 1) return set_error(SHB_EINVAL, "q must be a power of two >= 2, got %llu", (unsigned long long)q);
    if (qubit < 0 || qubit >= w) return set_error(SHB_EINVAL, "qubit index %d out of range for w=%d", qubit, w);
    const double s = 1.0 / sqrt(2.0);  // qft.py:174: inv_sqrt2 = 1.0 / math.sqrt(2.0)
    hadamard_kernel<<<gate_grid(q / 2), GATE_THREADS, 0, as_stream(stream)>>>((double2 *)state, q / 2, qubit, s);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

int shb_apply_controlled_phase(double *state, uint64_t q, int control, int target, double phase_re,
                               double phase_im, void *stream)
{
    const int w = width_of(q);
    if (!state) return set_error(SHB_EINVAL, "null state");
    if (w < 1) return set_error(SHB_EINVAL, "q must be a power of two >= 2, got %llu", (unsigned long long)q);
    if (control == target) return set_error(SHB_EINVAL, "control and target must differ");
    if (control < 0 || control >= w) return set_error(SHB_EINVAL, "qubit index %d out of range for w=%d", control, w);
    if (target < 0 || target >= w) return set_error(SHB_EINVAL, "qubit index %d out of range for w=%d", target, w);
    const int lo = control < target ? control : target, hi = control < target ? target : control;
    cphase_kernel<<<gate_grid(q / 4), GATE_THREADS, 0, as_stream(stream)>>>((double2 *)state, q / 4, lo, hi,
                                                                           phase_re, phase_im);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

int shb_bit_reverse_permute(const double *in, double *out, uint64_t q, void *stream)
{
    const int w = width_of(q);
    if (!in || !out) return set_error(SHB_EINVAL, "null buffer");
    if (in == out) return set_error(SHB_EINVAL, "bit_reverse_permute is out of place");
    if (w < 1) return set_error(SHB_EINVAL, "q must be a power of two >= 2, got %llu", (unsigned long long)q);
    bitrev_kernel<<<gate_grid(q), GATE_THREADS, 0, as_stream(stream)>>>((const double2 *)in, (double2 *)out, q, w);
    SHB_LAUNCHED();
    SHB_TRY_CUDA(cudaGetLastError());
    return SHB_OK;
}

}  // extern "C"
