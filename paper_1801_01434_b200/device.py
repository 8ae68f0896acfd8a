"""Device-resident register parts and thin wrappers over the C ABI.

The reference keeps the register as two numpy arrays (qstate.py:36-42).  At
q = 2^30 those are 16 GiB + 8 GiB and every stage would round-trip them
through host memory, so the B200 path keeps them on the GPU and exposes
them through ``DeviceVector``: an array-like whose ``__array__`` copies to
host on demand.  Code written against the reference (``np.asarray(reg.amplitudes)``,
``np.abs(spectrum) ** 2``, indexing) keeps working; the pipeline itself never
materialises anything on the host.

Device memory comes from torch (caching allocator, current stream); all math
is in libshorb200.so.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as nat


# ----------------------------------------------------------------- op wrappers

def _t():
    return nat.require_cuda()


def _stream():
    return ctypes.c_void_p(nat.stream_ptr())


def _vp(tensor_or_int):
    if tensor_or_int is None:
        return ctypes.c_void_p(0)
    if isinstance(tensor_or_int, int):
        return ctypes.c_void_p(tensor_or_int)
    return ctypes.c_void_p(int(tensor_or_int.data_ptr()))


def modexp(x: int, n: int, count: int, a_begin: int = 0):
    """residues[i] = x^(a_begin+i) mod n as a uint32 device tensor (int32 storage)."""
    t = _t()
    res = t.empty(count, dtype=t.int32, device="cuda")
    nat.check(nat.load().shb_modexp(_vp(res), a_begin, count, x, n, _stream()), "modexp")
    return res


def class_counts(res, ncls: int, out=None):
    t = _t()
    counts = out if out is not None else t.zeros(ncls, dtype=t.int64, device="cuda")
    nat.check(nat.load().shb_class_counts(_vp(res), res.numel(), _vp(counts), ncls, _stream()),
              "class_counts")
    return counts


def compact_eq(res, k: int, a_begin: int = 0, capacity: int | None = None, expected: int | None = None):
    """Ascending indices a_begin+i with res[i] == k (device int64 tensor).

    `expected` (the class count, when the caller has it) sizes the output
    directly and skips the counting probe."""
    t = _t()
    lib = nat.load()
    m = ctypes.c_uint64(0)
    if expected is not None:
        sup = t.empty(max(expected, 1), dtype=t.int64, device="cuda")
        nat.check(lib.shb_compact_eq(_vp(res), res.numel(), k & 0xFFFFFFFF, a_begin, _vp(sup), expected,
                                     ctypes.byref(m), _stream()), "compact_eq")
        if int(m.value) != expected:
            raise RuntimeError(f"compaction found {m.value} indices, class count says {expected}")
        return sup[:expected]
    cap = res.numel() if capacity is None else capacity
    # count first (cheap) so the output is exactly sized
    probe = t.empty(1, dtype=t.int64, device="cuda")
    rc = lib.shb_compact_eq(_vp(res), res.numel(), k & 0xFFFFFFFF, a_begin, _vp(probe), 0,
                            ctypes.byref(m), _stream())
    if rc not in (nat.SHB_OK, nat.SHB_ERANGE):
        nat.check(rc, "compact_eq")
    M = int(m.value)
    if M > cap:
        raise ValueError(f"support of {M} entries exceeds capacity {cap}")
    sup = t.empty(max(M, 1), dtype=t.int64, device="cuda")
    if M:
        nat.check(lib.shb_compact_eq(_vp(res), res.numel(), k & 0xFFFFFFFF, a_begin, _vp(sup), M,
                                     ctypes.byref(m), _stream()), "compact_eq")
    return sup[:M]


def support_progression(support) -> tuple[int, int, int]:
    a0, st, ln = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    nat.check(nat.load().shb_support_progression(_vp(support), support.numel(), ctypes.byref(a0),
                                                 ctypes.byref(st), ctypes.byref(ln), _stream()),
              "support_progression")
    return int(a0.value), int(st.value), int(ln.value)


def state_progression(state) -> tuple[int, int, int]:
    """Progression of nonzeros of a complex128 device vector (float64 [2q] storage)."""
    a0, st, ln = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    nat.check(nat.load().shb_state_progression(_vp(state), state.numel() // 2, ctypes.byref(a0),
                                               ctypes.byref(st), ctypes.byref(ln), _stream()),
              "state_progression")
    return int(a0.value), int(st.value), int(ln.value)


def gather_progression(state, a0: int, stride: int, length: int):
    t = _t()
    amps = t.empty(2 * max(length, 1), dtype=t.float64, device="cuda")
    nat.check(nat.load().shb_gather_progression(_vp(state), a0, stride, length, _vp(amps), _stream()),
              "gather_progression")
    return amps


def progression_uniform(amps, length: int):
    """The common amplitude if all progression amplitudes are equal, else None."""
    if length == 0:
        return None
    u = ctypes.c_int(0)
    re, im = ctypes.c_double(), ctypes.c_double()
    nat.check(nat.load().shb_progression_is_uniform(_vp(amps), length, ctypes.byref(u), ctypes.byref(re),
                                                    ctypes.byref(im), _stream()), "progression_is_uniform")
    return complex(re.value, im.value) if u.value else None


def progression_kind(amps, length: int):
    """(uniform amplitude or None, all imaginary parts zero) of a progression."""
    if length == 0:
        return None, True
    u, real = ctypes.c_int(0), ctypes.c_int(0)
    re, im = ctypes.c_double(), ctypes.c_double()
    nat.check(nat.load().shb_progression_kind(_vp(amps), length, ctypes.byref(u), ctypes.byref(real),
                                              ctypes.byref(re), ctypes.byref(im), _stream()), "progression_kind")
    return (complex(re.value, im.value) if u.value else None), bool(real.value)


def fill_progression(support, m: int, a0: int, stride: int, length: int, amp: complex):
    t = _t()
    amps = t.empty(2 * max(length, 1), dtype=t.float64, device="cuda")
    nat.check(nat.load().shb_fill_progression(_vp(support), m, a0, stride, length, float(amp.real),
                                              float(amp.imag), _vp(amps), _stream()),
              "fill_progression")
    return amps


PRECISIONS = {"fp64": nat.FP64, "fp32": nat.FP32}


def dft(amps, length: int, a0: int, stride: int, q: int, c_begin: int, c_count: int,
        tiles: int = 1, scale: float | None = None, precision: str = "fp64",
        want_prob: bool = True, real: bool = False):
    """Direct DFT over a support progression; returns (out, prob, block_sums).

    real=True: the amplitudes' imaginary parts are zero (shb_dft_real)."""
    t = _t()
    prec = PRECISIONS[precision]
    scale = 1.0 / math.sqrt(q) if scale is None else scale
    out = t.empty(2 * max(c_count, 1), dtype=t.float64, device="cuda")
    prob = t.empty(max(c_count, 1), dtype=t.float64, device="cuda") if want_prob else None
    nb = int(nat.load().shb_dft_num_blocks(c_count, prec))
    bsum = t.empty(max(nb, 1), dtype=t.float64, device="cuda") if want_prob else None
    fn = nat.load().shb_dft_real if real else nat.load().shb_dft
    nat.check(fn(_vp(amps), length, a0, stride, q, c_begin, c_count, tiles, scale, prec,
                 _vp(out), _vp(prob), _vp(bsum), _stream()), "dft")
    out = out[: 2 * c_count]
    if want_prob:
        prob, bsum = prob[:c_count], bsum[:nb]
    return out, prob, bsum


def dft_uniform(amp: complex, length: int, a0: int, stride: int, q: int, c_begin: int, c_count: int,
                tiles: int = 1, scale: float | None = None, precision: str = "fp64",
                want_prob: bool = True):
    """Direct DFT of a uniform comb (all `length` amplitudes equal `amp`)."""
    t = _t()
    prec = PRECISIONS[precision]
    scale = 1.0 / math.sqrt(q) if scale is None else scale
    out = t.empty(2 * max(c_count, 1), dtype=t.float64, device="cuda")
    prob = t.empty(max(c_count, 1), dtype=t.float64, device="cuda") if want_prob else None
    nb = int(nat.load().shb_dft_num_blocks(c_count, prec))
    bsum = t.empty(max(nb, 1), dtype=t.float64, device="cuda") if want_prob else None
    nat.check(nat.load().shb_dft_uniform(float(amp.real), float(amp.imag), length, a0, stride, q, c_begin,
                                         c_count, tiles, scale, prec, _vp(out), _vp(prob), _vp(bsum),
                                         _stream()), "dft_uniform")
    out = out[: 2 * c_count]
    if want_prob:
        prob, bsum = prob[:c_count], bsum[:nb]
    return out, prob, bsum


def apply_hadamard(state, q: int, qubit: int) -> None:
    """In place on a device float64 [2q] vector (qft.py:164-177)."""
    nat.check(nat.load().shb_apply_hadamard(_vp(state), q, qubit, _stream()), "apply_hadamard")


def apply_controlled_phase(state, q: int, control: int, target: int, phase: complex) -> None:
    """In place; `phase` = np.exp(1j * angle) computed by the caller (qft.py:193)."""
    nat.check(nat.load().shb_apply_controlled_phase(_vp(state), q, control, target, float(phase.real),
                                                    float(phase.imag), _stream()), "apply_controlled_phase")


def bit_reverse_permute(state, q: int):
    """Out of place (qft.py:199-212); returns a new device float64 [2q] vector."""
    t = _t()
    out = t.empty_like(state)
    nat.check(nat.load().shb_bit_reverse_permute(_vp(state), _vp(out), q, _stream()), "bit_reverse_permute")
    return out


def probabilities(state):
    t = _t()
    n = state.numel() // 2
    p = t.empty(max(n, 1), dtype=t.float64, device="cuda")
    nat.check(nat.load().shb_probabilities(_vp(state), n, _vp(p), _stream()), "probabilities")
    return p[:n]


def dsum(x) -> float:
    out = ctypes.c_double(0.0)
    nat.check(nat.load().shb_sum(_vp(x), x.numel(), ctypes.byref(out), _stream()), "sum")
    return float(out.value)


def cumsum_total(p) -> float:
    out = ctypes.c_double(0.0)
    nat.check(nat.load().shb_cumsum_total(_vp(p), p.numel(), ctypes.byref(out), _stream()), "cumsum_total")
    return float(out.value)


def cumsum_search(p, target: float) -> int:
    out = ctypes.c_uint64(0)
    nat.check(nat.load().shb_cumsum_search(_vp(p), p.numel(), float(target), ctypes.byref(out), _stream()),
              "cumsum_search")
    return int(out.value)


def cumsum_total_from(p, s_in: float) -> float:
    """Running sum after p, continuing a sequential cumsum that stood at s_in."""
    out = ctypes.c_double(0.0)
    nat.check(nat.load().shb_cumsum_total_from(_vp(p), p.numel(), float(s_in), ctypes.byref(out), _stream()),
              "cumsum_total_from")
    return float(out.value)


def cumsum_search_from(p, s_in: float, target: float) -> int:
    """First i with running sum s_in + p[0] + ... + p[i] > target (sequential), else len(p)."""
    out = ctypes.c_uint64(0)
    nat.check(nat.load().shb_cumsum_search_from(_vp(p), p.numel(), float(s_in), float(target),
                                                ctypes.byref(out), _stream()), "cumsum_search_from")
    return int(out.value)


def cumsum_plan(p, s_hint: float):
    """Records of the split sequential cumsum (shb_cumsum_records): parallel,
    from a hint of the running value entering p.  Returns (records, tile_S)."""
    t = _t()
    lib = nat.load()
    nt = int(lib.shb_cumsum_tiles(p.numel()))
    recs = t.empty(max(nt, 1) * int(lib.shb_cumsum_record_bytes()), dtype=t.uint8, device=p.device)
    tile_s = t.empty(max(nt, 1), dtype=t.float64, device=p.device)
    nat.check(lib.shb_cumsum_records(_vp(p), p.numel(), float(s_hint), _vp(recs), _stream()), "cumsum_records")
    return recs, tile_s


def cumsum_walk(p, plan, s_in: float) -> float:
    """The exact walk from s_in over p (shb_cumsum_walk): the running value after p."""
    recs, tile_s = plan
    out = ctypes.c_double(0.0)
    nat.check(nat.load().shb_cumsum_walk(_vp(p), p.numel(), _vp(recs), float(s_in), _vp(tile_s),
                                         ctypes.byref(out), _stream()), "cumsum_walk")
    return float(out.value)


def cumsum_find(p, plan, s_out: float, target: float) -> int:
    """First i whose running value exceeds target, from a walked plan (shb_cumsum_find)."""
    _, tile_s = plan
    out = ctypes.c_uint64(0)
    nat.check(nat.load().shb_cumsum_find(_vp(p), p.numel(), _vp(tile_s), float(s_out), float(target),
                                         ctypes.byref(out), _stream()), "cumsum_find")
    return int(out.value)


def sample_index(p, u: float) -> tuple[int, float]:
    """searchsorted(cumsum(p), u * cumsum(p)[-1], "right") exactly, and cumsum(p)[-1]."""
    out = ctypes.c_uint64(0)
    tot = ctypes.c_double(0.0)
    nat.check(nat.load().shb_sample_index(_vp(p), p.numel(), float(u), ctypes.byref(out), ctypes.byref(tot),
                                          _stream()), "sample_index")
    return int(out.value), float(tot.value)


# --------------------------------------------------------------- array types

class DeviceVector:
    """Array-like view of a device-resident register part (lazy host copy)."""

    dtype = np.dtype(np.complex128)

    def __init__(self, q: int):
        self.q = int(q)
        self._host = None

    # numpy protocol ---------------------------------------------------------
    @property
    def shape(self):
        return (self.q,)

    @property
    def size(self):
        return self.q

    @property
    def ndim(self):
        return 1

    def __len__(self):
        return self.q

    def numpy(self) -> np.ndarray:
        if self._host is None:
            self._host = self._materialize()
        return self._host

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        if dtype is not None and np.dtype(dtype) != a.dtype:
            return a.astype(dtype)
        return a.copy() if copy else a

    def __getitem__(self, idx):
        return self.numpy()[idx]

    def __iter__(self):
        return iter(self.numpy())

    def __repr__(self):
        return f"{type(self).__name__}(q={self.q})"

    def _materialize(self) -> np.ndarray:  # pragma: no cover - abstract
        raise NotImplementedError


class UniformAmplitudes(DeviceVector):
    """1/sqrt(q) everywhere (qstate.init_uniform, qstate.py:56-61); never stored."""

    def __init__(self, q: int):
        super().__init__(q)
        self.value = 1.0 / math.sqrt(q)

    def _materialize(self):
        return np.full(self.q, self.value, dtype=np.complex128)


class ZeroResidues(DeviceVector):
    dtype = np.dtype(np.int64)

    def _materialize(self):
        return np.zeros(self.q, dtype=np.int64)


class DeviceResidues(DeviceVector):
    """x^a mod n as uint32 on the device (int64 on the host, qstate.py:39)."""

    dtype = np.dtype(np.int64)

    def __init__(self, tensor):
        super().__init__(tensor.numel())
        self.tensor = tensor

    def _materialize(self):
        return self.tensor.cpu().numpy().view(np.uint32).astype(np.int64)


class CollapsedAmplitudes(DeviceVector):
    """Post-measurement part 1: amplitude `amp` on the device support, 0 elsewhere."""

    def __init__(self, q: int, support, amp: complex, progression: tuple[int, int, int]):
        super().__init__(q)
        self.support = support
        self.m = int(support.numel())
        self.amp = complex(amp)
        self.a0, self.stride, self.length = progression

    def _materialize(self):
        out = np.zeros(self.q, dtype=np.complex128)
        if self.m:
            out[self.support.cpu().numpy()] = self.amp
        return out

    @property
    def full_comb(self) -> bool:
        """Every slot of the progression is occupied (always true after measure_part2)."""
        return self.m == self.length

    def progression_amplitudes(self):
        return fill_progression(self.support, self.m, self.a0, self.stride, self.length, self.amp)


class DeviceSpectrum(DeviceVector):
    """A complex128 vector on the device (the QFT output), with |.|^2 fused."""

    def __init__(self, q: int, data, prob=None, block_sums=None, precision: str = "fp64"):
        super().__init__(q)
        self.precision = precision
        self.data = data  # float64 [2q] interleaved
        self.prob = prob  # float64 [q] = hypot(re, im)^2, or None
        self.block_sums = block_sums

    def _materialize(self):
        return self.data.cpu().numpy().view(np.complex128)

    def probabilities(self):
        if self.prob is None:
            self.prob = probabilities(self.data)
        return self.prob

    def sum_probabilities(self) -> float:
        if self.block_sums is not None:
            return dsum(self.block_sums)
        return dsum(self.probabilities())
