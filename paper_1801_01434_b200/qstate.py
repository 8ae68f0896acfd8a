"""Two-part register on the B200: drop-in for ``shorsim.qstate``.

Same public names and signatures as the reference (qstate.py:23-145).  The
register parts live on the GPU (``device.DeviceVector``); every stage runs in
libshorb200.so:

* ``entangle_modexp``  -> shb_modexp            (Barrett modexp, HBM-bound)
* ``measure_part2``    -> shb_class_counts + shb_compact_eq (histogram + ballot compaction)
* ``sample_part1``     -> fused |V|^2 + shb_cumsum_total / shb_cumsum_search
                          (exact emulation of numpy's sequential cumsum)

Host work is O(number of residue classes): the outcome k and the collapsed
amplitude are computed from exact integer class counts with the reference's
own float64 reductions, so k, the support and the amplitude are bit-identical
to the reference for every register width.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from . import device as dev

_NORM_TOL = 1e-9
_DUMP_MAGIC = b"QREG"
_DUMP_VERSION = 1
_DUMP_HEADER = struct.Struct("<4sIII")  # magic, version, width, reserved (qstate.py:18-20)


class Sampler:
    """Seeded uniform doubles in [0, 1): numpy PCG64, identical stream to qstate.py:23-32."""

    def __init__(self, seed: int):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self._gen = np.random.Generator(np.random.PCG64(self.seed))

    def uniform(self) -> float:
        return float(self._gen.random())


@dataclass
class CompositeRegister:
    """|r1, r2> (qstate.py:35-42); amplitudes / residues may be device-resident."""

    q: int
    amplitudes: object
    residues: object
    n: int | None = None
    x: int | None = None
    collapsed_k: int | None = None


def _require_power_of_two(q: int) -> None:
    if q < 2 or q & (q - 1):
        raise ValueError(f"q must be a power of two >= 2, got {q}")


def norm_tolerance(precision: str = "fp64") -> float:
    """_NORM_TOL (qstate.py:17) for FP64 registers; the FP32 fast path's own
    stated accuracy (1e-4) for spectra it produced."""
    return _NORM_TOL if precision == "fp64" else 1e-4


def _require_normalized(reg: CompositeRegister) -> None:
    norm = l2_norm(reg)
    prec = getattr(reg.amplitudes, "precision", "fp64")
    if abs(norm - 1.0) > norm_tolerance(prec):
        raise ValueError(f"register is not normalized (|amp| = {norm!r})")


def init_uniform(q: int) -> CompositeRegister:
    """(1/sqrt q) sum_a |a, 0> (qstate.py:56-61); the constant is never stored."""
    _require_power_of_two(q)
    return CompositeRegister(q=q, amplitudes=dev.UniformAmplitudes(q), residues=dev.ZeroResidues(q))


def entangle_modexp(reg: CompositeRegister, x: int, n: int) -> CompositeRegister:
    """residues[a] = x**a mod n for every a (qstate.py:64-83), on the GPU."""
    if n < 2:
        raise ValueError("modulus must be >= 2")
    if math.gcd(x, n) != 1:
        raise ValueError(f"x={x} shares a factor with n={n}")
    if reg.collapsed_k is not None:
        raise ValueError("register already collapsed")
    if n > 0xFFFFFFFF:
        raise ValueError(f"modulus {n} exceeds the 32-bit residue storage of the B200 path")
    res = dev.modexp(x % n, n, reg.q)  # the reference walks x % n (qstate.py:78): any int x
    return replace(reg, residues=dev.DeviceResidues(res), n=n, x=x)


def _device_residues(reg: CompositeRegister):
    r = reg.residues
    if isinstance(r, dev.DeviceResidues):
        return r.tensor
    t = nat.require_cuda()
    arr = np.asarray(r)
    if arr.size and (arr.min() < 0 or arr.max() > 0xFFFFFFFF):
        raise ValueError("residues must lie in [0, 2^32)")
    return t.from_numpy(np.ascontiguousarray(arr, dtype=np.int64).astype(np.uint32).view(np.int32)).cuda()


def _uniform_value(amps, q: int):
    """The common amplitude of a uniform register, or None."""
    if isinstance(amps, dev.UniformAmplitudes):
        return complex(amps.value)
    if isinstance(amps, dev.DeviceVector):
        return None
    a = np.asarray(amps, dtype=np.complex128)
    if a.shape == (q,) and q and np.all(a == a[0]):
        return complex(a[0])
    return None


def _class_probabilities(counts: np.ndarray, w0: float) -> np.ndarray:
    """np.bincount(res, weights=full(q, w0)) from exact counts (qstate.py:97).

    bincount adds each bin's weights left to right, so bin v holds the
    sequential float64 sum of counts[v] copies of w0.
    """
    out = np.zeros(counts.size, dtype=np.float64)
    nz = np.flatnonzero(counts)
    # the sum depends only on the count: one closed-form evaluation per distinct count
    uniq, inv = np.unique(np.asarray(counts)[nz], return_inverse=True)
    vals = np.array([nat.host_seqsum_const(w0, int(c)) for c in uniq], dtype=np.float64)
    out[nz] = vals[inv]
    return out


def uniform_weight(a_unif: complex) -> float:
    """|amp|^2 of the uniform amplitude, as np.abs(amp)**2 computes it (qstate.py:95)."""
    return float(np.abs(np.array([a_unif], dtype=np.complex128))[0] ** 2)


def draw_class(counts: np.ndarray, w0: float, u: float) -> int:
    """Outcome k from exact class counts and the draw u (qstate.py:96-100)."""
    nz = np.flatnonzero(counts)
    nclasses = int(nz[-1]) + 1
    probs = _class_probabilities(np.asarray(counts)[:nclasses], w0)
    cum = np.cumsum(probs)
    k = int(np.searchsorted(cum, u * cum[-1], side="right"))
    return min(k, nclasses - 1)


def collapsed_amplitude(a_unif: complex, w0: float, M: int) -> complex:
    """amp / sqrt(sum of the M kept weights) exactly as qstate.py:102-104 rounds it."""
    kept = np.sqrt(np.float64(nat.host_pairwise_sum_const(w0, M)))
    return complex((np.array([a_unif], dtype=np.complex128) / kept)[0])


def measure_part2(reg: CompositeRegister, s: Sampler) -> tuple[int, CompositeRegister]:
    """Observe part 2 and collapse part 1 onto {a : residue[a] == k} (qstate.py:86-105)."""
    _require_normalized(reg)
    if reg.collapsed_k is not None:
        raise ValueError("part 2 was already measured")
    q = reg.q
    a_unif = _uniform_value(reg.amplitudes, q)
    if a_unif is None:
        raise ValueError("measure_part2 on the B200 path expects the uniform superposition "
                         "from init_uniform (the only state Shor's algorithm measures)")
    res = _device_residues(reg)
    ncls_bound = reg.n if reg.n is not None else int(res.max().item()) + 1
    counts = dev.class_counts(res, ncls_bound).cpu().numpy()
    w0 = uniform_weight(a_unif)
    k = draw_class(counts, w0, s.uniform())
    support = dev.compact_eq(res, k, expected=int(counts[k]))
    amp = collapsed_amplitude(a_unif, w0, int(support.numel()))
    prog = dev.support_progression(support)
    amps = dev.CollapsedAmplitudes(q, support, amp, prog)
    return k, replace(reg, amplitudes=amps, collapsed_k=k)


def _device_probabilities(reg: CompositeRegister):
    """|amp|^2 of part 1 as a device float64 tensor (qstate.py:111)."""
    t = nat.require_cuda()
    a = reg.amplitudes
    if isinstance(a, dev.DeviceSpectrum):
        return a.probabilities()
    if isinstance(a, dev.UniformAmplitudes):
        w0 = float(np.abs(np.complex128(a.value)) ** 2)
        return t.full((reg.q,), w0, dtype=t.float64, device="cuda")
    if isinstance(a, dev.CollapsedAmplitudes):
        p = t.zeros(reg.q, dtype=t.float64, device="cuda")
        if a.m:
            p[a.support] = float(np.abs(np.complex128(a.amp)) ** 2)
        return p
    host = np.ascontiguousarray(np.asarray(a), dtype=np.complex128)
    return dev.probabilities(t.from_numpy(host.view(np.float64)).cuda())


def sample_part1(reg: CompositeRegister, s: Sampler) -> int:
    """Born-rule read of part 1 (qstate.py:108-114), exact sequential CDF on the GPU."""
    _require_normalized(reg)
    p = _device_probabilities(reg)
    m, _ = dev.sample_index(p, s.uniform())  # target = u * cum[-1], as qstate.py:113
    return min(m, reg.q - 1)


def l2_norm(reg: CompositeRegister) -> float:
    """sqrt(sum |amp|^2) (qstate.py:117-118)."""
    a = reg.amplitudes
    if isinstance(a, dev.UniformAmplitudes):
        return math.sqrt(a.q) * abs(a.value)
    if isinstance(a, dev.CollapsedAmplitudes):
        return math.sqrt(a.m) * abs(a.amp)
    if isinstance(a, dev.DeviceSpectrum):
        return math.sqrt(a.sum_probabilities())
    return float(np.linalg.norm(np.asarray(a)))


def dump_state(reg: CompositeRegister, path) -> None:
    """QREG dump: 16-byte header + q little-endian complex128 (qstate.py:121-130).

    Device spectra are streamed to the file in 64 MiB slices, never as one
    host copy of the whole register.
    """
    q = reg.q
    w = q.bit_length() - 1
    with open(path, "wb") as fh:
        fh.write(_DUMP_HEADER.pack(_DUMP_MAGIC, _DUMP_VERSION, w, 0))
        a = reg.amplitudes
        if isinstance(a, dev.DeviceSpectrum):
            step = 1 << 22
            for lo in range(0, q, step):
                hi = min(q, lo + step)
                fh.write(a.data[2 * lo: 2 * hi].cpu().numpy().astype("<f8").tobytes())
        else:
            fh.write(np.ascontiguousarray(np.asarray(a), dtype="<c16").tobytes())


def load_state(path) -> np.ndarray:
    """Read a dump_state file back (qstate.py:133-145)."""
    with open(path, "rb") as fh:
        magic, version, w, _ = _DUMP_HEADER.unpack(fh.read(_DUMP_HEADER.size))
        if magic != _DUMP_MAGIC:
            raise ValueError(f"not a register dump (magic {magic!r})")
        if version != _DUMP_VERSION:
            raise ValueError(f"unsupported dump version {version}")
        q = 1 << w
        data = np.frombuffer(fh.read(q * 16), dtype="<c16")
        if data.size != q:
            raise ValueError("truncated register dump")
        return data.astype(np.complex128)
