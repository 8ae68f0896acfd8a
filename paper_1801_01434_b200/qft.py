"""QFT engines on the B200: drop-in for ``shorsim.qft``.

Same public names, signatures and validation as the reference (qft.py:29-253).
Every engine name maps to ONE implementation, the sm_100a direct-DFT kernel
(``shb_dft``): it evaluates exactly the sum the reference's ``dense_dft``
defines, V_k = (1/sqrt q) sum_j e^{+2 pi i jk/q} V_j, over the nonzero
support only.  ``tiled_dft`` keeps its split-K meaning (input segments summed
in ascending order).  ``fft_dft`` is the same unitary and is served by the
same kernel (no second backend, no CPU fallback).  ``circuit_qft`` is built
from the reference's gate primitives (``apply_hadamard``,
``apply_controlled_phase``, ``bit_reverse_permute``), which run as their own
device kernels (csrc/gates.cu), so the circuit engine is an independent
gate-level cross-check of the DFT kernels for w <= 12.

``block_size`` / ``workers`` of ``KernelPlan`` describe the reference's CPU
thread decomposition; they are validated as before but do not change the GPU
decomposition (fixed for sm_100a: 256 threads x 4 outputs per CTA).
``KernelPlan.precision`` ("fp64" default, "fp32" fast path) is the one added
knob.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from . import device as dev

ENGINES = ("dense", "tiled", "fft", "circuit")
CIRCUIT_MAX_WIDTH = 12


def _require_power_of_two(q: int) -> None:
    if q < 2 or q & (q - 1):
        raise ValueError(f"size must be a power of two >= 2, got {q}")


class TwiddleTable:
    """roots[j] = e^{+2 pi i j/q} (qft.py:39-44).

    The GPU kernel derives every phase from the exact integer index, so the
    16*q-byte table is only built if a caller reads ``roots``.
    """

    __slots__ = ("q", "_roots")

    def __init__(self, q: int, roots: np.ndarray | None = None):
        self.q = q
        self._roots = roots

    @property
    def roots(self) -> np.ndarray:
        if self._roots is None:
            self._roots = np.exp((2j * np.pi / self.q) * np.arange(self.q))
        return self._roots

    def __eq__(self, other):
        return isinstance(other, TwiddleTable) and other.q == self.q

    def __hash__(self):
        return hash(("TwiddleTable", self.q))

    def __repr__(self):
        return f"TwiddleTable(q={self.q})"


@dataclass(frozen=True)
class KernelPlan:
    """Work decomposition (qft.py:47-72) plus the arithmetic precision."""

    block_size: int = 256
    tiles: int = 1
    workers: int | None = None
    precision: str = "fp64"

    def resolved(self, q: int) -> "KernelPlan":
        bs = min(self.block_size, q)
        if bs < 1 or q % bs:
            raise ValueError(f"block_size {self.block_size} does not divide q={q}")
        if self.tiles < 1 or q % self.tiles:
            raise ValueError(f"tiles {self.tiles} does not divide q={q}")
        workers = self.workers if self.workers is not None else (os.cpu_count() or 1)
        if workers < 1:
            raise ValueError("workers must be >= 1")
        if self.precision not in dev.PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(dev.PRECISIONS)}")
        return replace(self, block_size=bs, workers=workers)

    def num_blocks(self, q: int) -> int:
        return q // min(self.block_size, q)


def build_twiddles(q: int, max_width: int = 24) -> TwiddleTable:
    """qft.py:75-80 (validation identical; the table itself is lazy)."""
    _require_power_of_two(q)
    if q.bit_length() - 1 > max_width:
        raise ValueError(f"q={q} exceeds the configured maximum width {max_width}")
    return TwiddleTable(q)


# ------------------------------------------------------------- device engine

def _support_of(state, q: int):
    """(amps, length, a0, stride, host_input, real) for any state form.

    amps is a device tensor, or a Python complex when every progression slot
    holds the same amplitude (the uniform-comb kernel is selected from the data).
    """
    t = nat.require_cuda()
    if isinstance(state, dev.CollapsedAmplitudes):
        if state.q != q:
            raise ValueError(f"state length {(state.q,)} does not match q={q}")
        if state.full_comb:
            return state.amp, state.length, state.a0, state.stride, False, True
        return (state.progression_amplitudes(), state.length, state.a0, state.stride, False,
                complex(state.amp).imag == 0.0)
    if isinstance(state, dev.UniformAmplitudes):
        if state.q != q:
            raise ValueError(f"state length {(state.q,)} does not match q={q}")
        return complex(state.value), q, 0, 1, False, True
    if isinstance(state, dev.DeviceSpectrum):
        if state.q != q:
            raise ValueError(f"state length {(state.q,)} does not match q={q}")
        data = state.data
        host = False
    else:
        arr = np.ascontiguousarray(state, dtype=np.complex128)
        if arr.shape != (q,):
            raise ValueError(f"state length {arr.shape} does not match q={q}")
        data = t.from_numpy(arr.view(np.float64)).cuda()
        host = True
    a0, stride, length = dev.state_progression(data)
    amps = dev.gather_progression(data, a0, stride, length) if length else None
    uni, real = dev.progression_kind(amps, length) if length else (None, True)
    if uni is not None:
        return uni, length, a0, stride, host, True
    return amps, length, a0, stride, host, real


def _run(state, q: int, tiles: int, precision: str):
    if not isinstance(state, (dev.DeviceVector, dev.CollapsedAmplitudes, dev.UniformAmplitudes)):
        # host in, host out: the C-ABI drop-in overlaps both copies with the DFT
        # (capi.cu dft_host_common) and picks the same kernel from the same data
        arr = np.ascontiguousarray(state, dtype=np.complex128)
        if arr.shape != (q,):
            raise ValueError(f"state length {arr.shape} does not match q={q}")
        nat.require_cuda()
        lib = nat.load()
        out = np.empty(q, dtype=np.complex128)
        nat.check(lib.shb_dense_dft_host(arr.ctypes.data, q, tiles, dev.PRECISIONS[precision], out.ctypes.data),
                  "dense_dft")
        return out
    amps, length, a0, stride, host, real = _support_of(state, q)
    if isinstance(amps, complex):
        out, prob, bsum = dev.dft_uniform(amps, length, a0, stride, q, 0, q, tiles=tiles,
                                          scale=1.0 / math.sqrt(q), precision=precision)
    else:
        out, prob, bsum = dev.dft(amps, length, a0, stride, q, 0, q, tiles=tiles,
                                  scale=1.0 / math.sqrt(q), precision=precision, real=real)
    spec = dev.DeviceSpectrum(q, out, prob, bsum, precision=precision)
    return spec.numpy() if host else spec


def _check_length(state, q: int) -> None:
    """The reference validates the state length before the plan (qft.py:98-101)."""
    n = (state.q,) if isinstance(state, dev.DeviceVector) else np.shape(state)
    if tuple(n) != (q,):
        raise ValueError(f"state length {tuple(n)} does not match q={q}")


def dense_dft(state, tw: TwiddleTable, plan: KernelPlan):
    """Direct DFT, untiled (qft.py:95-112), on the GPU.

    A numpy input returns a numpy array (drop-in); a device-resident register
    part returns a DeviceSpectrum that stays on the GPU.
    """
    q = tw.q
    _check_length(state, q)
    plan = plan.resolved(q)
    if plan.tiles != 1:
        raise ValueError("dense_dft is untiled; use tiled_dft for tiles >= 2")
    return _run(state, q, 1, plan.precision)


def tiled_dft(state, tw: TwiddleTable, plan: KernelPlan):
    """Split-K DFT (qft.py:115-142): input segments reduced in ascending order."""
    q = tw.q
    _check_length(state, q)
    plan = plan.resolved(q)
    if plan.tiles < 2:
        raise ValueError("tiled_dft needs tiles >= 2; use dense_dft otherwise")
    return _run(state, q, plan.tiles, plan.precision)


def _length(state) -> int:
    return state.q if isinstance(state, dev.DeviceVector) else int(np.size(state))


def fft_dft(state, precision: str = "fp64"):
    """Same transform as qft.py:145-161 (served by the direct-DFT kernel).

    `precision` is the plan's (transform passes it): the fast path is
    honoured here exactly as for the dense engine."""
    q = _length(state)
    _require_power_of_two(q)
    if precision not in dev.PRECISIONS:
        raise ValueError(f"precision must be one of {tuple(dev.PRECISIONS)}")
    return _run(state, q, 1, precision)


# ------------------------------------------------------------- gate level
# The reference's circuit engine (qft.py:164-231) on device kernels
# (csrc/gates.cu), bit-identical to its numpy arithmetic.  A numpy input
# returns numpy; a device vector (register part or spectrum) returns a
# DeviceSpectrum that stays on the GPU.  Like the reference, every call
# works on a copy.

def _dense_device_copy(state):
    """(float64 [2q] device copy of the state, q, came_from_host)."""
    t = nat.require_cuda()
    if isinstance(state, dev.DeviceSpectrum):
        return state.data.clone(), state.q, False
    if isinstance(state, dev.CollapsedAmplitudes):
        data = t.zeros(2 * state.q, dtype=t.float64, device="cuda")
        if state.m:
            v = data.view(t.complex128)
            v[state.support] = complex(state.amp)
        return data, state.q, False
    if isinstance(state, dev.UniformAmplitudes):
        data = t.zeros(2 * state.q, dtype=t.float64, device="cuda")
        data[0::2] = float(state.value)
        return data, state.q, False
    arr = np.array(state, dtype=np.complex128)
    return t.from_numpy(arr.view(np.float64).reshape(-1)).cuda(), arr.size, True


def _finish(data, q: int, host: bool):
    spec = dev.DeviceSpectrum(q, data)
    return spec.numpy().copy() if host else spec


def apply_hadamard(state, qubit_index: int):
    """qft.py:164-177: (u, v) -> ((u+v)/sqrt2, (u-v)/sqrt2) on bit `qubit_index`."""
    q = _length(state)
    _require_power_of_two(q)
    w = q.bit_length() - 1
    if not 0 <= qubit_index < w:
        raise ValueError(f"qubit index {qubit_index} out of range for w={w}")
    data, q, host = _dense_device_copy(state)
    dev.apply_hadamard(data, q, qubit_index)
    return _finish(data, q, host)


def _phase(angle: float) -> complex:
    """np.exp(1j * angle) as qft.py:193 evaluates it."""
    return complex(np.exp(1j * angle))


def apply_controlled_phase(state, control: int, target: int, angle: float):
    """qft.py:180-196: amplitudes with both index bits set times e^{+i angle}."""
    if control == target:
        raise ValueError("control and target must differ")
    q = _length(state)
    _require_power_of_two(q)
    w = q.bit_length() - 1
    for bit in (control, target):
        if not 0 <= bit < w:
            raise ValueError(f"qubit index {bit} out of range for w={w}")
    data, q, host = _dense_device_copy(state)
    dev.apply_controlled_phase(data, q, control, target, _phase(angle))
    return _finish(data, q, host)


def bit_reverse_permute(state):
    """qft.py:199-212: output[reverse_bits(a)] = input[a] over the full width.

    The reference keeps the input dtype; real and integer inputs are moved
    as complex128 (exact for |values| < 2^53) and cast back."""
    if isinstance(state, dev.DeviceVector):
        _require_power_of_two(state.q)
        data, q, _ = _dense_device_copy(state)
        return _finish(dev.bit_reverse_permute(data, q), q, False)
    a = np.asarray(state)
    _require_power_of_two(a.size)
    if a.dtype == np.complex128:
        return _run_permute(a)
    if a.dtype.kind == "c":
        return _run_permute(a.astype(np.complex128)).astype(a.dtype)
    if a.dtype.kind in "iu" and a.size and int(np.abs(a.astype(object)).max()) >= 1 << 53:
        raise ValueError("bit_reverse_permute on the device moves values as complex128: "
                         "integers must be below 2^53 in magnitude")
    return _run_permute(a.astype(np.complex128)).real.astype(a.dtype)


def _run_permute(a: np.ndarray) -> np.ndarray:
    data, q, _ = _dense_device_copy(a)
    return _finish(dev.bit_reverse_permute(data, q), q, True)


def circuit_qft(state, max_width: int = CIRCUIT_MAX_WIDTH):
    """Gate-level QFT (qft.py:215-231): Hadamards plus controlled phases, then
    the bit reversal -- O(w^2) device gate launches, width cap kept.  An
    independent construction of the same unitary as the DFT kernels."""
    q = _length(state)
    _require_power_of_two(q)
    w = q.bit_length() - 1
    if w > max_width:
        raise ValueError(f"circuit engine capped at w <= {max_width}, got w={w}")
    data, q, host = _dense_device_copy(state)
    for i in range(w - 1, -1, -1):
        dev.apply_hadamard(data, q, i)
        for j in range(i - 1, -1, -1):
            dev.apply_controlled_phase(data, q, j, i, _phase(2.0 * np.pi / (1 << (i - j + 1))))
    return _finish(dev.bit_reverse_permute(data, q), q, host)


def transform(state, engine: str, tw: TwiddleTable | None = None, plan: KernelPlan | None = None):
    """Engine dispatch with the reference's argument semantics (qft.py:234-253)."""
    if engine not in ENGINES:
        raise ValueError(f"unknown engine {engine!r}; expected one of {ENGINES}")
    if engine == "fft":
        return fft_dft(state, plan.precision if plan is not None else "fp64")
    if engine == "circuit":
        if plan is not None and plan.precision != "fp64":
            raise ValueError("the circuit engine is gate-level FP64 only; use dense/tiled/fft for precision="
                             f"{plan.precision!r}")
        return circuit_qft(state)
    if tw is None:
        tw = build_twiddles(_length(state))
    if plan is None:
        plan = KernelPlan()
    if engine == "dense":
        return dense_dft(state, tw, plan)
    return tiled_dft(state, tw, plan)
