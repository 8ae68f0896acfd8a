"""Owning handle over the C ABI register (``shb_ctx``, include/shorb200.h).

This is the FFI-facing form of one attempt of ``shor.single_attempt``
(shor.py:73-133): the register lives in library-owned device memory, sharded
over the handle's devices, and only integers, draws and host arrays cross the
boundary.  The stages mirror the reference's qstate calls:

    with NativeRegister() as reg:
        reg.entangle(x, n, w)          # init_uniform + entangle_modexp (qstate.py:56-83)
        k, M, amp = reg.measure(u2)    # measure_part2 with u2 = s.uniform() (qstate.py:86-105)
        reg.transform("fp64", tiles=1) # qft.dense_dft / tiled_dft (qft.py:95-142)
        m = reg.sample(u3)             # sample_part1 (qstate.py:108-114)

``qstate``/``qft`` remain the drop-in Python API (torch-tensor registers);
this class exercises the same kernels through the handle ABI, which is what a
C, Go or JNI caller would bind.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat

_PRECISION = {"fp64": nat.FP64, "fp32": nat.FP32}
STAGES = ("empty", "entangled", "collapsed", "transformed")


def host_measure_class(counts, q: int, u: float) -> tuple[int, int, float]:
    """The host half of measure_part2 from exact class counts (no device work)."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    k, M, amp = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_double()
    nat.check(nat.load().shb_host_measure_class(c.ctypes.data, c.size, q, float(u), ctypes.byref(k),
                                                ctypes.byref(M), ctypes.byref(amp)), "host_measure_class")
    return int(k.value), int(M.value), float(amp.value)


class NativeRegister:
    """A Shor register behind ``shb_ctx``; ``devices`` may repeat a device id."""

    def __init__(self, devices=None):
        lib = nat.load()
        h = ctypes.c_void_p()
        if devices is None:
            nat.check(lib.shb_init(0, ctypes.byref(h)), "shb_init")
        else:
            arr = (ctypes.c_int * len(devices))(*devices)
            nat.check(lib.shb_init_devices(ctypes.cast(arr, ctypes.c_void_p), len(devices), ctypes.byref(h)),
                      "shb_init_devices")
        self._h = h

    # ---------------------------------------------------------------- lifetime
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            nat.load().shb_free(self._h)
            self._h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, name, *args):
        nat.check(getattr(nat.load(), name)(self._h, *args), name)

    @property
    def state(self) -> dict:
        st, q, n, ns = ctypes.c_int(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int()
        self._call("shb_ctx_state", ctypes.byref(st), ctypes.byref(q), ctypes.byref(n), ctypes.byref(ns))
        return {"stage": STAGES[st.value], "q": int(q.value), "n": int(n.value), "shards": int(ns.value)}

    # ------------------------------------------------------------------ stages
    def entangle(self, x: int, n: int, w: int) -> None:
        self._call("shb_ctx_modexp", int(x), int(n), int(w))

    def class_counts(self) -> np.ndarray:
        n = self.state["n"]
        out = np.zeros(n, dtype=np.uint64)
        self._call("shb_ctx_class_counts", out.ctypes.data if n else None, n)
        return out

    def collapse(self, k: int) -> tuple[int, float]:
        M, amp = ctypes.c_uint64(), ctypes.c_double()
        self._call("shb_collapse", int(k), ctypes.byref(M), ctypes.byref(amp))
        return int(M.value), float(amp.value)

    def measure(self, u: float) -> tuple[int, int, float]:
        k, M, amp = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_double()
        self._call("shb_measure", float(u), ctypes.byref(k), ctypes.byref(M), ctypes.byref(amp))
        return int(k.value), int(M.value), float(amp.value)

    def transform(self, precision: str = "fp64", tiles: int = 1) -> None:
        if precision not in _PRECISION:
            raise ValueError(f"unknown precision {precision!r}")
        self._call("shb_ctx_dft", _PRECISION[precision], int(tiles))

    def l2_norm(self) -> float:
        out = ctypes.c_double()
        self._call("shb_norm", ctypes.byref(out))
        return float(out.value)

    def sample(self, u: float) -> int:
        m = ctypes.c_uint64()
        self._call("shb_sample", float(u), ctypes.byref(m))
        return int(m.value)

    # ----------------------------------------------------------------- readers
    def spectrum(self, c0: int = 0, c1: int | None = None) -> np.ndarray:
        q = self.state["q"]
        c1 = q if c1 is None else c1
        out = np.empty(max(c1 - c0, 0), dtype=np.complex128)
        self._call("shb_copy_spectrum", int(c0), int(c1), out.ctypes.data if out.size else None)
        return out

    def support(self) -> np.ndarray:
        m = ctypes.c_uint64()
        rc = nat.load().shb_copy_support(self._h, None, 0, ctypes.byref(m))
        if rc not in (nat.SHB_OK, nat.SHB_ERANGE):
            nat.check(rc, "shb_copy_support")
        out = np.empty(int(m.value), dtype=np.uint64)
        self._call("shb_copy_support", out.ctypes.data if out.size else None, out.size, ctypes.byref(m))
        return out

    def residues(self, a0: int = 0, a1: int | None = None) -> np.ndarray:
        q = self.state["q"]
        a1 = q if a1 is None else a1
        out = np.empty(max(a1 - a0, 0), dtype=np.int64)
        self._call("shb_copy_residues", int(a0), int(a1), out.ctypes.data if out.size else None)
        return out

    def dump_state(self, path) -> None:
        self._call("shb_dump_state", str(path).encode())
