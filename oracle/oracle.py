"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the Shor hot path.

Restates the reference ``shorsim`` algorithm (``/root/reference/pkg/src/shorsim``)
for the stages the B200 path replaces, so the CUDA kernels can be checked
on the same inputs.  Nothing in ``paper_1801_01434_b200`` imports this module;
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (the cpu_baseline
leg and ``--impl reference``) do, and only as the checker / CPU baseline.

Parity pin: ``tests/test_oracle_golden.py`` checks these functions against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by running the reference package itself.

Heavy loops live in ``oracle/shor_oracle.c`` (built by ``oracle/Makefile``);
this module holds the ctypes binding and the numpy-level restatements.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None


def build() -> Path:
    """Compile oracle/shor_oracle.c with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        u64, vp, i32, f64 = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.oracle_roots.argtypes = [u64, u64, vp, vp]
        L.oracle_dft_rows.argtypes = [u64, u64, vp, vp, u64, vp, i32, f64, vp, i32]
        L.oracle_dense_rows_literal.argtypes = [u64, vp, u64, u64, u64, vp, vp, i32]
        L.oracle_modexp.argtypes = [u64, u64, u64, u64, vp]
        L.oracle_class_counts.argtypes = [vp, u64, u64, vp]
        L.oracle_cumsum_search.argtypes = [vp, u64, f64, vp]
        L.oracle_cumsum_search.restype = u64
        L.oracle_comb_rows_exact.argtypes = [u64, u64, u64, u64, f64, f64, f64, u64, vp, vp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------- twiddles

def roots(q: int, idx) -> np.ndarray:
    """Entries of qft.build_twiddles(q).roots at `idx` (qft.py:79), bitwise."""
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.empty(2 * idx.size, dtype=np.float64)
    lib().oracle_roots(q, idx.size, _ptr(idx), _ptr(out))
    return out.view(np.complex128)


# ---------------------------------------------------------------- QFT rows

def dft_rows(state_support, amps, q: int, rows, scale: bool = True,
             threads: int | None = None) -> np.ndarray:
    """Rows `rows` of qft.dense_dft (qft.py:95-112 / _kernels.py:16-30).

    `state_support` are the ascending indices of the nonzero amplitudes and
    `amps` their complex values.  With scale=True the 1/sqrt(q) factor is
    applied exactly as qft.py:111 does; bitwise identical to the reference.
    """
    supp = np.ascontiguousarray(state_support, dtype=np.uint64)
    a = np.ascontiguousarray(amps, dtype=np.complex128)
    r = np.ascontiguousarray(rows, dtype=np.uint64)
    if supp.size != a.size:
        raise ValueError("support / amplitude length mismatch")
    if supp.size > 1 and np.any(np.diff(supp.astype(np.int64)) <= 0):
        raise ValueError("support must be strictly ascending")
    out = np.empty(2 * r.size, dtype=np.float64)
    s = 1.0 / math.sqrt(q)
    lib().oracle_dft_rows(q, supp.size, _ptr(supp), _ptr(a.view(np.float64)),
                          r.size, _ptr(r), 1 if scale else 0, s, _ptr(out),
                          threads or default_threads())
    return out.view(np.complex128)


def dense_dft(state: np.ndarray, threads: int | None = None) -> np.ndarray:
    """Whole reference dense_dft output for a dense state vector (any q)."""
    state = np.ascontiguousarray(state, dtype=np.complex128)
    q = state.size
    nz = np.flatnonzero(state)
    return dft_rows(nz, state[nz], q, np.arange(q, dtype=np.uint64), True, threads)


def tiled_dft(state: np.ndarray, tiles: int, threads: int | None = None) -> np.ndarray:
    """Reference tiled_dft (qft.py:115-142): per-segment partials, ascending add."""
    state = np.ascontiguousarray(state, dtype=np.complex128)
    q = state.size
    seg = q // tiles
    rows = np.arange(q, dtype=np.uint64)
    out = None
    for t in range(tiles):
        lo, hi = t * seg, (t + 1) * seg
        nz = np.flatnonzero(state[lo:hi]) + lo
        part = dft_rows(nz, state[nz], q, rows, False, threads)
        out = part.copy() if out is None else out + part
    return out * (1.0 / math.sqrt(q))


def dense_rows_literal(state: np.ndarray, rows, j0: int = 0, j1: int | None = None,
                       threads: int | None = None) -> np.ndarray:
    """_kernels.partial_row_sums over ALL j in [j0, j1) (zeros included), unscaled."""
    state = np.ascontiguousarray(state, dtype=np.complex128)
    q = state.size
    j1 = q if j1 is None else j1
    r = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.empty(2 * r.size, dtype=np.float64)
    lib().oracle_dense_rows_literal(q, _ptr(state.view(np.float64)), j0, j1, r.size,
                                    _ptr(r), _ptr(out), threads or default_threads())
    return out.view(np.complex128)


# ---------------------------------------------------------------- modexp

def modexp_residues(x: int, n: int, q: int, a_begin: int = 0) -> np.ndarray:
    """entangle_modexp residues (qstate.py:64-83) as uint32, by recurrence."""
    out = np.empty(q, dtype=np.uint32)
    lib().oracle_modexp(x, n, a_begin, q, _ptr(out))
    return out


def modexp_residues_cycle(x: int, n: int, q: int) -> np.ndarray:
    """The reference's own construction: one cycle of x^a, tiled to q (qstate.py:77-82)."""
    seq = [1 % n]
    v = x % n
    while v != 1 % n:
        seq.append(v)
        v = v * x % n
    return np.resize(np.asarray(seq, dtype=np.int64), q)


# ---------------------------------------------------------------- collapse

def class_counts(residues: np.ndarray, ncls: int) -> np.ndarray:
    r = np.ascontiguousarray(residues, dtype=np.uint32)
    out = np.empty(ncls, dtype=np.uint64)
    lib().oracle_class_counts(_ptr(r), r.size, ncls, _ptr(out))
    return out


def measure_part2(amplitudes: np.ndarray, residues: np.ndarray, u: float):
    """qstate.measure_part2 (qstate.py:86-105) on host arrays with draw u.

    Returns (k, collapsed amplitude vector).
    """
    amps = np.asarray(amplitudes, dtype=np.complex128)
    res = np.asarray(residues, dtype=np.int64)
    w = np.abs(amps) ** 2
    ncls = int(res.max()) + 1
    probs = np.bincount(res, weights=w, minlength=ncls)
    cdf = np.cumsum(probs)
    k = min(int(np.searchsorted(cdf, u * cdf[-1], side="right")), ncls - 1)
    sel = res == k
    norm = np.sqrt(w[sel].sum())
    out = np.zeros_like(amps)
    out[sel] = amps[sel] / norm
    return k, out


def attempt_register(n: int, seed: int) -> dict:
    """The collapsed register of attempt 1 of run_shor(ShorConfig(n, seed=seed)),
    with the reference's own float64 arithmetic and no q-sized arrays.

    Draw #1 is the base, x = 2 + int(u (n - 3)) (shor.py:67-70); q from
    numtheory.py:166-175; the residues x^a mod n repeat with period r, so
    class cycle[j] holds floor((q - 1 - j) / r) + 1 indices (qstate.py:77-82).
    np.bincount adds each bin's weights sequentially, so a class's probability
    is the sequential sum of its count copies of |1/sqrt q|^2; the outcome k
    is the inverse CDF at draw #2 (qstate.py:95-100) and the kept amplitude
    is amp / sqrt(pairwise sum of the M kept weights) (qstate.py:102-104).
    Raises ValueError when x shares a factor with n (the gcd shortcut).
    """
    w = (n * n - 1).bit_length()
    q = 1 << w
    gen = np.random.Generator(np.random.PCG64(int(seed) & 0xFFFFFFFFFFFFFFFF))
    x = 2 + int(float(gen.random()) * (n - 3))
    if math.gcd(x, n) != 1:
        raise ValueError(f"seed {seed}: x={x} shares a factor with n={n}")
    cycle = [1]
    v = x % n
    while v != 1:
        cycle.append(v)
        v = v * x % n
    r = len(cycle)
    amp0 = np.full(1, 1.0 / math.sqrt(q), dtype=np.complex128)
    w0 = float(np.abs(amp0[0]) ** 2)
    counts = np.array([(q - 1 - j) // r + 1 for j in range(r)], dtype=np.int64)
    seq = {int(c): float(np.cumsum(np.full(int(c), w0))[-1]) for c in np.unique(counts)}
    ncls = max(cycle) + 1
    probs = np.zeros(ncls, dtype=np.float64)
    probs[np.asarray(cycle, dtype=np.int64)] = [seq[int(c)] for c in counts]
    cum = np.cumsum(probs)
    k = min(int(np.searchsorted(cum, float(gen.random()) * cum[-1], side="right")), ncls - 1)
    c0 = cycle.index(k)
    M = int(counts[c0])
    amp = complex((amp0 / np.sqrt(np.full(M, w0).sum()))[0])
    return {"n": n, "q": q, "x": x, "r": r, "k": k, "c0": c0, "M": M, "amp": amp}


# ---------------------------------------------------------------- sampling

def probabilities(spectrum: np.ndarray) -> np.ndarray:
    """|amp|**2 as qstate.py:111 computes it (np.abs -> hypot, then square)."""
    return np.abs(np.asarray(spectrum, dtype=np.complex128)) ** 2


def sample_index(probs: np.ndarray, u: float) -> int:
    """qstate.sample_part1 tail (qstate.py:112-114) via the C sequential scan."""
    p = np.ascontiguousarray(probs, dtype=np.float64)
    return int(lib().oracle_cumsum_search(_ptr(p), p.size, u, None))


def sample_index_numpy(probs: np.ndarray, u: float) -> int:
    cdf = np.cumsum(probs)
    m = int(np.searchsorted(cdf, u * cdf[-1], side="right"))
    return min(m, probs.size - 1)


def cumsum_total_from(probs: np.ndarray, s_in: float) -> float:
    """Running value of np.cumsum (qstate.py:112, a strictly sequential chain of
    float64 adds) after `probs`, when the chain stood at s_in before them."""
    return float(np.cumsum(np.concatenate([[float(s_in)], np.asarray(probs, dtype=np.float64)]))[-1])


def cumsum_search_from(probs: np.ndarray, s_in: float, target: float) -> int:
    """searchsorted(cumsum, target, "right") (qstate.py:113) restricted to a
    shard whose chain starts at s_in: first i with s_in + p[0] + ... + p[i] >
    target, else len(probs)."""
    c = np.cumsum(np.concatenate([[float(s_in)], np.asarray(probs, dtype=np.float64)]))[1:]
    return int(np.searchsorted(c, target, side="right"))


# ---------------------------------------------------------------- closed form

def comb_probabilities(q: int, r: int, c0: int, M: int, rows) -> np.ndarray:
    """Independent closed form of |V_c|^2 for a uniform comb {c0 + j r}, j < M.

    |V_c|^2 = sin^2(pi c r M / q) / (q M sin^2(pi c r / q)), and M/q when
    c r = 0 mod q.  Phases are reduced exactly in integers to a signed residue
    before the sine.  Not derived from the reference code;
    used as a size-independent property check at q = 2^24..2^32.
    """
    rows = np.asarray(rows, dtype=np.uint64)
    out = np.empty(rows.size, dtype=np.float64)
    for i, c in enumerate(rows.tolist()):
        a = (c * r) % q
        if a == 0:
            out[i] = M / q
            continue
        b = (c * r * M) % q
        a_s = a - q if a > q // 2 else a
        b_s = b - q if b > q // 2 else b
        num = math.sin(math.pi * b_s / q)
        den = math.sin(math.pi * a_s / q)
        out[i] = (num * num) / (q * M * den * den)
    return out


def comb_rows_exact(q: int, r: int, c0: int, M: int, amp: complex, rows, scale: bool = True) -> np.ndarray:
    """Accuracy reference for a uniform comb's DFT rows (oracle_comb_rows_exact):
    the geometric-series closed form in long double with exact integer phase
    reduction, ~1e-18 relative before the final rounding.  Not the reference's
    arithmetic -- the reference's sequential sum (dft_rows) is the less
    accurate of the two on peak rows; this says which side of a disagreement
    is right."""
    r_ = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.empty(2 * r_.size, dtype=np.float64)
    s = 1.0 / math.sqrt(q) if scale else 1.0
    lib().oracle_comb_rows_exact(q, r, c0, M, complex(amp).real, complex(amp).imag, s, r_.size, _ptr(r_), _ptr(out))
    return out.view(np.complex128)


def comb_probabilities_vec(q: int, r: int, c0: int, M: int, rows) -> np.ndarray:
    """comb_probabilities for many rows at once (same arithmetic, numpy).

    Exact integer reduction without overflow for q <= 2^32, r < 2^16, M < 2^20:
    a = c r mod q < 2^32 from a product < 2^48, then b = a M mod q from a
    product < 2^52 (c r M mod q = (c r mod q) M mod q).
    """
    if q > 1 << 32 or r >= 1 << 16 or M >= 1 << 20:
        return comb_probabilities(q, r, c0, M, rows)
    c = np.asarray(rows, dtype=np.uint64)
    qq, half = np.uint64(q), np.uint64(q // 2)
    a = (c * np.uint64(r)) % qq
    b = (a * np.uint64(M)) % qq
    a_s = np.where(a > half, a.astype(np.float64) - float(q), a.astype(np.float64))
    b_s = np.where(b > half, b.astype(np.float64) - float(q), b.astype(np.float64))
    with np.errstate(divide="ignore", invalid="ignore"):
        num = np.sin(np.pi * (b_s / q))
        den = np.sin(np.pi * (a_s / q))
        out = (num * num) / (float(q) * M * den * den)
    out[a == 0] = M / q
    return out
