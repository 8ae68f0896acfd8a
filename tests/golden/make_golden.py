"""Generate golden vectors by running the REFERENCE package (not our code).

Run in the build container only (the reference does not exist on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [qreg|gates]

It imports ``shorsim`` from /root/reference/pkg/src (read-only; the numba cache
is redirected to /tmp so nothing is written into the reference tree) and
writes small fixtures next to this script.  The fixtures, not the reference,
are what tests/ read at run time.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from dataclasses import asdict, replace
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from shorsim import numtheory as nt  # noqa: E402
from shorsim import qft, qstate, shor  # noqa: E402
from shorsim import _kernels  # noqa: E402

OUT = Path(__file__).resolve().parent


class Forced(qstate.Sampler):
    """Sampler whose uniform() replays scripted values."""

    def __init__(self, values):
        super().__init__(0)
        self._vals = list(values)

    def uniform(self):
        return self._vals.pop(0)


def outcome_dict(o):
    return {"kind": o.kind, "factors": list(o.factors) if o.factors else None,
            "reason": o.reason, "shortcut": o.shortcut}


def trace_dict(t):
    return {
        "x": t.x, "q": t.q, "k": t.k, "m": t.m,
        "candidate": None if t.candidate is None else {
            "p": t.candidate.p, "source_convergent": list(t.candidate.source_convergent),
            "multiplier": t.candidate.multiplier},
        "outcome": outcome_dict(t.outcome),
    }


def f64bits(v: float) -> str:
    return np.float64(v).view(np.uint64).item().__format__("016x")


def kats():
    d = {}
    d["modpow"] = [[b, e, m, nt.modpow(b, e, m)] for b, e, m in
                   [(7, 0, 13), (2, 13, 15), (2, 4, 15), (3, 200, 1000003), (12345, 67890, 46927)]]
    d["gcd"] = [[a, b, nt.gcd(a, b)] for a, b in [(12, 8), (7, 1), (3, 15), (0, 9)]]
    d["register_width"] = [[n, nt.choose_register_width(n, 32).q, nt.choose_register_width(n, 32).w]
                           for n in (15, 21, 77, 221, 3127, 32399, 46927)]
    d["classical_period"] = [[x, n, nt.classical_period(x, n)] for x, n in
                             [(2, 15), (7, 15), (2, 21), (2, 32399), (7, 32399), (3, 46927), (2, 3127)]]
    d["convergents"] = [[m, q, [list(c) for c in nt.convergents(m, q)]] for m, q in
                        [(85, 512), (192, 256), (0, 256), (57344, 65536), (874074104, 1 << 30)]]
    ep = []
    for m, q, n, x in [(192, 256, 15, 2), (85, 512, 21, 2), (0, 256, 15, 2), (57344, 65536, 221, 5),
                       (578525, 1 << 24, 3127, 1991), (874074104, 1 << 30, 32399, 8477),
                       (342163047, 1 << 30, 32399, 10594)]:
        r = nt.extract_period(m, q, n, x)
        if isinstance(r, nt.PeriodCandidate):
            ep.append([m, q, n, x, {"p": r.p, "source_convergent": list(r.source_convergent),
                                    "multiplier": r.multiplier}])
        else:
            ep.append([m, q, n, x, outcome_dict(r)])
    d["extract_period"] = ep
    d["derive_factors"] = [[n, x, p, outcome_dict(nt.derive_factors(n, x, p))] for n, x, p in
                           [(15, 2, 4), (15, 14, 2), (21, 2, 6), (32399, 8477, 5340), (3127, 1991, 116)]]
    # entangle residue vectors
    ent = []
    for q, x, n in [(16, 2, 15), (8, 1, 15), (8, 7, 15), (64, 5, 221), (1 << 12, 20637, 32399)]:
        reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
        ent.append([q, x, n, reg.residues.tolist()])
    d["entangle"] = ent
    # twiddles
    d["twiddles"] = {str(q): [[z.real, z.imag] for z in qft.build_twiddles(q).roots] for q in (2, 4, 8)}
    # init_uniform amplitude bits for even and odd widths
    d["init_uniform"] = [[q, f64bits(qstate.init_uniform(q).amplitudes[0].real)] for q in (2, 4, 8, 256, 512, 1 << 15)]
    return d


def collapse_info(reg_c, k):
    amps = reg_c.amplitudes
    supp = np.flatnonzero(amps)
    info = {"k": k, "M": int(supp.size), "c0": int(supp[0]),
            "r": int(supp[1] - supp[0]) if supp.size > 1 else 0,
            "amp_re_bits": f64bits(amps[supp[0]].real), "amp_im_bits": f64bits(amps[supp[0]].imag),
            "uniform": bool(np.all(amps[supp] == amps[supp[0]])),
            "comb": bool(supp.size < 2 or np.all(np.diff(supp) == supp[1] - supp[0]))}
    return info


def measure_sweep():
    """k / support / amplitude for many draws, odd and even widths."""
    rows = []
    for n in (15, 21, 33, 35, 143, 221):
        q = nt.choose_register_width(n, 32).q
        for x in range(2, min(n - 1, 40)):
            if math.gcd(x, n) != 1:
                continue
            reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
            for u in (0.0, 0.13, 0.5, 0.77, 0.999999):
                k, rc = qstate.measure_part2(reg, Forced([u]))
                info = collapse_info(rc, k)
                info.update({"n": n, "x": x, "q": q, "u": u})
                rows.append(info)
    return rows


def spectra():
    res = {}
    # n=15, x=7 (configs[0]) seed 0 attempt: full spectrum, bitwise, dense engine
    cfg = shor.ShorConfig(n=15, base_override=7, seed=0, kernel="dense")
    s = qstate.Sampler(0)
    reg = qstate.entangle_modexp(qstate.init_uniform(256), 7, 15)
    k, rc = qstate.measure_part2(reg, s)
    tw = qft.build_twiddles(256)
    V = qft.dense_dft(rc.amplitudes, tw, qft.KernelPlan())
    m = qstate.sample_part1(replace(rc, amplitudes=V), s)
    res["n15"] = dict(q=256, n=15, x=7, info=collapse_info(rc, k), m=m,
                      rows=np.arange(256, dtype=np.uint64), V=V)
    # n=15 x=2 forced k=1
    reg = qstate.entangle_modexp(qstate.init_uniform(256), 2, 15)
    k, rc = qstate.measure_part2(reg, Forced([0.0]))
    V = qft.dense_dft(rc.amplitudes, tw, qft.KernelPlan())
    res["n15x2"] = dict(q=256, n=15, x=2, info=collapse_info(rc, k), m=-1,
                        rows=np.arange(256, dtype=np.uint64), V=V)
    # n=221 seed 0: both attempts (x=140 then x=5), dense engine, full spectra
    q = 1 << 16
    tw = qft.build_twiddles(q)
    s = qstate.Sampler(0)
    for tag in ("n221a1", "n221a2"):
        x = shor._draw_base(221, s)
        reg = qstate.entangle_modexp(qstate.init_uniform(q), x, 221)
        k, rc = qstate.measure_part2(reg, s)
        t0 = time.time()
        V = qft.dense_dft(rc.amplitudes, tw, qft.KernelPlan())
        print(f"  {tag}: dense q=2^16 in {time.time() - t0:.1f}s", flush=True)
        m = qstate.sample_part1(replace(rc, amplitudes=V), s)
        info = collapse_info(rc, k)
        # keep 4096 sampled rows + all rows with p > 1e-6 (the peaks)
        rng = np.random.default_rng(221)
        p = np.abs(V) ** 2
        rows = np.unique(np.concatenate([rng.choice(q, 4096, replace=False), np.flatnonzero(p > 1e-6),
                                         [0, 1, q // 2, q - 1]])).astype(np.uint64)
        res[tag] = dict(q=q, n=221, x=x, info=info, m=m, rows=rows, V=V[rows.astype(np.int64)],
                        p_total=float(np.cumsum(p)[-1]))
    # n=3127 seed 0 attempt 1: collapse + 192 sampled rows via the reference kernel itself
    q = 1 << 24
    s = qstate.Sampler(0)
    x = shor._draw_base(3127, s)
    reg = qstate.entangle_modexp(qstate.init_uniform(q), x, 3127)
    k, rc = qstate.measure_part2(reg, s)
    info = collapse_info(rc, k)
    del reg
    tw = qft.build_twiddles(q)
    rng = np.random.default_rng(3127)
    r = info["r"]
    peaks = [(j * q + r // 2) // r for j in range(0, r, 7)]  # near multiples of q/r
    rows = np.unique(np.concatenate([rng.choice(q, 160, replace=False), peaks, [0, 1, q - 1]])).astype(np.int64)
    V = np.empty(rows.size, dtype=np.complex128)
    t0 = time.time()
    for i, c in enumerate(rows):
        out = np.empty(1, dtype=np.complex128)
        _kernels.partial_row_sums(out, rc.amplitudes, tw.roots, q, int(c), int(c) + 1, 0, q)
        V[i] = out[0]
    V *= 1.0 / math.sqrt(q)
    print(f"  n3127: {rows.size} rows in {time.time() - t0:.1f}s", flush=True)
    res["n3127"] = dict(q=q, n=3127, x=x, info=info, m=-1, rows=rows.astype(np.uint64), V=V)
    return res


def random_states():
    """Random unit states -> reference dense and tiled outputs."""
    out = {}
    rng = np.random.default_rng(1801)
    for q in (16, 256, 1024, 4096):
        z = rng.standard_normal(q) + 1j * rng.standard_normal(q)
        z /= np.linalg.norm(z)
        tw = qft.build_twiddles(q)
        d = qft.dense_dft(z, tw, qft.KernelPlan())
        t = qft.tiled_dft(z, tw, qft.KernelPlan(tiles=8))
        out[q] = dict(state=z, dense=d, tiled8=t)
    # sparse irregular support (not a comb) to exercise the generic path
    q = 2048
    z = np.zeros(q, dtype=np.complex128)
    idx = np.sort(rng.choice(q, 37, replace=False))
    z[idx] = rng.standard_normal(37) + 1j * rng.standard_normal(37)
    z /= np.linalg.norm(z)
    tw = qft.build_twiddles(q)
    out["sparse2048"] = dict(state=z, dense=qft.dense_dft(z, tw, qft.KernelPlan()),
                             tiled8=qft.tiled_dft(z, tw, qft.KernelPlan(tiles=8)))
    return out


def traces():
    runs = []
    for n, kw in [(15, dict(base_override=7, seed=0, kernel="dense")),
                  (15, dict(seed=0, kernel="dense")),
                  (221, dict(seed=0, kernel="dense")),
                  (77, dict(seed=0, kernel="fft")), (143, dict(seed=0, kernel="fft")),
                  (231, dict(seed=0, kernel="fft")), (255, dict(seed=0, kernel="fft")),
                  (423, dict(seed=0, kernel="fft")),
                  (3127, dict(seed=0, kernel="fft")),
                  ] + [(n, dict(seed=s, kernel="dense")) for n in (15, 21, 33, 35) for s in range(6)]:
        t0 = time.time()
        r = shor.run_shor(shor.ShorConfig(n=n, **kw))
        runs.append({"n": n, "cfg": kw, "factors": r.factors, "succeeded": r.succeeded,
                     "attempts": [trace_dict(t) for t in r.attempts]})
        print(f"  run_shor n={n} {kw}: {r.factors} in {time.time() - t0:.1f}s", flush=True)
    return runs


def sampling():
    """sample_part1 on reference spectra with scripted draws (exact m)."""
    rows = []
    q = 1 << 12
    rng = np.random.default_rng(7)
    z = rng.standard_normal(q) + 1j * rng.standard_normal(q)
    z /= np.linalg.norm(z)
    reg = qstate.CompositeRegister(q=q, amplitudes=z, residues=np.zeros(q, dtype=np.int64))
    us = [0.0, 1e-9, 0.25, 0.5, 0.999999999, float(np.nextafter(1.0, 0.0))] + rng.random(40).tolist()
    for u in us:
        rows.append([u, qstate.sample_part1(reg, Forced([u]))])
    return {"state": z, "draws": rows}


def qreg_dumps():
    """QREG files written by the reference's own dump path: run_shor with
    ShorConfig.dump_state_path (shor.py:113-114 -> qstate.dump_state,
    qstate.py:121-130).  Each attempt overwrites the file, so it holds the
    last quantum attempt's post-QFT spectrum; stored gzip-compressed."""
    import gzip
    import tempfile
    out = {}
    for tag, n, kw in [("n15", 15, dict(base_override=7, seed=0)), ("n221", 221, dict(seed=0))]:
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "ref.qreg")
            r = shor.run_shor(shor.ShorConfig(n=n, kernel="dense", dump_state_path=path, **kw))
            raw = Path(path).read_bytes()
        (OUT / f"qreg_{tag}.qreg.gz").write_bytes(gzip.compress(raw, mtime=0))
        last = [t for t in r.attempts if t.k is not None][-1]
        out[tag] = {"n": n, "cfg": kw, "factors": r.factors, "bytes": len(raw),
                    "last_attempt": trace_dict(last)}
        print(f"  qreg {tag}: {len(raw)} bytes, last attempt x={last.x} m={last.m}", flush=True)
    (OUT / "qreg_dumps.json").write_text(json.dumps(out, indent=1))


def gates():
    """The reference's gate primitives and gate-level QFT (qft.py:164-231) on
    random states: outputs for a bitwise check of the device gate kernels."""
    rng = np.random.default_rng(1434)
    out = {}
    q = 64
    z = rng.standard_normal(q) + 1j * rng.standard_normal(q)
    z[5] = complex(-0.0, -0.0)  # signed zeros through the complex products
    z[9] = complex(0.0, -0.0)
    out["state64"] = z
    for b in range(6):
        out[f"hadamard_{b}"] = qft.apply_hadamard(z, b)
    for c, t, ang in [(0, 1, 0.7), (5, 2, -1.3), (3, 4, 2.0 * np.pi / 8), (1, 5, 1e-3)]:
        out[f"cphase_{c}_{t}"] = qft.apply_controlled_phase(z, c, t, ang)
    out["bitrev64"] = qft.bit_reverse_permute(z)
    for w in (1, 4, 8, 12):
        s = rng.standard_normal(1 << w) + 1j * rng.standard_normal(1 << w)
        s /= np.linalg.norm(s)
        out[f"circuit_in_{w}"] = s
        out[f"circuit_out_{w}"] = qft.circuit_qft(s)
    np.savez_compressed(OUT / "gates.npz", **out)
    print("gates.npz written", flush=True)


def main():
    if sys.argv[1:] == ["qreg"]:
        qreg_dumps()
        return
    if sys.argv[1:] == ["gates"]:
        gates()
        return
    t0 = time.time()
    k = kats()
    k["measure_sweep"] = measure_sweep()
    k["traces"] = traces()
    (OUT / "kats.json").write_text(json.dumps(k, indent=1))
    print("kats.json written", flush=True)
    sp = spectra()
    for tag, d in sp.items():
        np.savez_compressed(OUT / f"spectrum_{tag}.npz", q=d["q"], n=d["n"], x=d["x"], m=d["m"],
                            info=json.dumps(d["info"]), rows=d["rows"], V=d["V"],
                            p_total=d.get("p_total", np.nan))
    print("spectra written", flush=True)
    rs = random_states()
    np.savez_compressed(OUT / "random_states.npz",
                        **{f"{key}_{f}": v for key, d in rs.items() for f, v in d.items()})
    smp = sampling()
    np.savez_compressed(OUT / "sampling.npz", state=smp["state"], draws=np.array(smp["draws"]))
    qreg_dumps()
    gates()
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
