"""Golden (u, m) pairs from the REFERENCE's own spectra (run in the build
container; the reference is not on GPU boxes):

* n=3127 seed 0 attempt 1 (q=2^24): reference fft engine (ShorConfig default)
* n=221 seed 0 attempt 2 (q=2^16): reference dense engine

m = qstate.sample_part1(post, Forced([u])) for 1000 seeded u each, plus u
values placed exactly on / next to CDF boundaries.  Output: sampling_sweep.npz
"""
import os
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from shorsim import qft, qstate, shor  # noqa: E402

OUT = Path(__file__).resolve().parent


class Forced(qstate.Sampler):
    def __init__(self, values):
        super().__init__(0)
        self._v = list(values)

    def uniform(self):
        return self._v.pop(0)


def sweep(n, attempt, engine):
    s = qstate.Sampler(0)
    for _ in range(attempt):
        x = shor._draw_base(n, s)
        q = 1 << (n * n - 1).bit_length()
        reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
        k, rc = qstate.measure_part2(reg, s)
        if _ < attempt - 1:
            s.uniform()  # the m draw of the earlier attempt
    if engine == "fft":
        V = qft.fft_dft(rc.amplitudes)
    else:
        V = qft.dense_dft(rc.amplitudes, qft.build_twiddles(q), qft.KernelPlan())
    post = replace(rc, amplitudes=V)
    p = np.abs(V) ** 2
    cum = np.cumsum(p)
    rng = np.random.default_rng(n)
    us = list(rng.random(1000))
    # u placed so that u*total lands exactly on / just around peak CDF values
    peaks = np.argsort(p)[-20:]
    for i in peaks:
        for t in (cum[i], np.nextafter(cum[i], 0), np.nextafter(cum[i], 2)):
            us.append(float(t / cum[-1]))
    ms = [qstate.sample_part1(post, Forced([u])) for u in us]
    return x, k, np.array(us), np.array(ms, dtype=np.int64)


def main():
    x1, k1, u1, m1 = sweep(3127, 1, "fft")
    x2, k2, u2, m2 = sweep(221, 2, "dense")
    np.savez_compressed(OUT / "sampling_sweep.npz", n3127_x=x1, n3127_k=k1, n3127_u=u1, n3127_m=m1,
                        n221_x=x2, n221_k=k2, n221_u=u2, n221_m=m2)
    print("n3127", x1, k1, len(u1), "n221", x2, k2, len(u2))


if __name__ == "__main__":
    main()
