"""Every BASELINE.json config on one GPU through the public API (shor.run_shor),
beside the CPU port of the reference dense rows timed on this host's cores.
Prints one JSON line per config.

    python scripts/configs_table.py [--skip-46927]
"""
import json
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1801_01434_b200 import qft, shor  # noqa: E402

CONFIGS = [  # (label, n, seed, base_override)
    ("configs[0] n=15 x=7 q=2^8", 15, 0, 7),
    ("configs[1] n=221 q=2^16", 221, 0, None),
    ("configs[2] n=3127 q=2^24", 3127, 0, None),
    ("configs[3] n=32399 q=2^30 (seed 8)", 32399, 8, None),
    ("configs[4] n=46927 q=2^32", 46927, 0, None),
]


def cpu_rate(q, x, n, k, m_support, seconds=3.0):
    """Oracle port of the reference dense rows for the attempt's collapsed comb."""
    r = next(p for p in range(1, n + 1) if pow(x, p, n) == 1)
    c0 = next(j for j in range(r) if pow(x, j, n) == k)
    M = (q - 1 - c0) // r + 1
    supp = c0 + r * np.arange(M, dtype=np.uint64)
    amps = np.full(M, 1 / math.sqrt(M), dtype=np.complex128)
    thr = len(os.sched_getaffinity(0))
    rows, t0 = 0, time.perf_counter()
    rng = np.random.default_rng(0)
    while time.perf_counter() - t0 < seconds:
        oracle.dft_rows(supp, amps, q, rng.integers(0, q, 4 * thr, dtype=np.uint64), True, thr)
        rows += 4 * thr
    el = time.perf_counter() - t0
    return rows * M / el, thr, M


def main():
    skip = "--skip-46927" in sys.argv
    for label, n, seed, base in CONFIGS:
        if skip and n == 46927:
            continue
        cfg = shor.ShorConfig(n=n, seed=seed, base_override=base, kernel="dense", max_width=32,
                              plan=qft.KernelPlan())
        shor.run_shor(cfg) if n < 32399 else None  # warm (small configs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = shor.run_shor(cfg)
        wall = time.perf_counter() - t0
        qatt = [a for a in res.attempts if a.q]
        terms = 0
        for a in qatt:
            r = next(p for p in range(1, n + 1) if pow(a.x, p, n) == 1)
            c0 = next(j for j in range(r) if pow(a.x, j, n) == a.k)
            terms += a.q * ((a.q - 1 - c0) // r + 1)
        qft_s = sum(a.phase_times["qft"] for a in qatt)
        line = {"config": label, "factors": res.factors, "attempts": len(res.attempts),
                "quantum_attempts": len(qatt), "wall_s": wall, "qft_s": qft_s,
                "phase_terms": terms, "gpu_terms_per_s": terms / qft_s if qft_s else None,
                "ms": [a.m for a in res.attempts]}
        if qatt:
            a = qatt[-1]
            rate, thr, M = cpu_rate(a.q, a.x, n, a.k, None)
            line.update({"cpu_port_terms_per_s": rate, "cpu_threads": thr,
                         "cpu_est_qft_s": terms / rate,
                         "gpu_speedup_vs_cpu_port": (terms / qft_s) / rate if qft_s else None})
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
