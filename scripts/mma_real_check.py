"""Real-amplitude DMMA form vs the complex DMMA form vs the vector kernel:
accuracy against oracle rows and time, uniform comb and real generic amplitudes."""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


cases = [(1 << 12, 3, 7, 500), (1 << 16, 11, 12, 5461), (1 << 24, 29, 116, 144631)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases.append((1 << 30, 10943, 16020, 67025))
for q, c0, r, M in cases:
    rng = np.random.default_rng(q)
    amps_h = rng.standard_normal(M) + 0j
    amps_h /= np.linalg.norm(amps_h)
    amps = torch.from_numpy(amps_h.view(np.float64)).cuda()
    rows = np.unique(np.concatenate([rng.choice(q, 200, replace=False), [0, 1, q - 1]])).astype(np.uint64)
    supp = c0 + r * np.arange(M, dtype=np.uint64)
    ref_g = oracle.dft_rows(supp, amps_h, q, rows)
    ref_u = oracle.dft_rows(supp, np.full(M, 1 / math.sqrt(M) + 0j), q, rows)
    for eng, real in (("vector", "1"), ("mma", "0"), ("mma", "1")):
        os.environ["SHB_DFT_ENGINE"] = eng
        os.environ["SHB_MMA_REAL"] = real
        ms_g, (og, pg, bg) = timed(lambda: dev.dft(amps, M, c0, r, q, 0, q, real=True))
        ms_u, (ou, pu, bu) = timed(lambda: dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q))
        gg = og.cpu().numpy().view(np.complex128)[rows.astype(np.int64)]
        gu = ou.cpu().numpy().view(np.complex128)[rows.astype(np.int64)]
        key = f"q{q.bit_length()-1}_{eng}_real{real}"
        res = {"generic_real_ms": round(ms_g, 3), "generic_real_Gterms": round(q * M / ms_g / 1e6, 1),
               "generic_maxdV": float(np.max(np.abs(gg - ref_g))),
               "uniform_ms": round(ms_u, 3), "uniform_Gterms": round(q * M / ms_u / 1e6, 1),
               "uniform_maxdV": float(np.max(np.abs(gu - ref_u))),
               "norm_g": dev.dsum(bg), "norm_u": dev.dsum(bu)}
        print(json.dumps({key: res}), flush=True)
        del og, pg, bg, ou, pu, bu
        torch.cuda.empty_cache()
