"""Time both DFT instantiations at q = 2^24 on the n=3127 comb (M = 144631):
uniform-comb kernel and the generic TMA-staged kernel with random complex
amplitudes (checked against oracle rows).  Prints one JSON line."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402

q, c0, r, M = 1 << 24, 29, 116, 144631
rng = np.random.default_rng(0)
amps_h = (rng.standard_normal(M) + 1j * rng.standard_normal(M))
amps_h /= np.linalg.norm(amps_h)
amps = torch.from_numpy(amps_h.view(np.float64)).cuda()
res = {}


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


for prec in ("fp64", "fp32"):
    ms, (out, prob, _) = timed(lambda: dev.dft(amps, M, c0, r, q, 0, q, precision=prec))
    rows = rng.choice(q, 256, replace=False).astype(np.uint64)
    ref = oracle.dft_rows(c0 + r * np.arange(M, dtype=np.uint64), amps_h, q, rows)
    got = out.cpu().numpy().view(np.complex128)[rows.astype(np.int64)]
    pr, pg = np.abs(ref) ** 2, np.abs(got) ** 2
    res[f"generic_{prec}"] = {"ms": ms, "TFLOP/s": 8 * q * M / ms / 1e9, "terms/s": q * M / ms * 1e3,
                              "max_abs_dV": float(np.max(np.abs(got - ref))),
                              "max_dp_over_maxp": float(np.max(np.abs(pg - pr)) / np.max(pr))}
    ms, _ = timed(lambda: dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision=prec))
    res[f"uniform_{prec}"] = {"ms": ms, "TFLOP/s": 8 * q * M / ms / 1e9, "terms/s": q * M / ms * 1e3}
print(json.dumps(res))
