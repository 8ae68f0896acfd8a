"""Time every sub-operation of one device attempt (host wall clock around
synchronised calls) to locate non-DFT overhead.  Usage:
    python scripts/step_breakdown.py [n] [seed]
"""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402
from paper_1801_01434_b200 import numtheory as nt  # noqa: E402
from paper_1801_01434_b200 import qstate, shor  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32399
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 8
q = nt.choose_register_width(n, 32).q
T = {}


def timed(name, fn, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn(*a, **k)
    torch.cuda.synchronize()
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1000
    return r


for rep in range(3):
    T.clear()
    s = qstate.Sampler(seed)
    x = shor._draw_base(n, s)
    res = timed("modexp", dev.modexp, x, n, q)
    counts = timed("class_counts", dev.class_counts, res, n)
    ch = timed("counts_d2h", lambda: counts.cpu().numpy())
    a_unif = complex(1.0 / math.sqrt(q))
    w0 = qstate.uniform_weight(a_unif)
    k = timed("draw_class(host)", qstate.draw_class, ch, w0, s.uniform())
    sup = timed("compact_eq", dev.compact_eq, res, k)
    M = int(sup.numel())
    amp = timed("collapsed_amp(host)", qstate.collapsed_amplitude, a_unif, w0, M)
    a0, stride, length = timed("progression", dev.support_progression, sup)
    del res
    out, prob, bsum = timed("dft_uniform", dev.dft_uniform, amp, length, a0, stride, q, 0, q)
    norm2 = timed("dsum(bsum)", dev.dsum, bsum)
    m, tot = timed("sample_index", dev.sample_index, prob, s.uniform())
    del out, prob, bsum
    print(f"rep {rep}: " + ", ".join(f"{k}={v:.2f}ms" for k, v in T.items()), flush=True)
print("m", m, "M", M, "norm2", norm2)
