"""Every libshorb200 kernel at small sizes, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per run)."""
import ctypes
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_01434_b200 import _native as nat  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402
from paper_1801_01434_b200 import qft, qstate, shor  # noqa: E402

q, n, x = 1 << 14, 221, 140
res = dev.modexp(x, n, q)
dev.modexp(3, 1000003, 5000)                       # Barrett64 path
c = dev.class_counts(res, n)                        # smem histogram
dev.class_counts(dev.modexp(3, 1000003, 5000), 1000003)   # global-atomic histogram
k = int(res[17].item())
sup = dev.compact_eq(res, k)
sup2 = dev.compact_eq(res, k, expected=int(c[k].item()))
a0, st, ln = dev.support_progression(sup)
amps = dev.fill_progression(sup, sup.numel(), a0, st, ln, complex(0.1, 0.2))
for prec in ("fp64", "fp32"):
    dev.dft(amps, ln, a0, st, q, 0, q, precision=prec)
    dev.dft(amps, ln, a0, st, q, 0, q, tiles=4, precision=prec)
    dev.dft_uniform(complex(0.1), ln, a0, st, q, 100, 1000, precision=prec)
    dev.dft_uniform(complex(0.1), ln, a0, st, q, 0, q, tiles=2, precision=prec)
z = np.random.default_rng(0).standard_normal(4096) + 0j
zt = torch.from_numpy(z.view(np.float64)).cuda()
dev.state_progression(zt)
dev.gather_progression(zt, 0, 1, 4096)
dev.progression_uniform(dev.gather_progression(zt, 0, 1, 4096), 4096)
p = dev.probabilities(zt)
dev.dsum(p)
rng = np.random.default_rng(1)
for arr in (np.abs(rng.standard_normal(20000)) ** 4, (2 * rng.integers(0, 1024, 20000) + 1) * 2.0 ** -54,
            np.where(rng.random(20000) < 0.9, 0.0, rng.random(20000))):
    pt = torch.from_numpy(arr).cuda()
    dev.cumsum_total(pt)
    dev.cumsum_search(pt, 0.3 * float(arr.sum()))
    dev.sample_index(pt, 0.7)
lib = nat.load()
out = np.empty_like(z)
nat.check(lib.shb_dense_dft_host(ctypes.c_void_p(z.ctypes.data), 4096, 1, 0, ctypes.c_void_p(out.ctypes.data)))
rows = np.empty(8, dtype=np.complex128)
nat.check(lib.shb_partial_row_sums_host(ctypes.c_void_p(rows.ctypes.data), ctypes.c_void_p(z.ctypes.data), None,
                                        4096, 10, 18, 100, 900))
tf = ctypes.c_double()
nat.check(lib.shb_fp64_peak(0.01, ctypes.byref(tf), None))
r = shor.run_shor(shor.ShorConfig(n=221, seed=0, kernel="dense"))
torch.cuda.synchronize()
print("ok", r.factors)
