"""Time real-A DMMA variants (scripts/build_mma_real_variants.sh) at q = 2^24 on
the n=3127 comb: uniform comb and real generic amplitudes, FP64."""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_01434_b200 import _native as nat  # noqa: E402

os.environ["SHB_DFT_ENGINE"] = "mma"
from paper_1801_01434_b200 import device as dev  # noqa: E402

q, c0, r, M = 1 << 24, 29, 116, 144631
rng = np.random.default_rng(0)
amps_h = rng.standard_normal(M) + 0j
amps_h /= np.linalg.norm(amps_h)
amps = torch.from_numpy(amps_h.view(np.float64)).cuda()
ref = None
for so in sorted(Path(nat.LIB_PATH.parent / "_variants").glob("*.so")) + [nat.LIB_PATH]:
    nat._lib = nat.load(so)
    res = {"lib": so.name}
    for name, fn in (("generic_real", lambda: dev.dft(amps, M, c0, r, q, 0, q, real=True)),
                     ("uniform", lambda: dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[name] = {"ms": round(ms, 2), "Gterms/s": round(q * M / ms / 1e6, 1),
                     "TF_exec": round(4 * q * M / ms / 1e9, 2)}
        v = out[0][:4096].cpu().numpy()
        if name == "uniform":
            if ref is None:
                ref = v
            res[name]["maxdiff_vs_first"] = float(np.max(np.abs(v - ref)))
    print(json.dumps(res), flush=True)
