"""int8 tensor-core FP64 DFT variants (scripts/build_i8_variants.sh): time and
agreement with the DMMA FP64 spectrum at q = 2^24 and q = 2^30 (uniform combs)."""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import _native as nat  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402

libs = sorted(Path(nat.LIB_PATH.parent / "_variants").glob("libshorb200_i8_*.so")) + [nat.LIB_PATH]
cases = [(1 << 24, 29, 116, 144631), (1 << 26, 4828, 300, 201075), (1 << 26, 10943, 900, 67025)]
if "big" in sys.argv:
    cases.append((1 << 30, 10943, 16020, 67025))
for q, c0, r, M in cases:
    amp = complex(1 / math.sqrt(M))
    nat._lib = nat.load(nat.LIB_PATH)
    os.environ["SHB_DFT_ENGINE"] = "mma"
    o64, _, _ = dev.dft_uniform(amp, M, c0, r, q, 0, q, precision="fp64")
    vmax = float(o64.abs().max())
    os.environ["SHB_DFT_ENGINE"] = "i8"
    for so in libs:
        nat._lib = nat.load(so)
        fn = lambda: dev.dft_uniform(amp, M, c0, r, q, 0, q, precision="fp64")  # noqa: E731
        o = fn()
        del o
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, p, bs = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"q": f"2^{q.bit_length() - 1}", "lib": so.name, "ms": round(ms, 2),
                          "Gterms/s": round(q * M / ms / 1e6, 1),
                          "max_dV_over_max_V": float((out - o64).abs().max()) / vmax}), flush=True)
        del out, p, bs
        torch.cuda.empty_cache()
