"""FP32 fast path: tcgen05 (TMEM) form vs the mma.sync form -- time and
max|dp|/max p against the FP64 spectrum, uniform comb at q = 2^16/2^24/2^30."""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

cases = [(1 << 16, 11, 12, 5461), (1 << 24, 29, 116, 144631)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases.append((1 << 30, 10943, 16020, 67025))
for q, c0, r, M in cases:
    amp = complex(1 / math.sqrt(M))
    _, p64, _ = dev.dft_uniform(amp, M, c0, r, q, 0, q, precision="fp64")
    pmax = float(p64.max())
    for eng in ("mma", "tcgen05"):
        os.environ["SHB_FP32_ENGINE"] = eng
        fn = lambda: dev.dft_uniform(amp, M, c0, r, q, 0, q, precision="fp32")  # noqa: E731
        o = fn()
        del o
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, p32, bs = fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        err = float((p32 - p64).abs().max()) / pmax
        print(json.dumps({"q": f"2^{q.bit_length() - 1}", "engine": eng, "ms": round(ms, 3),
                          "Gterms/s": round(q * M / ms / 1e6, 1), "TFLOPs_bf16": round(8 * q * M / ms / 1e9, 1),
                          "max_dp_over_max_p": err, "norm": dev.dsum(bs)}), flush=True)
        del out, p32, bs
        torch.cuda.empty_cache()
