"""FP32 uniform-path timing per library variant (K outputs per thread)."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import _native as nat  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402

q, c0, r, M = 1 << 24, 29, 116, 144631
for so in sorted(Path(nat.LIB_PATH.parent / "_variants").glob("*.so")):
    nat._lib = nat.load(so)
    fn = lambda: dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp32")  # noqa: E731
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"lib": so.name, "ms": round(ms, 2), "terms_per_s": q * M / ms * 1e3}))
