"""One launch of the FP32 tcgen05 DFT (uniform comb) at q = 2^24 and at the
bench config q = 2^30: ncu target."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

for q, c0, r, M in [(1 << 24, 29, 116, 144631), (1 << 30, 10943, 16020, 67025)]:
    out = dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp32")
    torch.cuda.synchronize()
    del out
    torch.cuda.empty_cache()
print("ok")
