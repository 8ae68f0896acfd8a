"""One launch of the int8 tensor-core FP64 DFT (uniform comb) at q = 2^24, or at
the bench configs q = 2^30 with `big` (seed 8) / `big2` (seed 2): ncu target."""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SHB_DFT_ENGINE"] = "i8"

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

cfg = {"big": (1 << 30, 10943, 16020, 67025), "big2": (1 << 30, 4828, 5340, 201075), "mid8": (1 << 26, 10943, 900, 67025), "mid2": (1 << 26, 4828, 300, 201075)}
q, c0, r, M = next((v for k, v in cfg.items() if k in sys.argv), (1 << 24, 29, 116, 144631))
out = dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp64")
torch.cuda.synchronize()
print("ok")
