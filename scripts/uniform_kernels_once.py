"""Launch the uniform-comb DFT once in FP64 and once in FP32 at q = 2^24 on the
n=3127 comb (M = 144631) -- the target of the ncu --set full capture."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

q, c0, r, M = 1 << 24, 29, 116, 144631
amp = complex(1 / math.sqrt(M))
for prec in ("fp64", "fp32"):
    dev.dft_uniform(amp, M, c0, r, q, 0, q, precision=prec)
torch.cuda.synchronize()
print("ok")
