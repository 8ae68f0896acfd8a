"""One launch each of the DMMA-engine DFT (generic complex, generic real, uniform) at q=2^24: ncu target."""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SHB_DFT_ENGINE"] = "mma"

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

q, c0, r, M = 1 << 24, 29, 116, 144631
a = np.random.default_rng(0).standard_normal(2 * M)
amps = torch.from_numpy(a).cuda()
dev.dft(amps, M, c0, r, q, 0, q)
ra = amps.clone().view(-1, 2)
ra[:, 1] = 0
dev.dft(ra.view(-1), M, c0, r, q, 0, q, real=True)
dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q)
torch.cuda.synchronize()
print("ok")
