"""One exact Born-rule read (shb_sample_index) over q = 2^30 probabilities of
the n=32399 attempt (computed once with the DFT): ncu launch-list target."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

q, M, c0, r = 1 << 30, 67025, 10943, 16020
# cheaper stand-in spectrum with the same size/scale: a sparse comb (M = 1031)
out, prob, _ = dev.dft_uniform(complex(1 / math.sqrt(1031)), 1031, 12345, 1_000_003, q, 0, q)
del out
for u in (0.3, 0.7):
    print(dev.sample_index(prob, u))
torch.cuda.synchronize()
