"""Bitwise comparison of the int8 engine's spectrum between two builds
(paper_1801_01434_b200/_variants/libshorb200_i8_<name>.so vs the in-tree
library) on the seed-2 / seed-8 combs at q = 2^26 and 2^24: a change meant
to keep every output bit (e.g. an arithmetic rewrite with the same single
rounding) must print equal=True."""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SHB_DFT_ENGINE"] = "i8"

import torch  # noqa: E402

from paper_1801_01434_b200 import _native as nat  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402

other = nat.LIB_PATH.parent / "_variants" / f"libshorb200_i8_{sys.argv[1]}.so"
for q, c0, r, M in [(1 << 24, 29, 116, 144631), (1 << 26, 4828, 300, 201075), (1 << 26, 10943, 900, 67025),
                    (1 << 21, 7, 13, 100003), (1 << 21, 7, 13, 24577)]:
    outs = []
    for so in (other, nat.LIB_PATH):
        nat._lib = nat.load(so)
        o, p, b = dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp64")
        torch.cuda.synchronize()
        outs.append((o, p))
    print(f"q=2^{q.bit_length() - 1} M={M} equal={torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])}",
          flush=True)
