"""The HBM-bound stages of one q = 2^30 attempt (n=32399, x=10594): modexp,
class histogram, compaction (count + scan + write), progression -- the
target of the ncu capture for their achieved DRAM bandwidth."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

n, x, q = 32399, 10594, 1 << 30
for _ in range(2):  # second pass is the steady state
    res = dev.modexp(x, n, q)
    counts = dev.class_counts(res, n)
    k = 31897
    sup = dev.compact_eq(res, k, expected=int(counts[k].item()))
    prog = dev.support_progression(sup)
    torch.cuda.synchronize()
    del res
print(prog)
