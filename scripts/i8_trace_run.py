"""clock64 timeline of CTA 0 of the int8 FP64 DFT (SHB_I8_TRACE variant built by
scripts/build_i8_variants.sh as libshorb200_i8_trace.so): per super-block the
worker (tid 0 / tid 160) and MMA-issuer events, at the bench config q = 2^30."""
import ctypes
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["SHB_DFT_ENGINE"] = "i8"

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1801_01434_b200 import _native as nat  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402

nat._lib = nat.load(nat.LIB_PATH.parent / "_variants" / "libshorb200_i8_trace.so")
q, c0, r, M = (1 << 30, 10943, 16020, 67025) if "big" in sys.argv else (1 << 24, 29, 116, 144631)
out = dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp64")
torch.cuda.synchronize()
buf = np.zeros(20000, dtype=np.uint64)
nat._lib.shb_i8_trace.argtypes = [ctypes.c_void_p]
print("rc", nat._lib.shb_i8_trace(buf.ctypes.data))
t0 = int(buf[10000])
rel = lambda v: int(v) - t0 if v else None  # noqa: E731
nsb = -(-M // (64 * 96))
for it in range(3):
    for who, base in (("w0", 0), ("w160", 5000)):
        b = base + it * 1000
        print(f"tile {it} {who}: start {rel(buf[b])} G_built {rel(buf[b + 1])}")
        for sb in range(min(nsb, 6)):
            e = [rel(buf[b + 2 + 8 * sb + k]) for k in range(6)]
            print(f"   sb{sb}: re_wait {e[0]} re_ok {e[1]} re_done {e[2]} im_ok {e[3]} im_done {e[4]} seeded {e[5]}")
    b = 10000 + it * 1000
    print(f"tile {it} MMA: a_ready_ok {rel(buf[b])}")
    for sb in range(min(nsb, 6)):
        e = [rel(buf[b + 1 + 8 * sb + k]) for k in range(6)]
        print(f"   sb{sb}: re(empty_wait {e[0]} ok {e[1]} issued {e[2]})  im(empty_wait {e[3]} ok {e[4]} issued {e[5]})")
