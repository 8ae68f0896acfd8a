"""clock64 timeline of CTA 0 of the int8 FP64 DFT (SHB_I8_TRACE variant built by
scripts/build_i8_variants.sh as libshorb200_i8_trace.so): per super-block the
MMA issuer (wait a_empty, issued), drain warp 0 (wait a_full, drained), per
tile the G builder (wait g_empty, built) and the drain's tile end."""
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

nat._lib = nat.load(nat.LIB_PATH.parent / "_variants" / os.environ.get("TRACE_LIB", "libshorb200_i8_trace.so"))
cfg = {"big": (1 << 30, 10943, 16020, 67025), "big2": (1 << 30, 4828, 5340, 201075)}
q, c0, r, M = next((v for k, v in cfg.items() if k in sys.argv), (1 << 24, 29, 116, 144631))
for _ in range(2):
    out = dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp64")
    torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
nat._lib.shb_i8_trace.argtypes = [ctypes.c_void_p]
print("rc", nat._lib.shb_i8_trace(buf.ctypes.data))
t0 = int(buf[4000])
rel = lambda v: int(v) - t0 if v else None  # noqa: E731
nsb = -(-M // int(os.environ.get("SBA", "16384")))
print(f"q=2^{q.bit_length() - 1} M={M} nsb={nsb}")
for it in range(4):
    print(f"tile {it}: MMA g_full wait {rel(buf[4000 + 4 * it])} ok {rel(buf[4001 + 4 * it])} | "
          f"G wait {rel(buf[5000 + 4 * it])} ok {rel(buf[5001 + 4 * it])} built {rel(buf[5002 + 4 * it])} | "
          f"drain tile start {rel(buf[2000 + 4 * it])} g_full {rel(buf[2001 + 4 * it])} "
          f"fold {rel(buf[2002 + 4 * it])} end {rel(buf[2003 + 4 * it])}")
    for sb in range(nsb):
        g = it * nsb + sb
        m = [rel(buf[4 * g + k]) for k in range(3)]
        d = [rel(buf[1000 + 4 * g + k]) for k in range(3)]
        print(f"   sb{sb}: MMA empty_wait {m[0]} ok {m[1]} issued {m[2]} | drain full_wait {d[0]} ok {d[1]} "
              f"loaded {d[2]}")
