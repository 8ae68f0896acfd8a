import ctypes, math, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1801_01434_b200 import _native as nat, device as dev
nat._lib = nat.load(nat.LIB_PATH.parent / "_variants" / "libshorb200_tc05trace.so")
lib = nat._lib
lib.shb_tc05_trace.argtypes = [ctypes.c_void_p]
q, c0, r, M = 1 << 30, 10943, 16020, 67025
out = dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, 0, q, precision="fp32")
torch.cuda.synchronize()
buf = np.zeros(4096, dtype=np.uint64)
lib.shb_tc05_trace(buf.ctypes.data)
base = int(buf[0])
for it in range(3):
    w = [int(buf[it*100 + j]) - base if buf[it*100+j] else None for j in range(0, 20)]
    m = [int(buf[1000 + it*100 + j]) - base if buf[1000+it*100+j] else None for j in range(0, 20)]
    print("tile", it, "worker", w[:2], "sb(wait_full_start, full_ok, fold_end):", [tuple(w[2+3*s:5+3*s]) for s in range(5)], "end", int(buf[it*100+99]) - base)
    print("      mma  a_ready(start,ok)", m[:2], "sb(wait_empty_start, empty_ok, committed):", [tuple(m[2+3*s:5+3*s]) for s in range(5)])
