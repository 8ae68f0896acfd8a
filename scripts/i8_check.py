"""FP64 int8-tensor-core engine (dft_i8.cu) vs the DMMA engine: spectrum
agreement (max|dV|/max|V|, max|dp|/max p), a shard (offset, ragged output
range) and time, uniform comb at q = 2^8/2^16/2^24 (+2^30 with `big`)."""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1801_01434_b200 import device as dev  # noqa: E402

cases = [(1 << 8, 1, 4, 64), (1 << 16, 11, 12, 5461), (1 << 16, 3, 7, 9000)]
# super-block / K-chunk edges of the engine (4096 amplitudes per chunk, 16384 per super-block)
cases += [(1 << 20, 5, 3, M) for M in (1, 31, 4095, 4096, 4097, 16383, 16384, 16385, 40000, 2 * 16384 + 97)]
cases.append((1 << 24, 29, 116, 144631))
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cases += [(1 << 30, 10943, 16020, 67025), (1 << 30, 4828, 5340, 201075)]


def run(eng, amp, M, c0, r, q, cb, cc):
    os.environ["SHB_DFT_ENGINE"] = eng
    fn = lambda: dev.dft_uniform(amp, M, c0, r, q, cb, cc, precision="fp64")  # noqa: E731
    if q >= 1 << 20:
        o = fn()
        del o
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out, p, bs = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, p, bs, e0.elapsed_time(e1)


for q, c0, r, M in cases:
    amp = complex(1 / math.sqrt(M))
    o64, p64, b64, ms64 = run("mma", amp, M, c0, r, q, 0, q)
    o8, p8, b8, ms8 = run("i8", amp, M, c0, r, q, 0, q)
    vmax = float(o64.abs().max())
    rec = {"q": f"2^{q.bit_length() - 1}", "M": M, "ms_mma": round(ms64, 3), "ms_i8": round(ms8, 3),
           "Gterms_s_mma": round(q * M / ms64 / 1e6, 1), "Gterms_s_i8": round(q * M / ms8 / 1e6, 1),
           "max_dV_over_max_V": float((o8 - o64).abs().max()) / vmax,
           "max_dp_over_max_p": float((p8 - p64).abs().max()) / float(p64.max()),
           "norm_mma": dev.dsum(b64), "norm_i8": dev.dsum(b8)}
    if q <= 1 << 20:
        cb, cc = 1000 % q, min(7777, q - 1000 % q)
        os_, _, _, _ = run("i8", amp, M, c0, r, q, cb, cc)
        rec["shard_bitwise"] = bool(torch.equal(os_, o8[2 * cb: 2 * (cb + cc)]))
    print(json.dumps(rec), flush=True)
    del o64, p64, b64, o8, p8, b8
    torch.cuda.empty_cache()
