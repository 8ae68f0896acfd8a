"""Top stalled SASS instructions and per-opcode stall/instruction shares of one
kernel in an ncu report (--import-source capture).  Run in the build container.

    python scripts/ncu_sass_top.py <report.ncu-rep> [top_n]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
num = lambda v: float(v.replace(",", "") or 0)  # noqa: E731
tot = sum(num(r[iS]) for r in data)
print(f"kernel: {rows[0][1]}  stall samples: {tot:.0f}")
for r in sorted(data, key=lambda r: -num(r[iS]))[:top_n]:
    print(f"{num(r[iS]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[1][:80]:80s} exec={r[iE]}")
samp, ex = collections.Counter(), collections.Counter()
for r in data:
    toks = r[1].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    samp[op] += num(r[iS])
    ex[op] += num(r[iE])
print("stall share by opcode:", [(k, round(v / tot * 100, 1)) for k, v in samp.most_common(16)])
print("warp instructions by opcode (1e6):", [(k, round(v / 1e6)) for k, v in ex.most_common(20)])
