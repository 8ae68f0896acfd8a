"""Summaries of ncu output for profiles/ (run in the build container).

    python scripts/ncu_summary.py rep  <report.ncu-rep> [header lines...]
    python scripts/ncu_summary.py list <launches.csv>   [header lines...]

rep:  key pipe/DRAM/occupancy metrics and the top stall reasons per kernel.
list: per-kernel launch count, total time and share of a launch list taken
      with --metrics gpu__time_duration.sum.
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["launch__registers_per_thread", "gpu__time_duration.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"== {name}")
        for k in KEYS:
            if k in hdr:
                j = hdr.index(k)
                print(f"  {k:<76} {r[j]:>14} {units[j]}")
        stalls = []
        for j, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[j]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        print("  top stalls (warps per issue-active cycle):")
        for v, n in sorted(stalls, reverse=True)[:6]:
            print(f"      {v:6.3f} {n}")
        print()


def launch_list(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] == "ns" else v / 1e3 if r[ui] == "us" else v * 1e3 if r[ui] == "s" else v
        name = r[ki].split("(")[0][:58]
        tot[name] += v
        cnt[name] += 1
    allms = sum(tot.values())
    print(f"{'kernel':<60}{'launches':>9}{'total_ms':>13}{'share_all':>11}")
    for name, v in tot.most_common():
        print(f"{name:<60}{cnt[name]:>9}{v:>13.3f}{100 * v / allms:>10.3f}%")


if __name__ == "__main__":
    for h in sys.argv[3:]:
        print("# " + h)
    if sys.argv[3:]:
        print()
    (rep if sys.argv[1] == "rep" else launch_list)(sys.argv[2])
