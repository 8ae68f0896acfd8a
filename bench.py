#!/usr/bin/env python
"""QFT phase-terms/s and end-to-end factoring time at q = 2^30 (n = 32399) on B200.

One step = one full Shor attempt on the device (modexp -> class counts ->
collapse -> direct-DFT QFT -> exact Born-rule read), for n = 32399 = 179 x 181,
q = 2^30, Sampler seed 2 (x = 8477, r = 5340, M = 201075 support elements:
SURVEY.md 8(d)'s recommended north-star run, which factors n through the
quantum path in one attempt).  Phase terms per step = q * M (outputs x
collapsed support).  After the timed steps the line also carries warm
shor.run_shor factoring times for every BASELINE config (factoring_table),
the end-to-end C-ABI number with host buffers (e2e) and the CPU port beside
them.

    python bench.py [--gpus N --steps K --warmup W] [--seed 2] [--impl reference]

Under torchrun each rank owns q/N outputs and q/N exponents
(paper_1801_01434_b200.distributed); total work is fixed -> strong scaling.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "qft_phase_terms_per_s"
UNIT = "phase_terms/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--modulus", dest="n", type=int, default=32399)  # not --n: torchrun prefix-matches it
    p.add_argument("--seed", type=int, default=2)
    p.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    p.add_argument("--max-width", type=int, default=32)
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--ref-step-seconds", type=float, default=6.0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-factoring", action="store_true")
    p.add_argument("--no-fp32", action="store_true")
    p.add_argument("--no-dmma", action="store_true", help="skip the DMMA-engine comparison launch")
    return p.parse_args()


# ------------------------------------------------------------------ helpers

def workload(n: int, seed: int, max_width: int):
    """(q, x) of the seeded attempt through the package (the B200 arm)."""
    from paper_1801_01434_b200 import numtheory as nt
    from paper_1801_01434_b200 import qstate, shor
    rw = nt.choose_register_width(n, max_width)
    s = qstate.Sampler(seed)
    x = shor._draw_base(n, s)
    if math.gcd(x, n) != 1:
        raise SystemExit(f"seed {seed} draws x={x} sharing a factor with n={n}: pick another seed")
    return rw.q, x


def bench_config(n: int, seed: int, q: int, x: int, r: int, k: int, c0: int, M: int,
                 precision: str, world: int) -> dict:
    """The workload description, identical from both arms (only inputs-derived keys)."""
    w = q.bit_length() - 1
    return {"workload": f"n={n} q=2^{w} seed={seed} x={x} r={r} k={k} c0={c0} M={M}: "
                        f"one full attempt (modexp, collapse, QFT of q*M phase terms, Born read) per step",
            "n": n, "q": q, "seed": seed, "x": x, "r": r, "k": k, "c0": c0, "M": M,
            "precision": precision, "parallelism": f"c/a-sharded x{world}",
            "l2": f"no flush needed: each step writes {24 * q / 2**30:.3g} GiB (spectrum + |V|^2) "
                  f"{'>>' if 24 * q > 4 * 126e6 else 'vs'} the 126 MB L2"}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7
                          for i in range(4) if r[3 + i].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if len(r) >= 7 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------ CPU legs

def cpu_terms_rate(q: int, c0: int, r: int, M: int, amp: complex, seconds: float, threads: int):
    """Oracle port of the reference dense engine (support-only rows, bit-identical
    to _kernels.partial_row_sums) on a bounded sample of rows.  Test/baseline only."""
    import numpy as np
    from oracle import oracle
    supp = c0 + r * np.arange(M, dtype=np.uint64)
    amps = np.full(M, amp, dtype=np.complex128)
    rng = np.random.default_rng(1)
    rows_done = 0
    batch = max(threads, 8)
    t0 = time.perf_counter()
    while True:
        rows = rng.integers(0, q, batch, dtype=np.uint64)
        oracle.dft_rows(supp, amps, q, rows, True, threads)
        rows_done += batch
        el = time.perf_counter() - t0
        if el >= seconds:
            break
        batch = max(threads, int(batch * min(4.0, max(1.2, seconds / max(el, 1e-3) / 2))))
    el = time.perf_counter() - t0
    return rows_done * M / el, rows_done, el


def run_reference(args):
    """--impl reference: the reference's dense QFT arithmetic on the host cores.

    Imports nothing from paper_1801_01434_b200: the attempt's register comes
    from oracle.attempt_register (numpy restatement of qstate.py:95-104 and
    shor.py:67-70) and the rows from oracle/shor_oracle.c, the support-only
    restatement of _kernels.partial_row_sums (bit-identical to dense_dft)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle
    reg = oracle.attempt_register(args.n, args.seed)
    q, x, r, k, c0, M, amp = (reg[key] for key in ("q", "x", "r", "k", "c0", "M", "amp"))
    thr = cpu_threads()
    for _ in range(args.warmup):
        cpu_terms_rate(q, c0, r, M, amp, min(1.0, args.ref_step_seconds), thr)
    rows, secs = 0, 0.0
    for _ in range(args.steps):
        _, nr, el = cpu_terms_rate(q, c0, r, M, amp, args.ref_step_seconds, thr)
        rows += nr
        secs += el
    value = rows * M / secs
    sample = (f"{rows} random output rows of the n={args.n} q=2^{q.bit_length() - 1} attempt "
              f"(M={M} support terms each) over {args.steps} steps of ~{args.ref_step_seconds:.0f}s")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.precision == "fp64" else "f32",
        "data": "synthetic (the register is generated by the algorithm from n and the seed)",
        "config": bench_config(args.n, args.seed, q, x, r, k, c0, M, args.precision, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "port", "sample": sample,
                         "cpu": cpu_model(),
                         "note": "oracle/shor_oracle.c: support-only restatement of "
                                 "_kernels.partial_row_sums, bit-identical output; the reference's "
                                 f"own dense loop also walks the q-M zeros ({q / M:.0f}x more terms)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def run_b200(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink in production; SHB_DIST_BACKEND=gloo lets a test put
        # several ranks on one GPU (independent kernels, host-staged collectives)
        backend = os.environ.get("SHB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1801_01434_b200 import _native as nat
    from paper_1801_01434_b200 import build as buildmod
    from paper_1801_01434_b200 import distributed as D
    from paper_1801_01434_b200 import numtheory as nt
    from paper_1801_01434_b200 import qstate, shor

    if not nat.LIB_PATH.exists():
        buildmod.build()
    lib = nat.load()
    q, x = workload(args.n, args.seed, args.max_width)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def one_step(time_dft=False, keep=False, precision=None):
        s = qstate.Sampler(args.seed)
        xx = shor._draw_base(args.n, s)
        rec = D.sharded_attempt(args.n, xx, q, s, rank=rank, world=world, group=group,
                                precision=precision or args.precision, time_dft=time_dft, keep_spectrum=keep)
        est = nt.extract_period(rec.m, q, args.n, xx)
        out = nt.derive_factors(args.n, xx, est.p) if isinstance(est, nt.PeriodCandidate) else est
        return rec, out

    for _ in range(args.warmup):
        rec, outcome = one_step()
    barrier()
    uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    clocks = ClockSampler(uuid)
    clocks.start()
    launches0 = lib.shb_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    dft_ms, recs = [], []
    for i in range(args.steps):
        rec, outcome = one_step(time_dft=True, keep=(i == args.steps - 1 and not args.no_fp32))
        recs.append(rec)
        dft_ms.append(rec.dft_ms)
    e1.record()
    barrier()
    clk = clocks.stop()
    launches = lib.shb_kernel_launches() - launches0
    el_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([el_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        el_ms = float(t.item())
    rec = recs[-1]
    M = rec.M
    terms_step = q * M
    value = terms_step * args.steps / (el_ms / 1000.0)

    # roofline of the dominant kernel (the DFT), per GPU.  Peak: the nominal
    # FP64 rate (SMs x 64 DFMA/clk x 2 flops) at the SM clock measured during
    # the timed region -- a hard upper bound (MEASURED_PEAKS.json has no FP64
    # figure); the DFMA-chain probe is reported beside it.
    ptf, pdm = ctypes_double(), ctypes_double()
    nat.check(lib.shb_fp64_peak(2.0, ptf, None), "fp64 peak")
    nat.check(lib.shb_fp64_dmma_peak(2.0, pdm, None), "fp64 dmma peak")
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    clk_mhz = clk.get("sm_mhz") or 1965.0
    peak_tf = sms * 64 * 2 * clk_mhz * 1e6 / 1e12
    dft_s = statistics.mean(dft_ms) / 1000.0
    # the kernel the attempt launched (uniform comb) and its flops per phase term:
    # 4 in the real-A DMMA form (amp*cos, amp*sin), 8 for a complex multiply-add
    fpt = ctypes_int()
    kname = lib.shb_dft_engine(1, 1, q, nat.FP64 if args.precision == "fp64" else nat.FP32, 1, fpt)
    kname = kname.decode() if kname else "dft"
    achieved_tf = fpt.value * rec.phase_terms / dft_s / 1e12
    # DRAM bytes per DFT launch from the committed ncu --set full capture, only
    # when that capture was taken at this very configuration
    prof = ROOT / "profiles" / "dft_traffic.json"
    traffic, traffic_note = None, "no ncu --set full capture at this config"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            if tj.get("config") == f"n={args.n} q=2^{q.bit_length() - 1} M={rec.M}" and tj.get("kernel") == f"shb::{kname}":
                traffic = tj["dram_bytes_per_launch"] / world
                traffic_note = f"ncu capture {tj.get('source', '')}".strip()
            else:
                traffic_note = (f"ncu capture of {tj.get('kernel')} at {tj.get('config')} measured "
                                f"{tj['dram_bytes_per_launch'] / 1e6:.1f} MB "
                                f"vs {tj['algorithmic_bytes_per_launch'] / 1e6:.1f} MB algorithmic (24 B/output)")
        except Exception:
            pass
    if "i8" in kname:
        roof = _i8_roofline(rec, q, M, world, dft_s, sms, clk_mhz, kname, fpt.value, traffic, traffic_note,
                            peak_tf, ptf.value, pdm.value)
    else:
        roof = {"bound": "fp64", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_tf, "traffic": traffic, "traffic_note": traffic_note,
                "traffic_unit": "bytes/launch", "algorithmic_bytes_per_launch": 24 * (q // world),
                "peak_source": f"nominal FP64 (one datapath for DFMA and DMMA): {sms} SMs x 64 FMA/clk x 2 flops x {clk_mhz:.0f} MHz "
                               "(median SM clock in the timed region); MEASURED_PEAKS.json has no FP64 figure",
                "peak_probe": ptf.value,
                "peak_probe_note": "shb_fp64_peak: independent DFMA chains with constant operands on this GPU",
                "peak_probe_dmma": pdm.value,
                "peak_probe_dmma_note": "shb_fp64_dmma_peak: independent DMMA m8n8k4 chains on this GPU (the "
                                        "tensor path of the same FP64 datapath)",
                "kernel": f"shb::{kname}", "dft_ms_per_launch": dft_s * 1000.0,
                "flops_per_phase_term": fpt.value, "flops_per_launch": fpt.value * rec.phase_terms}

    # the same attempt's QFT on the FP64-pipe DMMA engine, for comparison (one launch)
    dmma = None
    if not args.no_dmma and args.precision == "fp64" and "i8" in kname:
        os.environ["SHB_DFT_ENGINE"] = "mma"
        try:
            rec_m, _ = one_step(time_dft=True)
        finally:
            del os.environ["SHB_DFT_ENGINE"]
        t_m = torch.tensor([rec_m.dft_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(t_m, op=torch.distributed.ReduceOp.MAX)
        dmma = {"kernel": "shb::dft_mma_kernel<uniform, real A>", "dft_ms": float(t_m.item()),
                "phase_terms_per_s": q * M / (float(t_m.item()) / 1000.0),
                "fp64_tflops": 4 * q * M / (float(t_m.item()) / 1000.0) / 1e12 / world,
                "frac_of_fp64_peak": 4 * q * M / (float(t_m.item()) / 1000.0) / 1e12 / world / peak_tf,
                "m_equal": rec_m.m == rec.m,
                "note": "FP64 DMMA (mma.sync m8n8k4 f64) engine on the same attempt, one launch; "
                        "SHB_DFT_ENGINE=mma selects it"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
        "data": "synthetic (the register is generated by the algorithm from n and the seed)",
        "config": bench_config(args.n, args.seed, q, x, rec.r, rec.k, rec.c0, M, args.precision, world),
        "result": {"m": rec.m, "outcome": outcome.kind,
                   "factors": list(outcome.factors) if outcome.factors else None},
        "gpu_launches": int(launches),
        "clocks": clk,
        "roofline": roof,
        "phase_ms_last_step": {k: v * 1000 for k, v in rec.phase_times.items()},
    }
    if dmma:
        line["fp64_dmma_engine"] = dmma

    # e2e: the reference-facing C-ABI drop-in with HOST buffers (H2D + DFT + D2H
    # inside the timed region).  N=1: shb_dense_dft_host (qft.dense_dft); N>1:
    # every rank runs the _kernels.partial_row_sums seam on its row shard.
    if not args.no_e2e:
        line["e2e"] = e2e_host(args, q, rec, lib, torch, nat, rank, world)
    # the sharded Born-rule read's pieces, timed on an eighth of this attempt's
    # probabilities (one rank's shard at N = 8): what an N-GPU step adds
    if world == 1 and hasattr(rec, "spectrum"):
        line["multi_gpu_model"] = _cdf_split_model(rec.spectrum[1], q, rec.dft_ms, el_ms / args.steps, torch)
    # FP32 fast path on the same attempt: Horner in FP32 with exact FP64
    # re-seeds every 256 terms; accuracy vs the FP64 spectrum just measured
    if not args.no_fp32 and args.precision == "fp64":
        _, p64 = rec.spectrum
        rec32, out32 = one_step(time_dft=True, keep=True, precision="fp32")
        _, p32 = rec32.spectrum
        err = torch.stack([(p32 - p64).abs().max(), p64.max()])
        del rec32.spectrum, rec.spectrum
        t32 = torch.tensor([rec32.dft_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(err, op=torch.distributed.ReduceOp.MAX)
            torch.distributed.all_reduce(t32, op=torch.distributed.ReduceOp.MAX)
        f32 = ctypes_int()
        k32 = lib.shb_dft_engine(1, 1, q, nat.FP32, 1, f32)
        k32 = k32.decode() if k32 else "dft"
        tf32 = f32.value * q * M / (float(t32.item()) / 1000.0) / 1e12
        line["fp32_fast_path"] = {
            "dft_ms": float(t32.item()), "phase_terms_per_s": q * M / (float(t32.item()) / 1000.0),
            "max_abs_dp_over_max_p": float(err[0] / err[1]), "tolerance": 1e-4,
            "m": rec32.m, "m_equal_fp64": rec32.m == rec.m, "kernel": f"shb::{k32}",
            "achieved_tflops": tf32, "flops_per_phase_term": f32.value,
            "note": "DFT kernel only; not the headline (FP64).  The tensor-core forms issue 4 bf16 MACs per "
                    "phase term (Re/Im x hi/lo split of the phase matrix): tcgen05.mma with TMEM "
                    "accumulators (default) or mma.sync m16n8k16 (SHB_FP32_ENGINE=mma)"}
        peaks = _measured_peaks()
        if peaks.get("bf16_tflops") and ("tc05" in k32 or "tc32" in k32):
            line["fp32_fast_path"]["frac_of_bf16_peak"] = tf32 / peaks["bf16_tflops"]
            line["fp32_fast_path"]["bf16_peak_source"] = "MEASURED_PEAKS.json bf16_tflops (cuBLAS, tcgen05)"

    if not args.no_factoring:
        barrier()
        if world == 1:
            line["factoring"] = factoring_table(args)
        else:
            line["factoring"] = {"api": "distributed.sharded_attempt", "time_s": el_ms / args.steps / 1000,
                                 "factors": list(outcome.factors) if outcome.factors else None}

    if not args.no_cpu_baseline and world == 1 and rank == 0:
        from oracle import oracle  # the CPU baseline leg: the reference's arithmetic, timed
        reg = oracle.attempt_register(args.n, args.seed)
        thr = cpu_threads()
        rate, rows, el = cpu_terms_rate(q, reg["c0"], reg["r"], reg["M"], reg["amp"], args.cpu_seconds, thr)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": thr, "kind": "port",
                                "sample": f"{rows} random rows x M={reg['M']} terms of the same attempt in {el:.1f}s",
                                "cpu": cpu_model()}
        if "factoring" in line:
            _cpu_column(line["factoring"], args, thr)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _cdf_split_model(prob, q: int, dft_ms: float, step_ms: float, torch, world: int = 8) -> dict:
    """Time the split sequential cumsum on one 1/world shard of the spectrum's
    |V|^2 (device events): records (parallel on every rank) and the exact walk
    (the only rank-to-rank serial hop), next to the unsplit per-shard scan the
    round-1 chain serialised.  Model of an N-rank step from these (not a
    multi-GPU measurement)."""
    from paper_1801_01434_b200 import device as dev
    shard = prob[: q // world]

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, out

    hint = 0.0
    rec_ms, plan = timed(lambda: dev.cumsum_plan(shard, hint))
    walk_ms, _ = timed(lambda: dev.cumsum_walk(shard, plan, 0.0))
    old_ms, _ = timed(lambda: dev.cumsum_total_from(shard, 0.0))
    per_rank_dft = dft_ms / world
    other = step_ms - dft_ms  # entangle + collapse + sample on one GPU
    predicted = per_rank_dft + other / world + rec_ms + (world - 1) * walk_ms
    return {"world": world, "shard_outputs": q // world, "records_ms": rec_ms, "walk_ms_per_hop": walk_ms,
            "unsplit_scan_ms_per_hop": old_ms, "dft_ms_per_rank": per_rank_dft,
            "predicted_step_ms": predicted, "predicted_scaling_efficiency": step_ms / world / predicted,
            "note": "model from single-GPU timings: per-rank DFT = 1/world of this attempt's DFT (outputs split evenly, "
                    "same per-output work), the other stages split evenly, plus the parallel records and "
                    "(world - 1) serial carry hops; NCCL collectives (a few scalars and the class counts) not "
                    "included. No multi-GPU hardware was available to measure it."}


# BASELINE.json configs through the public driver, with SURVEY.md 8(d)'s traces:
# (label, n, seed, base_override, expected m per attempt, expected factors)
FACTORING_CONFIGS = [
    ("configs[0] n=15 x=7 q=2^8", 15, 0, 7, [64], [3, 5]),
    ("configs[1] n=221 q=2^16", 221, 0, None, [0, 57344], [13, 17]),
    ("configs[2] n=3127 q=2^24", 3127, 0, None, [578525], [53, 59]),
    ("configs[3] n=32399 q=2^30 seed 8 (light)", 32399, 8, None, [342163047], [179, 181]),
    ("configs[3] n=32399 q=2^30 seed 2 (north-star run)", 32399, 2, None, [874074104], [179, 181]),
    ("configs[3] n=32399 q=2^30 seed 0 (default seed: odd r, then gcd)", 32399, 0, None, [43968454, None], [179, 181]),
    ("configs[4] n=46927 q=2^32 seed 0", 46927, 0, None, [175938419, 3920174108], [167, 281]),
]


def factoring_table(args) -> dict:
    """Warm shor.run_shor (the reference's public driver, shor.py:136-201) for every
    BASELINE config on this GPU: wall time, per-phase split, QFT phase terms, and
    the trace checked against SURVEY.md 8(d)."""
    from paper_1801_01434_b200 import numtheory as nt
    from paper_1801_01434_b200 import qft, shor
    rows = []
    for label, n, seed, base, want_m, want_f in FACTORING_CONFIGS:
        if n == args.n and (n * n - 1).bit_length() > args.max_width:
            continue
        cfg = shor.ShorConfig(n=n, seed=seed, base_override=base, kernel="dense", max_width=32,
                              plan=qft.KernelPlan(precision=args.precision))
        t0 = time.perf_counter()
        res = shor.run_shor(cfg)
        wall = time.perf_counter() - t0
        phases = {ph: sum(a.phase_times.get(ph, 0.0) for a in res.attempts) for ph in shor.PHASES}
        terms = 0
        for a in res.attempts:
            if a.k is None:
                continue
            r = nt.classical_period(a.x, n)
            c0 = next(j for j in range(r) if pow(a.x, j, n) == a.k)
            terms += a.q * ((a.q - 1 - c0) // r + 1)
        ms = [a.m for a in res.attempts]
        rows.append({"config": label, "n": n, "seed": seed, "time_s": wall, "factors": res.factors,
                     "attempts": [{"x": a.x, "k": a.k, "m": a.m, "outcome": a.outcome.kind} for a in res.attempts],
                     "phase_s": phases, "qft_fraction": phases["qft"] / max(sum(phases.values()), 1e-12),
                     "phase_terms": terms, "qft_phase_terms_per_s": terms / phases["qft"] if phases["qft"] else None,
                     "trace_matches_survey": ms == want_m and res.factors == want_f})
    return {"api": "shor.run_shor(ShorConfig(n, seed, kernel='dense', max_width=32))", "runs": rows,
            "north_star_time_s": next((r["time_s"] for r in rows if r["n"] == 32399 and r["seed"] == 2), None),
            "note": "one warm run per config after the timed steps; SURVEY.md 8(d) traces "
                    "(reference-measured for n <= 3127, closed-form replay of the reference for 2^30 / 2^32)"}


def _cpu_column(fact: dict, args, thr: int, seconds: float = 2.0) -> None:
    """CPU-port QFT estimate beside each factoring row: the oracle rate on a
    bounded sample of the run's first quantum attempt x its phase terms."""
    from oracle import oracle
    for row in fact.get("runs", []):
        try:
            reg = oracle.attempt_register(row["n"], row["seed"]) if row["n"] != 15 else None
        except ValueError:
            reg = None
        if row["n"] == 15:
            q, c0, r, M, amp = 256, 1, 4, 64, complex(0.125)
        elif reg is None:
            continue
        else:
            q, c0, r, M, amp = reg["q"], reg["c0"], reg["r"], reg["M"], reg["amp"]
        rate, nrows, el = cpu_terms_rate(q, c0, r, M, amp, seconds, thr)
        row["cpu_port"] = {"phase_terms_per_s": rate, "cores": thr, "sample_rows": nrows,
                           "est_qft_s": row["phase_terms"] / rate if row["phase_terms"] else 0.0,
                           "gpu_speedup": (row["qft_phase_terms_per_s"] / rate
                                           if row["qft_phase_terms_per_s"] and rate else None)}


def _i8_roofline(rec, q, M, world, dft_s, sms, clk_mhz, kname, ops_per_term, traffic, traffic_note,
                 fp64_peak_tf, probe_dfma, probe_dmma) -> dict:
    """Roofline of the int8 tensor-core FP64 engine (csrc/dft_i8.cu), per GPU.

    Tensor: 16 int8 MACs (32 integer ops) per phase term (Re/Im x 8 digits of
    G*2^55); peak = 2x the measured cuBLAS bf16 rate (kind::i8 dense issues at
    twice kind::f16 on B200: 4.5 POPS vs 2.25 PFLOPS nominal).  The MMA is
    M128 (row-blocks) x N24 (outputs) x K32 with the weights in TMEM; its
    measured issue floor at N = 24 (15.4 cycles, scripts/i8t_probe.cu) is
    reported beside the tensor peak, and the accumulator drain (FP64
    combine + Horner, profiles/r02_i8_timeline_q2_30_kch8.txt) overlaps it on the
    second accumulator set."""
    peaks = _measured_peaks()
    bf16 = peaks.get("bf16_tflops")
    peak_tops = 2 * bf16 if bf16 else 4500.0
    terms = rec.phase_terms
    achieved = ops_per_term * terms / dft_s / 1e12
    # MMA floor of this shape: 15.4 cycles per M128 N24 K32 (524288 int8 ops... 128*24*32 MACs)
    n24_tops = 2 * 128 * 24 * 32 / 15.4 * sms * clk_mhz * 1e6 / 1e12
    # K-chunks per super-block as csrc/dft_i8.cu picks them: 8 when that needs
    # fewer super-blocks than 6 (4096 amplitudes per K-chunk)
    kch = 8 if -(-M // 32768) < -(-M // 24576) else 6
    nsb = -(-M // (4096 * kch))
    return {"bound": "tensor", "achieved": achieved, "peak": peak_tops, "unit": "TOPS",
            "frac": achieved / peak_tops, "traffic": traffic, "traffic_note": traffic_note,
            "traffic_unit": "bytes/launch", "algorithmic_bytes_per_launch": 24 * (q // world),
            "peak_source": ("2 x MEASURED_PEAKS.json bf16_tflops (cuBLAS bf16, tcgen05); kind::i8 dense = 2x kind::f16"
                            if bf16 else "nominal B200 int8 dense 4.5 POPS (MEASURED_PEAKS.json absent)"),
            "kernel": f"shb::{kname}", "dft_ms_per_launch": dft_s * 1000.0,
            "int8_ops_per_phase_term": ops_per_term, "ops_per_launch": ops_per_term * terms,
            "mma_shape": "M128 (row-blocks, weights in TMEM) x N24 (outputs, digits of G in smem) x K32",
            "n24_issue_floor": {"tops": n24_tops, "frac": achieved / n24_tops,
                                "source": "15.4 cycles per M128 N24 K32 kind::i8 MMA with A in TMEM, measured "
                                          "back to back on this B200 (scripts/i8t_probe.cu)"},
            "superblocks_per_tile": nsb, "kchunks_per_superblock": kch,
            "uniform_comb_only": "the weight operand is the all-ones amplitude matrix of the collapsed register: "
                                 "every row-block's T is the same number, so this throughput is specific to "
                                 "uniform combs (general amplitudes take the DMMA engine)",
            "fp64_equivalent": {"tflops": 4 * terms / dft_s / 1e12, "fp64_peak_tflops": fp64_peak_tf,
                                "note": "4 flops per phase term (the real-A FP64 form) for comparison with the "
                                        "FP64-pipe engines; not a roofline of this kernel (its products are "
                                        "exact int8 digit products on the tensor cores)",
                                "peak_probe_dfma": probe_dfma, "peak_probe_dmma": probe_dmma}}


def _measured_peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        return {}


def ctypes_int():
    import ctypes
    return ctypes.c_int(0)


def ctypes_double():
    import ctypes
    return ctypes.c_double(0.0)


def e2e_host(args, q, rec, lib, torch, nat, rank=0, world=1, calls=3):
    """The reference-facing C ABI with HOST buffers: H2D of the complex128[q]
    register, the DFT and D2H of the spectrum inside each timed call."""
    import ctypes
    import numpy as np
    from paper_1801_01434_b200 import qstate
    c0, r, M = rec.c0, rec.r, rec.M
    a_unif = complex(1.0 / math.sqrt(q))
    amp = qstate.collapsed_amplitude(a_unif, qstate.uniform_weight(a_unif), M)
    c_lo, c_hi = q * rank // world, q * (rank + 1) // world
    if world > 1:
        shared = _shared_state(q, c0, r, amp, rank, world, torch)
        if shared is not None:
            return _e2e_sharded(args, q, M, shared, c_lo, c_hi, lib, torch, nat, rank, world)
    need = 16 * q + 16 * (c_hi - c_lo)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # pragma: no cover
        avail = None
    ok = avail is None or world * need < 0.8 * avail
    if world > 1:
        flag = torch.tensor([1 if ok else 0], device="cuda")
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        ok = bool(flag.item())
    if not ok:
        return {"value": None, "unit": UNIT, "h2d_bytes_per_step": 16 * q, "d2h_bytes_per_step": 16 * q,
                "reason": f"host RAM: {world} ranks x {need / 2**30:.0f} GiB pinned exceeds 80% of available"}
    st = torch.empty(2 * q, dtype=torch.float64, pin_memory=True)
    out = torch.empty(2 * (c_hi - c_lo), dtype=torch.float64, pin_memory=True)
    stn = st.numpy().view(np.complex128)
    stn[:] = 0
    stn[c0::r] = amp
    prec = 0 if args.precision == "fp64" else 1
    def call():
        if world == 1:
            nat.check(lib.shb_dense_dft_host(ctypes.c_void_p(st.data_ptr()), q, 1, prec,
                                             ctypes.c_void_p(out.data_ptr())), "dense_dft_host")
        else:
            nat.check(lib.shb_partial_row_sums_host(ctypes.c_void_p(out.data_ptr()),
                                                    ctypes.c_void_p(st.data_ptr()), None, q, c_lo, c_hi, 0, q),
                      "partial_row_sums_host")

    api = ("shb_dense_dft_host (C ABI of qft.dense_dft, pinned host buffers)" if world == 1 else
           "shb_partial_row_sums_host (C ABI of _kernels.partial_row_sums), row shard per rank")
    secs = _time_calls(call, calls, world, torch)
    o = out.numpy().view(np.complex128)
    v0 = o[0] if rank == 0 else complex(0)
    del st, out
    return _e2e_line(q, M, secs, world, api, v0)


def _time_calls(call, calls: int, world: int, torch) -> list:
    """One untimed call (maps the library's stream-ordered pool, a one-off per
    process), then `calls` timed calls; each is the max over ranks."""
    call()
    torch.cuda.synchronize()
    secs = []
    for _ in range(calls):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        call()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            el = float(t.item())
        secs.append(el)
    return secs


def _e2e_line(q, M, secs, world, api, v0) -> dict:
    med = statistics.median(secs)
    return {"value": q * M / med, "unit": UNIT, "h2d_bytes_per_step": 16 * q * world,
            "d2h_bytes_per_step": 16 * q, "steps": len(secs), "warmup": 1,
            "seconds": {"median": med, "min": min(secs), "max": max(secs), "all": secs},
            "value_min_max": [q * M / max(secs), q * M / min(secs)], "api": api,
            "check_V0": [float(v0.real), float(v0.imag)]}


def _shared_state(q, c0, r, amp, rank, world, torch):
    """One host copy of the complex128[q] state for all local ranks: a /dev/shm
    file mapped by every rank and page-locked with cudaHostRegister, so 8 ranks
    do not need 8 x 16 GiB of private pinned memory.  None if unavailable."""
    import numpy as np
    path = Path("/dev/shm") / f"shb_e2e_{os.environ.get('MASTER_PORT', '0')}_{q}"
    try:
        free = os.statvfs("/dev/shm")
        if free.f_bavail * free.f_frsize < 16 * q * 1.1:
            return None
    except OSError:
        return None
    ok = torch.tensor([1], device="cuda")
    if int(os.environ.get("LOCAL_RANK", "0")) == 0:
        try:
            mm = np.memmap(path, dtype=np.complex128, mode="w+", shape=(q,))
            mm[c0::r] = amp
            mm.flush()
            del mm
        except OSError:
            ok[0] = 0
    torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
    if not int(ok.item()):
        return None
    mm = np.memmap(path, dtype=np.complex128, mode="r+", shape=(q,))
    ptr = mm.ctypes.data
    registered = False
    try:
        rc = torch.cuda.cudart().cudaHostRegister(ptr, 16 * q, 0)
        registered = int(rc) == 0 if not hasattr(rc, "value") else int(rc.value) == 0
    except Exception:
        registered = False
    if not registered:
        # a refused registration (e.g. a /dev/shm mapping in a container) leaves a
        # sticky runtime error that the next library launch check would report
        try:
            torch.cuda.cudart().cudaGetLastError()
        except Exception:
            pass
    return {"mm": mm, "ptr": ptr, "path": path, "registered": registered}


def _e2e_sharded(args, q, M, shared, c_lo, c_hi, lib, torch, nat, rank, world):
    import ctypes
    import numpy as np
    out = torch.empty(2 * (c_hi - c_lo), dtype=torch.float64, pin_memory=True)

    def call():
        nat.check(lib.shb_partial_row_sums_host(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(shared["ptr"]),
                                                None, q, c_lo, c_hi, 0, q), "partial_row_sums_host")

    try:
        call()
        ok = 1
    except RuntimeError:
        ok = 0  # e.g. several ranks sharing one GPU cannot all use the page-locked mapping
    flag = torch.tensor([ok], device="cuda")
    torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
    if not int(flag.item()) and shared["registered"]:
        try:
            torch.cuda.cudart().cudaHostUnregister(shared["ptr"])
        except Exception:
            pass
        shared["registered"] = False
    secs = _time_calls(call, 3, world, torch)
    v0 = out.numpy().view(np.complex128)[0] if rank == 0 else complex(0)
    if shared["registered"]:
        try:
            torch.cuda.cudart().cudaHostUnregister(shared["ptr"])
        except Exception:
            pass
    del shared["mm"]
    torch.distributed.barrier()
    if int(os.environ.get("LOCAL_RANK", "0")) == 0:
        try:
            shared["path"].unlink()
        except OSError:
            pass
    return _e2e_line(q, M, secs, world,
                     "shb_partial_row_sums_host (C ABI of _kernels.partial_row_sums), row shard per rank; "
                     "one shared /dev/shm host state" + (" page-locked (cudaHostRegister)" if shared["registered"]
                                                          else " (pageable)"), v0)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
