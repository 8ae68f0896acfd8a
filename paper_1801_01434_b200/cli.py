"""Command line: `factor` and `bench` (the reference declares
`shorsim.cli:main` in pyproject.toml:23-24 but does not ship it).

    python -m paper_1801_01434_b200.cli factor --n 221 --seed 0 --kernel dense
    python -m paper_1801_01434_b200.cli bench --suite table3-small --engines dense,fft --format csv

Exit codes: 0 success, 1 factoring failed within budget, 2 invalid input.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys
from dataclasses import asdict, dataclass

CSV_COLUMNS = ("n", "cofactors", "engine", "block_size", "tiles", "workers", "seed", "wall_time_s",
               "qft_fraction", "succeeded")
SUITES = {
    "table3-small": (77, 143, 231, 255),
    "table3-full": (77, 143, 323, 551, 589, 231, 255, 399, 423, 539),
}


@dataclass
class BenchRecord:
    n: int
    cofactors: str
    engine: str
    block_size: int
    tiles: int
    workers: int
    seed: int
    wall_time_s: float
    qft_fraction: float
    succeeded: bool


def emit_report(records: list[BenchRecord], fmt: str) -> str:
    """csv (exact SPEC columns), json (round-trips) or markdown (+ speed-up footer)."""
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_COLUMNS)
        for r in records:
            d = asdict(r)
            d["succeeded"] = "true" if r.succeeded else "false"
            d["wall_time_s"] = f"{r.wall_time_s:.6f}"
            d["qft_fraction"] = f"{r.qft_fraction:.6f}"
            w.writerow([d[c] for c in CSV_COLUMNS])
        return buf.getvalue()
    if fmt == "json":
        return json.dumps([asdict(r) for r in records], indent=1)
    if fmt == "markdown":
        engines = list(dict.fromkeys(r.engine for r in records))
        targets = list(dict.fromkeys(r.n for r in records))
        cell = {(r.n, r.engine): r for r in records}
        lines = ["| n | cofactors | " + " | ".join(f"T_{e} (s)" for e in engines) + " |",
                 "|---|---|" + "---|" * len(engines)]
        for n in targets:
            cof = next((cell[(n, e)].cofactors for e in engines if (n, e) in cell), "")
            vals = []
            for e in engines:
                r = cell.get((n, e))
                vals.append("—" if r is None or not r.succeeded else f"{r.wall_time_s:.3f}")
            lines.append(f"| {n} | {cof} | " + " | ".join(vals) + " |")
        if len(engines) >= 2:
            ref = "fft" if "fft" in engines else engines[0]
            common = [n for n in targets if all((n, e) in cell and cell[(n, e)].succeeded for e in engines)]
            if common:
                sref = sum(cell[(n, ref)].wall_time_s for n in common)
                sp = {e: sum(cell[(n, e)].wall_time_s for n in common) / sref for e in engines}
                lines.append("| Speed-up | | " + " | ".join(f"{sp[e]:.2f}" for e in engines) + " |")
        return "\n".join(lines) + "\n"
    raise ValueError(f"unknown format {fmt!r}")


def parse_records(text: str) -> list[BenchRecord]:
    return [BenchRecord(**d) for d in json.loads(text)]


def _config(a, n):
    from . import qft, shor
    return shor.ShorConfig(n=n, base_override=getattr(a, "base", None), seed=a.seed, kernel=a.kernel,
                           plan=qft.KernelPlan(block_size=a.block_size, tiles=a.tiles, workers=a.workers,
                                               precision=a.precision),
                           max_attempts=a.max_attempts, time_budget=a.time_budget, max_width=a.max_width,
                           dump_state_path=getattr(a, "dump_state", None))


def cmd_factor(a) -> int:
    from . import shor
    res = shor.run_shor(_config(a, a.n))
    prof = shor.profile_phases(res) if res.attempts else {}
    print(json.dumps({"n": a.n, "factors": res.factors, "succeeded": res.succeeded,
                      "attempts": [{"x": t.x, "q": t.q, "k": t.k, "m": t.m, "outcome": t.outcome.kind,
                                    "reason": t.outcome.reason} for t in res.attempts],
                      "total_time_s": res.total_time, "qft_fraction": prof.get("qft", 0.0)}))
    return 0 if res.succeeded else 1


def run_benchmark_suite(targets, a) -> list[BenchRecord]:
    from . import numtheory as nt
    from . import shor
    out = []
    for n in targets:
        for eng in a.engines:
            a.kernel = eng
            cfg = _config(a, n)
            try:
                res = shor.run_shor(cfg)
                frac = shor.profile_phases(res).get("qft", 0.0) if res.attempts else 0.0
                rec = BenchRecord(n=n, cofactors="x".join(map(str, res.factors)), engine=eng,
                                  block_size=cfg.plan.block_size, tiles=cfg.plan.tiles,
                                  workers=cfg.plan.workers or 0, seed=cfg.seed, wall_time_s=res.total_time,
                                  qft_fraction=frac, succeeded=res.succeeded)
            except (ValueError, nt.NothingToFactor):
                rec = BenchRecord(n=n, cofactors="", engine=eng, block_size=cfg.plan.block_size,
                                  tiles=cfg.plan.tiles, workers=cfg.plan.workers or 0, seed=cfg.seed,
                                  wall_time_s=0.0, qft_fraction=0.0, succeeded=False)
            out.append(rec)
    return out


def cmd_bench(a) -> int:
    targets = SUITES.get(a.suite) if a.suite != "custom" else tuple(int(t) for t in a.targets.split(",") if t)
    recs = run_benchmark_suite(targets, a)
    text = emit_report(recs, a.format)
    if a.output:
        with open(a.output, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0 if all(r.succeeded for r in recs) else 1


def _common(p):
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--kernel", default="dense", choices=["dense", "tiled", "fft", "circuit"])
    p.add_argument("--block-size", type=int, default=256)
    p.add_argument("--tiles", type=int, default=1)
    p.add_argument("--workers", type=int, default=None)
    p.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    p.add_argument("--max-attempts", type=int, default=32)
    p.add_argument("--time-budget", type=float, default=None)
    p.add_argument("--max-width", type=int, default=32)


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="shorb200")
    sub = p.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("factor")
    f.add_argument("--n", type=int, required=True)
    f.add_argument("--base", type=int, default=None)
    f.add_argument("--dump-state", default=None)
    _common(f)
    b = sub.add_parser("bench")
    b.add_argument("--suite", default="table3-small", choices=["table3-small", "table3-full", "custom"])
    b.add_argument("--targets", default="")
    b.add_argument("--engines", default="dense")
    b.add_argument("--output", default=None)
    b.add_argument("--format", default="csv", choices=["csv", "json", "markdown"])
    _common(b)
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        if a.cmd == "factor":
            return cmd_factor(a)
        a.engines = [e for e in a.engines.split(",") if e]
        return cmd_bench(a)
    except ValueError as e:  # NothingToFactor is a ValueError too
        sys.stderr.write(f"invalid input: {e}\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
