"""Run shor.run_shor on one GPU for a named config and compare its trace with
the SURVEY.md 8(d) expected trace (reference-measured for n <= 3127, predicted
by the closed-form replay for q = 2^30 / 2^32).  Prints one JSON line.

    python scripts/run_config.py 32399 2        # n, seed
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1801_01434_b200 import qft, shor  # noqa: E402

# (x, m, outcome kind/reason) per attempt, final factors
EXPECTED = {
    (15, 0): {"attempts": [(7, 64, "factors")], "factors": [3, 5], "base_override": 7},
    (221, 0): {"attempts": [(140, 0, "retry"), (5, 57344, "factors")], "factors": [13, 17]},
    (3127, 0): {"attempts": [(1991, 578525, "factors")], "factors": [53, 59]},
    (32399, 0): {"attempts": [(20637, 43968454, "retry"), (537, None, "classical_shortcut")], "factors": [179, 181]},
    (32399, 2): {"attempts": [(8477, 874074104, "factors")], "factors": [179, 181]},
    (32399, 3): {"attempts": [(2776, 860266936, "factors")], "factors": [179, 181]},
    (32399, 8): {"attempts": [(10594, 342163047, "factors")], "factors": [179, 181]},
    (46927, 0): {"attempts": [(29890, 175938419, "retry"), (777, 3920174108, "factors")], "factors": [167, 281]},
}


def main():
    n = int(sys.argv[1])
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    exp = EXPECTED.get((n, seed))
    cfg = shor.ShorConfig(n=n, seed=seed, kernel="dense", max_width=32,
                          base_override=(exp or {}).get("base_override"), plan=qft.KernelPlan())
    t0 = time.perf_counter()
    res = shor.run_shor(cfg)
    wall = time.perf_counter() - t0
    got = [(a.x, a.m, a.outcome.kind) for a in res.attempts]
    line = {"n": n, "seed": seed, "factors": res.factors, "succeeded": res.succeeded, "wall_s": wall,
            "attempts": [{"x": a.x, "q": a.q, "k": a.k, "m": a.m, "outcome": a.outcome.kind,
                          "reason": a.outcome.reason,
                          "p": a.candidate.p if a.candidate else None,
                          "phase_s": a.phase_times} for a in res.attempts]}
    if exp:
        line["expected"] = exp
        line["match"] = (res.factors == exp["factors"] and
                         [(x, m, k) for x, m, k in got] == [tuple(e) for e in exp["attempts"]])
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
