"""SURVEY.md 8(f) rows 1 and 2 on the device, pinned to the reference.

* Row 1 -- QREG dumps.  ``tests/golden/qreg_*.qreg.gz`` were written by the
  reference's own dump path (run_shor with ShorConfig.dump_state_path,
  shor.py:113-114 -> qstate.dump_state, qstate.py:121-130;
  tests/golden/make_golden.py qreg).  The repo's three writers -- the
  drop-in driver, ``distributed.dump_spectrum_sharded`` over device shards
  (1 rank, and 2 gloo ranks on one GPU) and the C-ABI handle's
  ``shb_dump_state`` -- must produce the identical 16-byte header and a
  payload within 1e-12 max|V| of the reference's (whose own sequential sum
  is good to ~M 2^-53).
* Row 2 -- concurrent attempts.  ``distributed.run_shor_concurrent`` with
  the device ``shor.single_attempt``, two gloo ranks sharing the GPU (one
  attempt each per round; the kernels never wait on each other), must
  reproduce the reference's sequential traces (shor.py:155-166) from
  tests/golden/kats.json: same x, q, k, m, outcome and factors.
"""

import gzip
import json
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1801_01434_b200 import distributed as D  # noqa: E402
from paper_1801_01434_b200 import shor  # noqa: E402
from paper_1801_01434_b200.register import NativeRegister  # noqa: E402

HEADER = 16
PAYLOAD_TOL = 1e-12


def _ref_qreg(golden_dir, tag) -> bytes:
    return gzip.decompress((golden_dir / f"qreg_{tag}.qreg.gz").read_bytes())


def _compare(got: bytes, want: bytes):
    assert len(got) == len(want)
    assert got[:HEADER] == want[:HEADER]
    g = np.frombuffer(got[HEADER:], dtype="<c16")
    w = np.frombuffer(want[HEADER:], dtype="<c16")
    err = float(np.abs(g - w).max()) / float(np.abs(w).max())
    assert err <= PAYLOAD_TOL, err
    return err


def _free_port() -> int:
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


@pytest.mark.parametrize("tag", ["n15", "n221"])
def test_run_shor_dump_matches_reference_qreg(golden_dir, tag, tmp_path):
    meta = json.loads((golden_dir / "qreg_dumps.json").read_text())[tag]
    path = tmp_path / "got.qreg"
    res = shor.run_shor(shor.ShorConfig(n=meta["n"], kernel="dense", dump_state_path=str(path), **meta["cfg"]))
    assert res.factors == meta["factors"]
    last = [t for t in res.attempts if t.k is not None][-1]
    want = meta["last_attempt"]
    assert (last.x, last.q, last.k, last.m) == (want["x"], want["q"], want["k"], want["m"])
    _compare(path.read_bytes(), _ref_qreg(golden_dir, tag))


def _n221_attempt2_sampler():
    """Seed 0's stream after attempt 1 (three draws: x, u_k, u_m)."""
    return D.sampler_at(0, 3)


def test_sharded_dump_one_rank_matches_reference_qreg(golden_dir, tmp_path):
    s = _n221_attempt2_sampler()
    x = shor._draw_base(221, s)
    rec = D.sharded_attempt(221, x, 1 << 16, s, keep_spectrum=True)
    assert (x, rec.k, rec.m) == (5, 168, 57344)
    out, _ = rec.spectrum
    D.dump_spectrum_sharded(out, 1 << 16, tmp_path / "one.qreg")
    _compare((tmp_path / "one.qreg").read_bytes(), _ref_qreg(golden_dir, "n221"))


def _dump_worker(rank, world, port, path, ret):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = _n221_attempt2_sampler()
        x = shor._draw_base(221, s)
        rec = D.sharded_attempt(221, x, 1 << 16, s, rank=rank, world=world, keep_spectrum=True)
        out, _ = rec.spectrum
        D.dump_spectrum_sharded(out, 1 << 16, path, rank=rank, world=world)
        ret[rank] = (x, rec.k, rec.m)
    finally:
        dist.destroy_process_group()


def test_sharded_dump_two_ranks_matches_reference_qreg(golden_dir, tmp_path):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    path = str(tmp_path / "two.qreg")
    port = _free_port()
    procs = [ctx.Process(target=_dump_worker, args=(r, 2, port, path, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    assert ret[0] == ret[1] == (5, 168, 57344)
    _compare((tmp_path / "two.qreg").read_bytes(), _ref_qreg(golden_dir, "n221"))


@pytest.mark.parametrize("shards", [1, 2])
def test_handle_dump_state_matches_reference_qreg(golden_dir, tmp_path, shards):
    s = _n221_attempt2_sampler()
    x = shor._draw_base(221, s)
    with NativeRegister([0] * shards) as reg:
        reg.entangle(x, 221, 16)
        k, M, _ = reg.measure(s.uniform())
        assert (k, M) == (168, 4096)
        reg.transform()
        assert reg.sample(s.uniform()) == 57344
        reg.dump_state(tmp_path / "c.qreg")
    _compare((tmp_path / "c.qreg").read_bytes(), _ref_qreg(golden_dir, "n221"))


# ------------------------------------------------------------ concurrent attempts

def _multi_attempt_runs(golden_dir):
    kats = json.loads((golden_dir / "kats.json").read_text())
    runs = [r for r in kats["traces"] if r["cfg"].get("kernel") == "dense" and len(r["attempts"]) >= 2]
    runs += [r for r in kats["traces"] if r["n"] == 15 and r["cfg"].get("base_override") == 7]
    return runs


def _concurrent_worker(rank, world, port, runs, ret):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for run in runs:
            cfg = shor.ShorConfig(n=run["n"], max_width=32, **run["cfg"])
            res = D.run_shor_concurrent(cfg, rank=rank, world=world)
            out.append({"factors": res.factors, "succeeded": res.succeeded,
                        "attempts": [(a.x, a.q, a.k, a.m, a.outcome.kind) for a in res.attempts]})
        ret[rank] = out
    finally:
        dist.destroy_process_group()


def test_concurrent_attempts_on_device_match_reference_traces(golden_dir):
    import torch.multiprocessing as mp
    runs = _multi_attempt_runs(golden_dir)
    assert len(runs) >= 5
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_concurrent_worker, args=(r, 2, port, runs, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    for rank in range(2):
        for run, got in zip(runs, ret[rank]):
            want = [(a["x"], a["q"], a["k"], a["m"], a["outcome"]["kind"]) for a in run["attempts"]]
            assert got["factors"] == run["factors"] and got["succeeded"] == run["succeeded"], run
            assert [tuple(a) for a in got["attempts"]] == want, (run["n"], run["cfg"])


def test_concurrent_attempts_single_rank_is_run_shor(golden_dir):
    """World 1: run_shor_concurrent is the sequential driver (same traces)."""
    for run in _multi_attempt_runs(golden_dir)[:4]:
        cfg = shor.ShorConfig(n=run["n"], max_width=32, **run["cfg"])
        a = D.run_shor_concurrent(cfg)
        b = shor.run_shor(cfg)
        assert a.factors == b.factors
        assert [(t.x, t.k, t.m) for t in a.attempts] == [(t.x, t.k, t.m) for t in b.attempts]
        assert [t.outcome.kind for t in a.attempts] == [t.outcome.kind for t in b.attempts]
