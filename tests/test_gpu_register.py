"""GPU parity of the register-handle ABI (shb_ctx, include/shorb200.h).

The handle runs the same kernels as the Python drop-in, so its results must
be bitwise identical to the qstate/qft pipeline (k, M, amplitude, spectrum,
m) and to the reference golden vectors, for one shard and for several shards
on one device (the sharded code path; shards never wait on one another).
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle  # noqa: E402
from paper_1801_01434_b200 import qft, qstate, shor  # noqa: E402
from paper_1801_01434_b200.register import NativeRegister  # noqa: E402


class Forced(qstate.Sampler):
    def __init__(self, values):
        super().__init__(0)
        self._v = list(values)

    def uniform(self):
        return self._v.pop(0)


def _python_attempt(x, n, q, u2, u3, precision="fp64", tiles=1):
    s = Forced([u2, u3])
    reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
    k, rc = qstate.measure_part2(reg, s)
    plan = qft.KernelPlan(tiles=tiles, precision=precision)
    spec = qft.transform(rc.amplitudes, "dense" if tiles == 1 else "tiled", qft.build_twiddles(q, 32), plan)
    m = qstate.sample_part1(qstate.CompositeRegister(q, spec, None), s)
    return k, rc.amplitudes, spec, m


CASES = [(7, 15, 8, 0.3, 0.5), (2, 15, 8, 0.0, 0.99), (140, 221, 16, 0.61, 0.27), (5, 221, 16, 0.9, 0.1),
         (19, 35, 11, 0.45, 0.72), (1991, 3127, 22, 0.2, 0.8)]


@pytest.mark.parametrize("shards", [1, 2, 3])
@pytest.mark.parametrize("x,n,w,u2,u3", CASES)
def test_handle_matches_python_pipeline_bitwise(x, n, w, u2, u3, shards):
    q = 1 << w
    k, amps, spec, m = _python_attempt(x, n, q, u2, u3)
    with NativeRegister([0] * shards) as reg:
        reg.entangle(x, n, w)
        assert reg.state == {"stage": "entangled", "q": q, "n": n, "shards": shards}
        k2, M2, amp2 = reg.measure(u2)
        assert (k2, M2) == (k, amps.m)
        assert np.float64(amp2).view(np.uint64) == np.float64(amps.amp.real).view(np.uint64)
        sup = reg.support()
        assert np.array_equal(sup, np.arange(amps.m, dtype=np.uint64) * np.uint64(amps.stride) + np.uint64(amps.a0))
        reg.transform()
        got = reg.spectrum()
        want = spec.data.cpu().numpy().view(np.complex128)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))  # bitwise, signed zeros included
        assert abs(reg.l2_norm() - 1.0) < 1e-9
        assert reg.sample(u3) == m


def test_handle_vs_reference_golden(golden_dir):
    """Residues, collapse and spectrum rows against the reference's own vectors."""
    kats = json.loads((golden_dir / "kats.json").read_text())
    for q, x, n, want in kats["entangle"]:
        w = q.bit_length() - 1
        with NativeRegister() as reg:
            reg.entangle(x, n, w)
            assert reg.residues().tolist() == want
    for tag in ["n15", "n15x2", "n221a1", "n221a2", "n3127"]:
        d = np.load(golden_dir / f"spectrum_{tag}.npz")
        info = json.loads(str(d["info"]))
        q = int(d["q"])
        rows = d["rows"].astype(np.int64)
        with NativeRegister([0, 0]) as reg:
            reg.entangle(int(d["x"]), int(d["n"]), q.bit_length() - 1)
            counts = reg.class_counts()
            k, M = info["k"], info["M"]
            assert int(counts[k]) == M
            M2, amp = reg.collapse(k)
            assert M2 == M
            assert np.float64(amp).view(np.uint64) == np.uint64(int(info["amp_re_bits"], 16))
            reg.transform()
            V = d["V"]
            pmax = float(np.max(np.abs(V) ** 2))
            got = np.concatenate([reg.spectrum(int(c), int(c) + 1) for c in rows[:256]])
            assert np.max(np.abs(got - V[:256])) <= 1e-12
            assert np.max(np.abs(np.abs(got) ** 2 - np.abs(V[:256]) ** 2)) / pmax <= 1e-9


def test_handle_q2_24_attempt_matches_survey_trace():
    # n=3127 seed 0 attempt 1: x=1991, k=825, c0=29, r=116, M=144631, m=578525
    s = qstate.Sampler(0)
    assert shor._draw_base(3127, s) == 1991
    u2, u3 = s.uniform(), s.uniform()
    with NativeRegister([0, 0, 0, 0]) as reg:
        reg.entangle(1991, 3127, 24)
        k, M, _ = reg.measure(u2)
        assert (k, M) == (825, 144631)
        sup = reg.support()
        assert sup[0] == 29 and np.all(np.diff(sup) == 116)
        reg.transform()
        assert reg.sample(u3) == 578525


def test_handle_tiled_and_fp32():
    x, n, w, u2, u3 = 140, 221, 16, 0.61, 0.27
    q = 1 << w
    _, _, spec_t, m_t = _python_attempt(x, n, q, u2, u3, tiles=4)
    _, _, spec_f, m_f = _python_attempt(x, n, q, u2, u3, precision="fp32")
    with NativeRegister([0, 0]) as reg:
        reg.entangle(x, n, w)
        reg.measure(u2)
        reg.transform(tiles=4)
        assert np.array_equal(reg.spectrum().view(np.uint64), spec_t.data.cpu().numpy().view(np.uint64))
        assert reg.sample(u3) == m_t
    with NativeRegister() as reg:
        reg.entangle(x, n, w)
        reg.measure(u2)
        reg.transform("fp32")
        assert np.array_equal(reg.spectrum().view(np.uint64), spec_f.data.cpu().numpy().view(np.uint64))
        assert abs(reg.l2_norm() - 1.0) < 1e-4
        assert reg.sample(u3) == m_f


def test_handle_dump_state_matches_qstate(tmp_path):
    x, n, w, u2, u3 = 2, 15, 8, 0.3, 0.5
    q = 1 << w
    k, amps, spec, m = _python_attempt(x, n, q, u2, u3)
    qstate.dump_state(qstate.CompositeRegister(q, spec, None), tmp_path / "py.qreg")
    with NativeRegister([0, 0, 0]) as reg:
        reg.entangle(x, n, w)
        reg.measure(u2)
        reg.transform()
        reg.dump_state(tmp_path / "c.qreg")
        with pytest.raises(OSError):
            reg.dump_state(tmp_path / "missing" / "dir" / "c.qreg")
    assert (tmp_path / "c.qreg").read_bytes() == (tmp_path / "py.qreg").read_bytes()
    assert np.array_equal(qstate.load_state(tmp_path / "c.qreg"), spec.data.cpu().numpy().view(np.complex128))


def test_handle_stage_errors_match_reference_semantics():
    with NativeRegister() as reg:
        with pytest.raises(ValueError, match="entangled"):
            reg.class_counts()
        with pytest.raises(ValueError, match="shares a factor"):
            reg.entangle(3, 15, 8)  # entangle_modexp's gcd check (qstate.py:73-74)
        with pytest.raises(ValueError, match="modulus"):
            reg.entangle(3, 1, 8)
        reg.entangle(7, 15, 8)
        with pytest.raises(ValueError, match="transformed"):
            reg.sample(0.5)
        with pytest.raises(ValueError, match="probability 0"):
            reg.collapse(2)  # 2 is not a power of 7 mod 15
        reg.measure(0.3)
        with pytest.raises(ValueError, match="already measured"):
            reg.measure(0.3)  # qstate.py:93-94
        with pytest.raises(ValueError, match="tiles"):
            reg.transform(tiles=3)
        reg.transform()
        with pytest.raises(ValueError, match="already transformed"):
            reg.transform()
        # a new entangle discards the old register
        reg.entangle(2, 15, 4)
        assert reg.state["stage"] == "entangled"
        assert reg.residues().tolist() == [1, 2, 4, 8] * 4
    with pytest.raises(ValueError):
        NativeRegister([0, 99])


def test_c_attempt_demo_matches_python(tmp_path):
    import subprocess
    from conftest import build_c_demo
    exe = build_c_demo(tmp_path, "c_attempt_demo")
    for x, n, w, u2, u3 in CASES[:4]:
        k, amps, spec, m = _python_attempt(x, n, 1 << w, u2, u3)
        for shards in (1, 3):
            r = subprocess.run([str(exe), str(n), str(x), str(w), repr(u2), repr(u3), str(shards)],
                               capture_output=True, text=True, timeout=120)
            assert r.returncode == 0, r.stderr
            got = json.loads(r.stdout)
            assert (got["k"], got["M"], got["m"]) == (k, amps.m, m)
            assert got["amp_bits"] == f"{int(np.float64(amps.amp.real).view(np.uint64)):016x}"
            row = spec.data.cpu().numpy().view(np.complex128)[m]
            assert got["row_m"] == [row.real, row.imag]


def test_handle_oracle_pipeline_large_shard_count():
    """8 shards at q = 2^20 (shards smaller than a cycle of x^a) vs the C oracle."""
    x, n, w = 7, 1019 * 3, 20
    q = 1 << w
    res = oracle.modexp_residues(x, n, q)
    with NativeRegister([0] * 8) as reg:
        reg.entangle(x, n, w)
        assert np.array_equal(reg.residues(), res.astype(np.int64))
        counts = reg.class_counts()
        assert np.array_equal(counts, np.bincount(res.astype(np.int64), minlength=n).astype(np.uint64))
        k, M, amp = reg.measure(0.77)
        amps = np.zeros(q, complex)
        amps[res == k] = amp
        reg.transform()
        rows = np.arange(0, q, 4099)
        ref = oracle.dft_rows(np.flatnonzero(res == k), np.full(M, amp, complex), q, rows)
        got = np.concatenate([reg.spectrum(int(c), int(c) + 1) for c in rows])
        assert np.max(np.abs(got - ref)) <= 1e-12
