"""Reference-facing API semantics that need no GPU: argument validation order,
error types and messages, dataclass shapes, Sampler stream, seed derivation.
(qstate.py / qft.py / shor.py of the reference are the spec.)"""

import dataclasses
import math

import numpy as np
import pytest

from paper_1801_01434_b200 import qft, qstate, shor
from paper_1801_01434_b200 import numtheory as nt


def test_sampler_stream_is_numpy_pcg64():
    s = qstate.Sampler(1234)
    g = np.random.Generator(np.random.PCG64(1234))
    assert [s.uniform() for _ in range(50)] == [float(g.random()) for _ in range(50)]
    assert qstate.Sampler(-1).seed == (1 << 64) - 1


def test_init_uniform_and_norm():
    for q, val in [(4, 0.5), (256, 0.0625), (2, 1 / math.sqrt(2))]:
        reg = qstate.init_uniform(q)
        assert np.all(np.asarray(reg.amplitudes) == val)
        assert np.asarray(reg.residues).tolist() == [0] * q
        assert reg.collapsed_k is None and reg.n is None and reg.x is None
    assert qstate.l2_norm(qstate.init_uniform(256)) == 1.0
    for bad in (0, 1, 3, 12):
        with pytest.raises(ValueError, match="power of two"):
            qstate.init_uniform(bad)


def test_entangle_validation_before_device_work():
    reg = qstate.init_uniform(16)
    with pytest.raises(ValueError, match="modulus must be >= 2"):
        qstate.entangle_modexp(reg, 2, 1)
    with pytest.raises(ValueError, match="shares a factor"):
        qstate.entangle_modexp(reg, 6, 15)
    collapsed = dataclasses.replace(reg, collapsed_k=1)
    with pytest.raises(ValueError, match="already collapsed"):
        qstate.entangle_modexp(collapsed, 2, 15)


def test_measure_validation_order():
    # unnormalized first (qstate.py:92), then already-measured (qstate.py:93)
    reg = qstate.CompositeRegister(q=4, amplitudes=np.full(4, 0.7, complex), residues=np.zeros(4, np.int64))
    with pytest.raises(ValueError, match="not normalized"):
        qstate.measure_part2(reg, qstate.Sampler(0))
    reg = qstate.CompositeRegister(q=4, amplitudes=np.full(4, 0.5, complex), residues=np.zeros(4, np.int64),
                                   collapsed_k=0)
    with pytest.raises(ValueError, match="already measured"):
        qstate.measure_part2(reg, qstate.Sampler(0))
    with pytest.raises(ValueError, match="not normalized"):
        qstate.sample_part1(qstate.CompositeRegister(q=4, amplitudes=np.zeros(4, complex),
                                                     residues=np.zeros(4, np.int64)), qstate.Sampler(0))
    assert qstate.l2_norm(qstate.CompositeRegister(q=4, amplitudes=np.zeros(4, complex),
                                                   residues=np.zeros(4, np.int64))) == 0.0


def test_qft_validation():
    assert qft.ENGINES == ("dense", "tiled", "fft", "circuit")
    with pytest.raises(ValueError, match="unknown engine"):
        qft.transform(np.zeros(4, complex), "gpu")
    with pytest.raises(ValueError, match="exceeds the configured maximum width"):
        qft.build_twiddles(1 << 25)
    assert qft.build_twiddles(1 << 30, max_width=30).q == 1 << 30  # lazy: no 16 GiB table
    tw = qft.build_twiddles(4)
    assert np.allclose(tw.roots, [1, 1j, -1, -1j])
    with pytest.raises(ValueError, match="block_size"):
        qft.KernelPlan(block_size=3).resolved(16)
    with pytest.raises(ValueError, match="tiles"):
        qft.KernelPlan(tiles=3).resolved(16)
    with pytest.raises(ValueError, match="workers"):
        qft.KernelPlan(workers=0).resolved(16)
    with pytest.raises(ValueError, match="precision"):
        qft.KernelPlan(precision="fp16").resolved(16)
    assert qft.KernelPlan(block_size=4096).resolved(256).block_size == 256
    assert qft.KernelPlan().num_blocks(1024) == 4
    with pytest.raises(ValueError, match="untiled"):
        qft.dense_dft(np.zeros(16, complex), qft.build_twiddles(16), qft.KernelPlan(tiles=2))
    with pytest.raises(ValueError, match="tiles >= 2"):
        qft.tiled_dft(np.zeros(16, complex), qft.build_twiddles(16), qft.KernelPlan())
    with pytest.raises(ValueError, match="capped"):
        qft.circuit_qft(np.zeros(1 << 13, complex))
    # length is checked before the plan, as in the reference (qft.py:98-101)
    with pytest.raises(ValueError, match="does not match q=16"):
        qft.dense_dft(np.zeros(8, complex), qft.build_twiddles(16), qft.KernelPlan(block_size=3))
    with pytest.raises(ValueError, match="does not match q=16"):
        qft.tiled_dft(np.zeros(8, complex), qft.build_twiddles(16), qft.KernelPlan(tiles=3))


def test_shor_driver_host_parts():
    assert shor.PHASES == ("setup", "entangle", "measure2", "qft", "sample", "postprocess")
    # splitmix64 child seeds (shor.py:58-64), known values
    z = shor._derive_seed(0, 3)
    assert 0 <= z < 1 << 64 and z == shor._derive_seed(0, 3) and z != shor._derive_seed(0, 5)
    s = qstate.Sampler(0)
    g = np.random.Generator(np.random.PCG64(0))
    assert shor._draw_base(221, s) == 2 + int(float(g.random()) * 218) == 140
    with pytest.raises(ValueError, match="unknown kernel"):
        shor.single_attempt(shor.ShorConfig(n=15, kernel="nope"), qstate.Sampler(0))
    with pytest.raises(ValueError, match="outside"):
        shor.single_attempt(shor.ShorConfig(n=15, base_override=15), qstate.Sampler(0))
    # gcd shortcut never touches the device
    tr = shor.single_attempt(shor.ShorConfig(n=15, base_override=6), qstate.Sampler(0))
    assert tr.outcome.kind == "classical_shortcut" and tr.outcome.shortcut == 3 and tr.q is None
    # pre-checks and recursion without the quantum path
    r = shor.run_shor(shor.ShorConfig(n=49))
    assert r.succeeded and r.factors == [7, 7] and r.attempts == []
    r = shor.run_shor(shor.ShorConfig(n=16))
    assert r.factors == [2, 2, 2, 2]
    with pytest.raises(nt.NothingToFactor):
        shor.run_shor(shor.ShorConfig(n=13))
    with pytest.raises(ValueError):
        shor.run_shor(shor.ShorConfig(n=2))
    # the register-width guard keeps the reference default (shor.py:34)
    with pytest.raises(ValueError, match="exceeds the configured maximum"):
        shor.single_attempt(shor.ShorConfig(n=32399, base_override=2), qstate.Sampler(0))


def test_profile_phases():
    tr = shor.AttemptTrace(x=2, q=16, k=1, m=0, candidate=None, outcome=nt.FactorOutcome.retry("zero_measurement"),
                           phase_times={"qft": 2.0, "sample": 2.0})
    res = shor.ShorResult(n=15, factors=[], attempts=[tr], total_time=1.0, succeeded=False)
    f = shor.profile_phases(res)
    assert f["qft"] == 0.5 and abs(sum(f.values()) - 1) < 1e-12
    with pytest.raises(ValueError):
        shor.profile_phases(shor.ShorResult(n=15, factors=[], attempts=[], total_time=0, succeeded=False))


def test_dump_load_roundtrip(tmp_path):
    z = np.random.default_rng(0).standard_normal(64) + 1j
    reg = qstate.CompositeRegister(q=64, amplitudes=z, residues=np.zeros(64, np.int64))
    p = tmp_path / "r.qreg"
    qstate.dump_state(reg, p)
    raw = p.read_bytes()
    assert raw[:4] == b"QREG" and len(raw) == 16 + 64 * 16
    assert np.array_equal(qstate.load_state(p), z)
    p.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="magic"):
        qstate.load_state(p)
    p.write_bytes(raw[:16 + 32])  # whole complex values, fewer than q
    with pytest.raises(ValueError, match="truncated"):
        qstate.load_state(p)


def test_gate_ops_validate_before_the_device():
    """The gate primitives (qft.py:164-212) check their arguments in the
    reference's order and with its messages before any device work."""
    z = np.ones(16, dtype=np.complex128) / 4
    with pytest.raises(ValueError, match="control and target must differ"):
        qft.apply_controlled_phase(z, 1, 1, 0.5)
    with pytest.raises(ValueError, match=r"qubit index 4 out of range for w=4"):
        qft.apply_controlled_phase(z, 4, 0, 0.5)
    with pytest.raises(ValueError, match=r"qubit index -1 out of range for w=4"):
        qft.apply_hadamard(z, -1)
    with pytest.raises(ValueError, match="size must be a power of two"):
        qft.apply_hadamard(np.ones(6, dtype=np.complex128), 0)
    with pytest.raises(ValueError, match="size must be a power of two"):
        qft.bit_reverse_permute(np.ones(6))
    with pytest.raises(ValueError, match="circuit engine capped at w <= 12, got w=13"):
        qft.circuit_qft(np.ones(1 << 13, dtype=np.complex128))
    with pytest.raises(ValueError, match="circuit engine is gate-level FP64"):
        qft.transform(z, "circuit", plan=qft.KernelPlan(precision="fp32"))
