"""Gate-level QFT on the device (csrc/gates.cu) against the reference.

tests/golden/gates.npz holds the reference's own apply_hadamard,
apply_controlled_phase, bit_reverse_permute and circuit_qft outputs
(qft.py:164-231, tests/golden/make_golden.py gates).  The device gates
reproduce numpy's arithmetic, so the comparison is bitwise, signed zeros
included.  The circuit engine then cross-checks the direct-DFT kernels:
two independent constructions of the same unitary.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402
from paper_1801_01434_b200 import qft, qstate  # noqa: E402


@pytest.fixture(scope="module")
def gates(golden_dir):
    d = np.load(golden_dir / "gates.npz")
    return {k: d[k] for k in d.files}


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.complex128).view(np.uint64)


def test_hadamard_bitwise(gates):
    z = gates["state64"]
    for b in range(6):
        got = qft.apply_hadamard(z, b)
        assert isinstance(got, np.ndarray)
        assert np.array_equal(_bits(got), _bits(gates[f"hadamard_{b}"])), b
    assert np.array_equal(_bits(z), _bits(gates["state64"]))  # the input is not mutated


def test_controlled_phase_bitwise(gates):
    z = gates["state64"]
    for c, t, ang in [(0, 1, 0.7), (5, 2, -1.3), (3, 4, 2.0 * np.pi / 8), (1, 5, 1e-3)]:
        got = qft.apply_controlled_phase(z, c, t, ang)
        assert np.array_equal(_bits(got), _bits(gates[f"cphase_{c}_{t}"])), (c, t)


def test_bit_reverse_permute_bitwise(gates):
    assert np.array_equal(_bits(qft.bit_reverse_permute(gates["state64"])), _bits(gates["bitrev64"]))
    ints = np.arange(16, dtype=np.int64) * 3
    got = qft.bit_reverse_permute(ints)
    assert got.dtype == np.int64
    rev = np.array([int(f"{i:04b}"[::-1], 2) for i in range(16)])
    want = np.empty_like(ints)
    want[rev] = ints
    assert np.array_equal(got, want)


@pytest.mark.parametrize("w", [1, 4, 8, 12])
def test_circuit_qft_bitwise_vs_reference(gates, w):
    got = qft.circuit_qft(gates[f"circuit_in_{w}"])
    assert np.array_equal(_bits(got), _bits(gates[f"circuit_out_{w}"])), w


@pytest.mark.parametrize("w", [4, 8, 12])
def test_circuit_engine_cross_checks_dft_kernels(gates, w):
    """Gate-level QFT vs the direct DFT (dense engine) and the oracle rows."""
    s = gates[f"circuit_in_{w}"]
    q = 1 << w
    circ = qft.transform(s, "circuit")
    dense = qft.transform(s, "dense")
    ref = oracle.dense_dft(s)
    assert np.abs(circ - dense).max() <= 1e-12
    assert np.abs(dense - ref).max() <= 1e-12
    assert circ.shape == (q,)


def test_circuit_engine_on_a_collapsed_register():
    """The collapsed Shor register (device-resident) through both engines."""
    reg = qstate.entangle_modexp(qstate.init_uniform(1 << 12), 7, 15)
    s = qstate.Sampler(3)
    k, rc = qstate.measure_part2(reg, s)
    circ = qft.transform(rc.amplitudes, "circuit")
    dense = qft.transform(rc.amplitudes, "dense")
    assert isinstance(circ, dev.DeviceSpectrum)
    assert np.abs(np.asarray(circ) - np.asarray(dense)).max() <= 1e-12
    assert abs(qstate.l2_norm(qstate.CompositeRegister(1 << 12, circ, None)) - 1.0) < 1e-12


def test_gate_argument_errors():
    z = np.ones(16, dtype=np.complex128) / 4
    with pytest.raises(ValueError, match="control and target must differ"):
        qft.apply_controlled_phase(z, 2, 2, 0.1)
    with pytest.raises(ValueError, match="out of range for w=4"):
        qft.apply_controlled_phase(z, 0, 4, 0.1)
    with pytest.raises(ValueError, match="out of range for w=4"):
        qft.apply_hadamard(z, 4)
    with pytest.raises(ValueError, match="size must be a power of two"):
        qft.apply_hadamard(np.ones(12), 0)
    with pytest.raises(ValueError, match="circuit engine capped"):
        qft.circuit_qft(np.ones(1 << 13) / np.sqrt(1 << 13))


def test_engine_precision_plan():
    """fft honours KernelPlan.precision (same kernel as dense); circuit rejects fp32."""
    rng = np.random.default_rng(5)
    z = rng.standard_normal(1 << 10) + 1j * rng.standard_normal(1 << 10)
    z /= np.linalg.norm(z)
    plan32 = qft.KernelPlan(precision="fp32")
    f32 = qft.transform(z, "fft", plan=plan32)
    d32 = qft.transform(z, "dense", plan=plan32)
    assert np.array_equal(f32, d32)
    assert not np.array_equal(f32, qft.transform(z, "fft"))
    with pytest.raises(ValueError, match="circuit engine is gate-level FP64"):
        qft.transform(z, "circuit", plan=plan32)
