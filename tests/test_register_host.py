"""Register-handle ABI (shb_ctx) without a GPU: the host half of
measure_part2 against the reference's golden sweep, and the error paths."""

import ctypes
import json

import numpy as np
import pytest

from oracle import oracle
from paper_1801_01434_b200 import _native as nat
from paper_1801_01434_b200 import qstate, register


@pytest.fixture(scope="module")
def lib():
    return nat.load()


def test_host_measure_class_matches_reference_sweep(golden_dir):
    """k, M and the amplitude bits of the reference's measure_part2 (605 draws,
    SURVEY 8(c) golden sweep), from exact class counts only."""
    rows = json.loads((golden_dir / "kats.json").read_text())["measure_sweep"]
    counts_of = {}
    for row in rows:
        key = (row["x"], row["n"], row["q"])
        if key not in counts_of:
            res = oracle.modexp_residues(row["x"], row["n"], row["q"]).astype(np.int64)
            counts_of[key] = np.bincount(res, minlength=row["n"]).astype(np.uint64)
        k, M, amp = register.host_measure_class(counts_of[key], row["q"], row["u"])
        assert (k, M) == (row["k"], row["M"]), row
        assert np.float64(amp).view(np.uint64) == np.uint64(int(row["amp_re_bits"], 16)), row
        assert row["amp_im_bits"] == "0000000000000000"


def test_host_measure_class_matches_python_recipe_random():
    rng = np.random.default_rng(5)
    for _ in range(400):
        w = int(rng.integers(1, 33))
        q = 1 << w
        counts = rng.integers(0, 6, int(rng.integers(1, 50))).astype(np.uint64)
        counts[-1] += np.uint64(1)
        if rng.random() < 0.5:
            counts *= np.uint64(int(rng.integers(1, 1 << 24)))
        u = float(rng.random())
        a = complex(1.0 / np.sqrt(q))
        w0 = qstate.uniform_weight(a)
        k = qstate.draw_class(counts, w0, u)
        amp = qstate.collapsed_amplitude(a, w0, int(counts[k]))
        assert register.host_measure_class(counts, q, u) == (k, int(counts[k]), amp.real)


def test_host_measure_class_errors(lib):
    with pytest.raises(ValueError, match="zero"):
        register.host_measure_class(np.zeros(4, np.uint64), 16, 0.5)
    with pytest.raises(ValueError, match="power of two"):
        register.host_measure_class(np.ones(4, np.uint64), 12, 0.5)
    # trailing empty classes do not count (nclasses = max residue + 1, qstate.py:96)
    assert register.host_measure_class(np.array([2, 2, 0, 0], np.uint64), 4, 0.99)[0] == 1


def test_handle_errors_without_device(lib):
    E = nat.SHB_EINVAL
    st = ctypes.c_int()
    assert lib.shb_ctx_state(None, ctypes.byref(st), None, None, None) == E
    assert lib.shb_ctx_modexp(None, 2, 15, 8) == E
    assert lib.shb_measure(None, 0.5, None, None, None) == E
    assert lib.shb_sample(None, 0.5, None) == E
    assert lib.shb_dump_state(None, b"/tmp/x") == E
    lib.shb_free(None)  # no-op
    h = ctypes.c_void_p()
    assert lib.shb_init_devices(None, 1, ctypes.byref(h)) == E
    assert lib.shb_init(1, ctypes.byref(h)) in (nat.SHB_ECUDA, nat.SHB_OK)
    if h.value:
        lib.shb_free(h)
    with pytest.raises(OSError):
        nat.check(nat.SHB_EIO, "dump")
