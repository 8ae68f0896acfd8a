"""CPU tests: the C-ABI library loads and exports every declared symbol, and the
host-side exact helpers reproduce numpy's float64 reductions bit for bit."""

import math
import re

import numpy as np
import pytest

from paper_1801_01434_b200 import _native as nat
from paper_1801_01434_b200 import build as build_mod

HEADER = build_mod.PKG.parent / "include" / "shorb200.h"


@pytest.fixture(scope="module")
def lib():
    build_mod.build()
    return nat.load()


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(shb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_binding_binds():
    assert declared_symbols() == sorted(nat.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.shb_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(nat.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


W_VALUES = [1 / 256, 1 / 512, (1 / math.sqrt(512)) ** 2, (1 / math.sqrt(1 << 15)) ** 2,
            (1 / math.sqrt(1 << 31)) ** 2, 0.1, 1e-9, 3e-7, 1 / 3, 2.0 ** -30, 5e-324 * 7]
N_VALUES = [0, 1, 2, 7, 8, 9, 127, 128, 129, 255, 256, 1000, 4096, 5461, 8193, 65535, 100003, 1 << 18]


@pytest.mark.parametrize("w", W_VALUES)
def test_seqsum_const_matches_cumsum_and_bincount(lib, w):
    for n in N_VALUES:
        got = nat.host_seqsum_const(w, n)
        if n == 0:
            assert got == 0.0
            continue
        assert got == np.cumsum(np.full(n, w))[-1]
        assert got == np.bincount(np.zeros(n, dtype=np.int64), weights=np.full(n, w))[0]


@pytest.mark.parametrize("w", W_VALUES)
def test_pairwise_const_matches_numpy_sum(lib, w):
    for n in N_VALUES + [1 << 20, 3_000_017]:
        assert nat.host_pairwise_sum_const(w, n) == np.full(n, w).sum()


def test_random_weights_seqsum(lib):
    rng = np.random.default_rng(3)
    for _ in range(200):
        w = float(rng.random() * 10.0 ** rng.integers(-15, 2))
        n = int(rng.integers(1, 200000))
        assert nat.host_seqsum_const(w, n) == np.cumsum(np.full(n, w))[-1]
        assert nat.host_pairwise_sum_const(w, n) == np.full(n, w).sum()


def test_abi_argument_errors_without_device(lib):
    import ctypes
    E = nat.SHB_EINVAL
    d = ctypes.c_double(0)
    u = ctypes.c_uint64(0)
    assert lib.shb_modexp(None, 0, 16, 2, 1, None) == E                      # modulus < 2
    assert lib.shb_modexp(None, 0, 16, 2, 1 << 33, None) == E                # > 32-bit residues
    assert b"32-bit" in lib.shb_last_error()
    assert lib.shb_class_counts(None, 16, None, 0, None) == E                # ncls == 0
    args = (None, 4, 0, 1, 1000, 0, 1000, 1, 1.0, 0, None, None, None, None)  # q not a power of two
    assert lib.shb_dft(*args) == E and b"power of two" in lib.shb_last_error()
    assert lib.shb_dft(None, 4, 0, 1, 1024, 0, 1024, 3, 1.0, 0, None, None, None, None) == E   # tiles
    assert lib.shb_dft(None, 4, 1020, 2, 1024, 0, 1024, 1, 1.0, 0, None, None, None, None) == E  # leaves [0,q)
    assert lib.shb_dft(None, 4, 0, 1, 1024, 1000, 100, 1, 1.0, 0, None, None, None, None) == E   # rows
    assert lib.shb_dft(None, 4, 0, 1, 1024, 0, 8, 1, 1.0, 7, None, None, None, None) == E        # precision
    assert lib.shb_dft_uniform(1.0, 0.0, 4, 0, 0, 1024, 0, 8, 1, 1.0, 0, None, None, None, None) == E  # stride 0
    assert lib.shb_dense_dft_host(None, 1024, 1, 0, None) == E
    assert lib.shb_partial_row_sums_host(None, None, None, 1024, 0, 8, 0, 8) == E
    assert lib.shb_sum(None, 0, None, None) == E
    assert lib.shb_cumsum_search(None, 0, 0.5, None, None) == E
    assert lib.shb_sample_index(None, 0, 0.5, ctypes.byref(u), ctypes.byref(d), None) == nat.SHB_OK
    assert u.value == 0  # empty input: index = count = 0
    with pytest.raises(ValueError):
        nat.check(E, "x")
    with pytest.raises(MemoryError):
        nat.check(nat.SHB_ENOMEM, "x")
    with pytest.raises(RuntimeError):
        nat.check(nat.SHB_ECUDA, "x")


def test_c_abi_demo_compiles_and_links(lib, tmp_path):
    # plain C against include/shorb200.h and the .so (running it needs a GPU: test_gpu_parity)
    from conftest import build_c_demo
    assert build_c_demo(tmp_path).exists()


def test_dft_engine_choice(lib, monkeypatch):
    """shb_dft_engine names the kernel each DFT entry point launches (no GPU
    call): the int8 tensor-core engine for the FP64 uniform comb (16 int8
    MACs = 32 integer ops per phase term), real-A DMMA for real amplitudes (4
    flops per phase term), complex DMMA otherwise (8), the vector kernel for
    tiles > 1, the BF16 tensor-core form for the FP32 uniform comb; env
    overrides."""
    import ctypes

    def eng(uniform, real, q=1 << 30, prec=nat.FP64, tiles=1):
        f = ctypes.c_int(0)
        name = lib.shb_dft_engine(uniform, real, q, prec, tiles, ctypes.byref(f)).decode()
        return name, f.value

    for var in ("SHB_DFT_ENGINE", "SHB_MMA_REAL", "SHB_FP32_ENGINE"):
        monkeypatch.delenv(var, raising=False)
    assert eng(1, 1) == ("i8::dft_i8_uniform_kernel", 32)
    assert eng(0, 1) == ("dft_mma_kernel<generic, real A>", 4)
    assert eng(0, 0) == ("dft_mma_kernel<generic, complex A>", 8)
    assert eng(1, 1, tiles=4)[0] == "dft_kernel<uniform>"
    assert eng(1, 1, prec=nat.FP32) == ("dft_tc05_uniform_kernel", 8)
    assert eng(0, 1, prec=nat.FP32)[0] == "dft_kernel<generic>"
    # the choice never depends on the output range, only on q and the data
    assert eng(1, 1, q=1 << 8) == eng(1, 1, q=1 << 32)
    monkeypatch.setenv("SHB_DFT_ENGINE", "i8")
    assert eng(1, 1) == ("i8::dft_i8_uniform_kernel", 32)
    assert eng(0, 1) == ("dft_mma_kernel<generic, real A>", 4)
    monkeypatch.setenv("SHB_DFT_ENGINE", "mma")
    assert eng(1, 1) == ("dft_mma_kernel<uniform, real A>", 4)
    monkeypatch.setenv("SHB_DFT_ENGINE", "vector")
    assert eng(1, 1) == ("dft_kernel<uniform>", 8)
    monkeypatch.setenv("SHB_DFT_ENGINE", "mma")
    monkeypatch.setenv("SHB_MMA_REAL", "0")
    assert eng(1, 1) == ("dft_mma_kernel<uniform, complex A>", 8)
    monkeypatch.setenv("SHB_FP32_ENGINE", "mma")
    assert eng(1, 1, prec=nat.FP32)[0] == "dft_tc32_uniform_kernel"
    monkeypatch.setenv("SHB_FP32_ENGINE", "vector")
    assert eng(1, 1, prec=nat.FP32)[0] == "dft_kernel<uniform>"
