"""GPU parity: every sm_100a stage against the CPU oracle / reference golden vectors.

Tolerances (BASELINE.json north_star):
* modexp residues, class counts, support, k, M, amplitude bits, m, r, factors: bit-exact
* FP64 spectrum: max elementwise |dV| <= 1e-12 and max|dp| / max p <= 1e-9
* FP32 spectrum: max|dp| / max p <= 1e-4
* exact-cumsum emulation: bit-identical to numpy's np.cumsum / searchsorted
"""

import json
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle  # noqa: E402
from paper_1801_01434_b200 import _native as nat  # noqa: E402
from paper_1801_01434_b200 import device as dev  # noqa: E402
from paper_1801_01434_b200 import numtheory as nt  # noqa: E402
from paper_1801_01434_b200 import qft, qstate, shor  # noqa: E402


class Forced(qstate.Sampler):
    def __init__(self, values):
        super().__init__(0)
        self._v = list(values)

    def uniform(self):
        return self._v.pop(0)


@pytest.fixture(scope="module")
def kats(golden_dir):
    return json.loads((golden_dir / "kats.json").read_text())


def _spec(golden_dir, tag):
    d = np.load(golden_dir / f"spectrum_{tag}.npz")
    return {k: d[k] for k in d.files}


def _amp(info):
    return complex(np.uint64(int(info["amp_re_bits"], 16)).view(np.float64),
                   np.uint64(int(info["amp_im_bits"], 16)).view(np.float64))


def _rows(out_dev, rows):
    v = out_dev.cpu().numpy().view(np.complex128)
    return v[np.asarray(rows, dtype=np.int64)]


# ------------------------------------------------------------------ modexp

@pytest.mark.parametrize("x,n,q", [(7, 15, 256), (2, 15, 16), (1, 15, 8), (140, 221, 1 << 16),
                                   (1991, 3127, 1 << 20), (20637, 32399, 1 << 22),
                                   (29890, 46927, 1 << 21), (3, 1000003, 1 << 18),
                                   (123456789, 4294967291, 1 << 16)])
def test_modexp_bitexact(x, n, q):
    got = dev.modexp(x, n, q).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.modexp_residues(x, n, q))


def test_modexp_shards_match_full():
    full = oracle.modexp_residues(8477, 32399, 1 << 20)
    for lo, cnt in [(0, 1000), (12345, 77777), ((1 << 20) - 5000, 5000)]:
        got = dev.modexp(8477, 32399, cnt, a_begin=lo).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, full[lo:lo + cnt])


def test_entangle_kats(kats):
    for q, x, n, res in kats["entangle"]:
        reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
        assert np.asarray(reg.residues).tolist() == res


# ------------------------------------------------------------------ collapse

@pytest.mark.parametrize("x,n,q", [(7, 15, 256), (140, 221, 1 << 16), (1991, 3127, 1 << 22),
                                   (3, 1000003, 1 << 17)])
def test_class_counts_and_compaction(x, n, q):
    res_d = dev.modexp(x, n, q)
    res = oracle.modexp_residues(x, n, q)
    counts = dev.class_counts(res_d, n).cpu().numpy()
    assert np.array_equal(counts.astype(np.uint64), oracle.class_counts(res, n))
    for k in {int(res[0]), int(res[q // 3]), int(res[-1])}:
        sup = dev.compact_eq(res_d, k).cpu().numpy()
        assert np.array_equal(sup, np.flatnonzero(res == k))
        a0, stride, length = dev.support_progression(dev.compact_eq(res_d, k))
        assert (a0, length) == (int(sup[0]), len(sup))
        assert stride == nt.classical_period(x, n) if len(sup) > 1 else True
    assert dev.compact_eq(res_d, n + 5).numel() == 0


@pytest.mark.parametrize("lo,hi", [(0, 1), (0, 16383), (0, 16384), (0, 16385), (1, 1 << 20),
                                   (3, (1 << 22) - 5), (0, 148 * 16384 * 2 + 77)])
def test_class_counts_ragged_and_unaligned(lo, hi):
    """The shared-memory histogram's vector path (16 residues per thread per
    step, 16-byte loads) and its scalar tail: sizes around one CTA step
    (1024 x 16), several grid strides, and buffers that start off the 16-byte
    alignment (a shard view res[lo:]) -- all exact against the oracle."""
    x, n, q = 1991, 3127, 1 << 22
    full = dev.modexp(x, n, q)
    hi = min(hi, q)
    res = oracle.modexp_residues(x, n, q)[lo:hi]
    counts = dev.class_counts(full[lo:hi], n).cpu().numpy()
    assert np.array_equal(counts.astype(np.uint64), oracle.class_counts(res, n))
    with pytest.raises(ValueError):
        dev.class_counts(full[lo:hi], int(res.max()))  # a residue >= ncls is an error, not a silent drop


def test_measure_sweep_vs_reference(kats):
    rows = kats["measure_sweep"]
    for row in rows:
        q, x, n, u = row["q"], row["x"], row["n"], row["u"]
        reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
        k, rc = qstate.measure_part2(reg, Forced([u]))
        a = rc.amplitudes
        assert k == row["k"]
        assert a.m == row["M"] and a.a0 == row["c0"]
        if a.m > 1:
            assert a.stride == row["r"]
        assert np.float64(a.amp.real).view(np.uint64) == np.uint64(int(row["amp_re_bits"], 16))
        assert np.float64(a.amp.imag).view(np.uint64) == np.uint64(int(row["amp_im_bits"], 16))


def test_spec_collapse_examples():
    # SPEC.md:163-165
    reg = qstate.entangle_modexp(qstate.init_uniform(256), 2, 15)
    k, rc = qstate.measure_part2(reg, Forced([0.0]))
    assert k == 1
    host = np.asarray(rc.amplitudes)
    assert np.flatnonzero(host).tolist() == list(range(0, 256, 4))
    assert np.all(host[::4] == 0.125)
    k, rc = qstate.measure_part2(reg, Forced([0.3]))
    assert k == 2 and np.flatnonzero(np.asarray(rc.amplitudes)).tolist() == list(range(1, 256, 4))
    with pytest.raises(ValueError):
        qstate.measure_part2(rc, Forced([0.1]))
    assert abs(qstate.l2_norm(rc) - 1.0) < 1e-12


# ------------------------------------------------------------------ DFT

def _check_spectrum(got, ref, tol_abs=1e-12, tol_p=1e-9, pmax=None):
    """max |dV| <= tol_abs and max |dp| / max p <= tol_p, where max p is the
    spectrum's peak probability (pmax; defaults to the peak among `ref`)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert np.max(np.abs(got - ref)) <= tol_abs
    pg, pr = np.abs(got) ** 2, np.abs(ref) ** 2
    assert np.max(np.abs(pg - pr)) / (pmax if pmax is not None else np.max(pr)) <= tol_p


@pytest.mark.parametrize("tag", ["n15", "n15x2", "n221a1", "n221a2", "n3127"])
def test_dft_vs_reference_rows(golden_dir, tag):
    d = _spec(golden_dir, tag)
    info = json.loads(str(d["info"]))
    q, M, c0, r = int(d["q"]), info["M"], info["c0"], info["r"]
    sup = torch.arange(M, dtype=torch.int64, device="cuda") * r + c0
    amps = dev.fill_progression(sup, M, c0, r, M, _amp(info))
    rows = d["rows"].astype(np.int64)
    if q <= (1 << 16):
        out, prob, _ = dev.dft(amps, M, c0, r, q, 0, q)
        _check_spectrum(_rows(out, rows), d["V"])
        # fused probabilities are hypot(re, im)^2 (qstate.py:111); CUDA's hypot
        # is not glibc's, so equal to within a few ulp rather than bitwise
        p_host = prob.cpu().numpy()
        p_np = np.abs(out.cpu().numpy().view(np.complex128)) ** 2
        assert np.max(np.abs(p_host - p_np) / np.spacing(p_np)) <= 8
        # the uniform-comb kernel (selected for collapsed registers) agrees too
        ou, pu, _ = dev.dft_uniform(_amp(info), M, c0, r, q, 0, q)
        _check_spectrum(_rows(ou, rows), d["V"])
    else:
        pmax = float(np.max(np.abs(d["V"]) ** 2))  # the golden rows include the peaks
        for c in rows[:64]:
            out, _, _ = dev.dft(amps, M, c0, r, q, int(c), 1)
            _check_spectrum(out.cpu().numpy().view(np.complex128), d["V"][rows == c], pmax=pmax)
            ou, _, _ = dev.dft_uniform(_amp(info), M, c0, r, q, int(c), 1)
            _check_spectrum(ou.cpu().numpy().view(np.complex128), d["V"][rows == c], pmax=pmax)


def test_dft_full_vs_closed_form_2_24(golden_dir):
    d = _spec(golden_dir, "n3127")
    info = json.loads(str(d["info"]))
    q, M, c0, r = int(d["q"]), info["M"], info["c0"], info["r"]
    sup = torch.arange(M, dtype=torch.int64, device="cuda") * r + c0
    out, prob, bsum = dev.dft_uniform(_amp(info), M, c0, r, q, 0, q)
    p = prob.cpu().numpy()
    rows = np.random.default_rng(5).choice(q, 20000, replace=False)
    cf = oracle.comb_probabilities(q, r, c0, M, rows)
    assert np.max(np.abs(p[rows] - cf)) / p.max() < 1e-9
    # unitarity and the golden rows (computed by the reference kernel)
    assert abs(dev.dsum(bsum) - 1.0) < 1e-9
    _check_spectrum(_rows(out, d["rows"]), d["V"], tol_abs=1e-11)


def test_fp32_fast_path(golden_dir):
    d = _spec(golden_dir, "n221a1")
    info = json.loads(str(d["info"]))
    q, M, c0, r = int(d["q"]), info["M"], info["c0"], info["r"]
    sup = torch.arange(M, dtype=torch.int64, device="cuda") * r + c0
    amps = dev.fill_progression(sup, M, c0, r, M, _amp(info))
    _, p32, _ = dev.dft(amps, M, c0, r, q, 0, q, precision="fp32")
    _, p64, _ = dev.dft(amps, M, c0, r, q, 0, q, precision="fp64")
    _, pu32, _ = dev.dft_uniform(_amp(info), M, c0, r, q, 0, q, precision="fp32")
    p32, p64, pu32 = p32.cpu().numpy(), p64.cpu().numpy(), pu32.cpu().numpy()
    assert np.max(np.abs(p32 - p64)) / p64.max() <= 1e-4
    assert np.max(np.abs(pu32 - p64)) / p64.max() <= 1e-4


@pytest.mark.parametrize("engine", ["vector", "mma", "tcgen05"])
def test_fp32_engines_uniform_vs_oracle(engine, monkeypatch):
    """The FP32 fast path for a uniform comb: the FP32 Horner kernel and the
    BF16 tensor-core form (G = G_hi + G_lo, FP32 accumulation, FP64 segment
    sums).  Against the oracle rows at the stated tolerance, max|dp|/max p
    <= 1e-4 (and |dV| <= 1e-4 max|V|), on ragged lengths (partial last
    block, M < one block), output shards and a q = 2^24 comb."""
    monkeypatch.setenv("SHB_FP32_ENGINE", engine)
    amp = 0.3 - 0.1j
    for q, c0, r, M in [(2, 1, 1, 1), (4, 0, 1, 4), (8, 3, 2, 3), (1 << 10, 5, 3, 1), (1 << 10, 5, 3, 255),
                        (1 << 12, 1, 7, 585), (1 << 16, 11, 12, 5461), (1 << 20, 3, 1, (1 << 20) - 3),
                        (1 << 24, 29, 116, 144631)]:
        rows = np.unique(np.concatenate([np.arange(0, min(q, 4096)), np.arange(q - 130, q),
                                         np.random.default_rng(q).integers(0, q, 2000)])).astype(np.uint64)
        supp = c0 + r * np.arange(M, dtype=np.uint64)
        ref = oracle.dft_rows(supp, np.full(M, amp), q, rows)
        pref = np.abs(ref) ** 2
        for lo, cnt in ([(0, q), (77, min(q - 77, 129)), (q - 130, 130)] if q > 256 else [(0, q), (1, q - 1)]):
            out, prob, bs = dev.dft_uniform(amp, M, c0, r, q, lo, cnt, precision="fp32")
            sel = (rows >= lo) & (rows < lo + cnt)
            o = out.cpu().numpy().view(np.complex128)[(rows[sel] - lo).astype(np.int64)]
            pm = M * abs(amp) / math.sqrt(q)  # |V_0|, the peak of a uniform comb
            assert np.max(np.abs(o - ref[sel])) <= 1e-4 * pm, (q, M, lo)
            pr = prob.cpu().numpy()[(rows[sel] - lo).astype(np.int64)]
            assert np.max(np.abs(pr - pref[sel])) <= 1e-4 * pm ** 2, (q, M, lo)
            assert abs(dev.dsum(bs) - float(prob.sum())) <= 1e-6 * float(prob.sum())
            del out, prob, bs


def test_random_states_dense_tiled(golden_dir):
    d = np.load(golden_dir / "random_states.npz")
    for key in ("16", "256", "1024", "4096", "sparse2048"):
        z = d[f"{key}_state"]
        q = z.size
        tw = qft.build_twiddles(q)
        got = qft.dense_dft(z, tw, qft.KernelPlan())
        assert isinstance(got, np.ndarray)
        assert np.max(np.abs(got - d[f"{key}_dense"])) < 1e-12
        got_t = qft.tiled_dft(z, tw, qft.KernelPlan(tiles=8))
        assert np.max(np.abs(got_t - d[f"{key}_tiled8"])) < 1e-12
        # engine equivalence + unitarity
        for eng in ("fft", "circuit"):
            assert np.max(np.abs(qft.transform(z, eng) - d[f"{key}_dense"])) < 1e-9
        assert abs(np.linalg.norm(got) - 1.0) < 1e-9


def test_spec_qft_examples():
    q = 4
    basis = np.zeros(q, complex)
    basis[0] = 1
    tw = qft.build_twiddles(q)
    assert np.allclose(qft.dense_dft(basis, tw, qft.KernelPlan()), 0.5)
    u = np.full(256, 1 / 16, complex)
    out = qft.dense_dft(u, qft.build_twiddles(256), qft.KernelPlan())
    assert abs(out[0] - 1) < 1e-12 and np.max(np.abs(out[1:])) < 1e-12
    out = qft.tiled_dft(u, qft.build_twiddles(256), qft.KernelPlan(tiles=4))
    assert abs(out[0] - 1) < 1e-12 and np.max(np.abs(out[1:])) < 1e-12
    z = np.zeros(8, complex)
    z[0] = 1
    assert np.allclose(qft.fft_dft(z), 1 / math.sqrt(8))
    with pytest.raises(ValueError):
        qft.tiled_dft(u, qft.build_twiddles(256), qft.KernelPlan(tiles=1))
    with pytest.raises(ValueError):
        qft.dense_dft(u, qft.build_twiddles(256), qft.KernelPlan(tiles=2))


@pytest.mark.parametrize("q", [1 << 18, 1 << 21])
def test_dft_sharded_rows_bitwise_identical(q):
    # output sharding must not change any value (multi-GPU bitwise requirement),
    # including across the engine-selection threshold of the uniform path
    c0, r = 11, 12
    M = (q - 1 - c0) // r + 1
    sup = torch.arange(M, dtype=torch.int64, device="cuda") * r + c0
    amps = dev.fill_progression(sup, M, c0, r, M, complex(1 / math.sqrt(M)))
    for fn in (lambda lo, cnt: dev.dft(amps, M, c0, r, q, lo, cnt)[0],
               lambda lo, cnt: dev.dft_uniform(complex(1 / math.sqrt(M)), M, c0, r, q, lo, cnt)[0]):
        full = fn(0, q).cpu().numpy()
        for g in (2, 4, 8):
            parts = [fn(s * q // g, q // g).cpu().numpy() for s in range(g)]
            assert np.array_equal(np.concatenate(parts).view(np.uint64), full.view(np.uint64))


def test_host_abi_dropins(golden_dir):
    lib = nat.load()
    d = np.load(golden_dir / "random_states.npz")
    z = np.ascontiguousarray(d["1024_state"])
    out = np.empty_like(z)
    nat.check(lib.shb_dense_dft_host(z.ctypes.data, z.size, 1, 0, out.ctypes.data))
    assert np.max(np.abs(out - d["1024_dense"])) < 1e-12
    nat.check(lib.shb_dense_dft_host(z.ctypes.data, z.size, 8, 0, out.ctypes.data))
    assert np.max(np.abs(out - d["1024_tiled8"])) < 1e-12
    # the _kernels.partial_row_sums seam: unscaled rows over an input window
    rows = np.arange(100, 164, dtype=np.uint64)
    part = np.empty(64, dtype=np.complex128)
    nat.check(lib.shb_partial_row_sums_host(part.ctypes.data, z.ctypes.data, None, z.size, 100, 164, 256, 768))
    ref = oracle.dense_rows_literal(z, rows, 256, 768)
    assert np.max(np.abs(part - ref)) < 1e-12
    with pytest.raises(ValueError):
        nat.check(lib.shb_dense_dft_host(z.ctypes.data, 1000, 1, 0, out.ctypes.data))


@pytest.mark.parametrize("kind", ["full_comb", "partial_comb", "late_bump", "random_head"])
@pytest.mark.parametrize("pinned", [False, True])
def test_host_dense_dft_speculative_start(kind, pinned):
    """shb_dense_dft_host on a 2^24 state starts the first output slice's DFT
    from the uploaded head (1/64) when the head is a uniform progression,
    assuming a full comb, and confirms with a scan of the whole state.  Every
    outcome -- confirmed (full comb), refuted by the length (partial comb) or
    by the amplitudes (a bump past the head), or no speculation (non-uniform
    head) -- must give exactly the bits of the device-resident path
    (qft.dense_dft on a DeviceSpectrum), in pageable and in page-locked host
    memory."""
    q, c0, r = 1 << 24, 29, 116
    rng = np.random.default_rng(3)
    M = (q - 1 - c0) // r + 1
    st = torch.zeros(2 * q, dtype=torch.float64, pin_memory=pinned).numpy().view(np.complex128)
    idx = c0 + r * np.arange(M)
    st[idx] = 1 / math.sqrt(M)
    if kind == "partial_comb":
        st[idx[M // 2:]] = 0
    elif kind == "late_bump":
        st[idx[3 * M // 4]] *= 2
    elif kind == "random_head":
        st[idx[:100]] = rng.standard_normal(100)
    out = torch.empty(2 * q, dtype=torch.float64, pin_memory=pinned).numpy().view(np.complex128)
    lib = nat.load()
    nat.check(lib.shb_dense_dft_host(st.ctypes.data, q, 1, 0, out.ctypes.data))
    on_dev = dev.DeviceSpectrum(q, torch.from_numpy(st.view(np.float64)).cuda())
    ref = qft.dense_dft(on_dev, qft.build_twiddles(q, max_width=24), qft.KernelPlan()).numpy()
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))
    rows = rng.integers(0, q, 64, dtype=np.uint64)
    supp = np.flatnonzero(st).astype(np.uint64)
    want = oracle.dft_rows(supp, st[supp.astype(np.int64)], q, rows)
    assert np.max(np.abs(out[rows.astype(np.int64)] - want)) < 1e-12 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("tiles,precision", [(4, "fp64"), (1, "fp32"), (2, "fp32")])
def test_host_dense_dft_speculative_tiles_and_fp32(tiles, precision):
    """The speculative start with the split-K (tiled_dft) and FP32 fast-path
    kernels: the host-buffer call equals the device-resident path bit for bit."""
    q, c0, r = 1 << 24, 5, 300
    M = (q - 1 - c0) // r + 1
    st = np.zeros(q, dtype=np.complex128)
    st[c0 + r * np.arange(M)] = 1 / math.sqrt(M)
    out = np.empty(q, dtype=np.complex128)
    lib = nat.load()
    nat.check(lib.shb_dense_dft_host(st.ctypes.data, q, tiles, dev.PRECISIONS[precision], out.ctypes.data))
    on_dev = dev.DeviceSpectrum(q, torch.from_numpy(st.view(np.float64)).cuda())
    plan = qft.KernelPlan(tiles=tiles, precision=precision)
    fn = qft.tiled_dft if tiles > 1 else qft.dense_dft
    ref = fn(on_dev, qft.build_twiddles(q, max_width=24), plan).numpy()
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))


# ------------------------------------------------------------------ sampling

def _adversarial_probs(rng, n):
    kinds = [
        rng.random(n) ** 8,
        np.where(rng.random(n) < 0.9, 0.0, rng.random(n)),
        np.full(n, 2.0 ** -20),
        (rng.integers(0, 4, n) * 2.0 ** -30),
        np.exp(rng.normal(-30, 12, n)),
        np.concatenate([[1e-300, 5e-324], rng.random(max(n - 2, 0)) * 1e-9])[:n],
        # odd multiples of 2^-54: every add in [0.5, 1) is an exact round-half-even tie
        (2 * rng.integers(0, 1 << 10, n) + 1) * 2.0 ** -54,
    ]
    out = [np.ascontiguousarray(k / k.sum() if k.sum() > 0 else k) for k in kinds[:-1]]
    return out + [np.ascontiguousarray(kinds[-1])]


@pytest.mark.parametrize("n", [1, 7, 8192, 8193, 100003, 1 << 20])
def test_exact_cumsum_emulation(n):
    rng = np.random.default_rng(n)
    for p in _adversarial_probs(rng, n):
        pd = torch.from_numpy(p).cuda()
        cum = np.cumsum(p)
        total = dev.cumsum_total(pd)
        assert np.float64(total).view(np.uint64) == cum[-1].view(np.uint64)
        for u in (0.0, 0.25, 0.5, 0.999, float(np.nextafter(1.0, 0.0))) + tuple(rng.random(5)):
            target = u * cum[-1]
            want = int(np.searchsorted(cum, target, side="right"))
            assert dev.cumsum_search(pd, target) == want
        # exact hits on CDF values (the boundary case)
        for i in rng.integers(0, n, 5):
            want = int(np.searchsorted(cum, cum[i], side="right"))
            assert dev.cumsum_search(pd, float(cum[i])) == want
        # the fused Born-rule read used by sample_part1
        u = float(rng.random())
        m, tot = dev.sample_index(pd, u)
        assert tot == cum[-1] and m == int(np.searchsorted(cum, u * cum[-1], side="right"))


def test_sample_part1_vs_reference(golden_dir):
    d = np.load(golden_dir / "sampling.npz")
    z = d["state"]
    reg = qstate.CompositeRegister(q=z.size, amplitudes=z, residues=np.zeros(z.size, np.int64))
    for u, m in d["draws"]:
        assert qstate.sample_part1(reg, Forced([float(u)])) == int(m)
    # SPEC.md:170-172
    pure = np.zeros(16, complex)
    pure[3] = 1
    reg = qstate.CompositeRegister(q=16, amplitudes=pure, residues=np.zeros(16, np.int64))
    assert qstate.sample_part1(reg, Forced([0.7])) == 3
    reg = qstate.init_uniform(4)
    assert qstate.sample_part1(reg, Forced([0.99])) == 3


# ------------------------------------------------------------------ end to end

def test_run_shor_traces_vs_reference(kats):
    for run in kats["traces"]:
        cfg = dict(run["cfg"])
        cfg.setdefault("kernel", "fft")
        res = shor.run_shor(shor.ShorConfig(n=run["n"], max_width=32, **cfg))
        assert res.succeeded == run["succeeded"]
        assert res.factors == run["factors"], run
        assert len(res.attempts) == len(run["attempts"])
        for got, want in zip(res.attempts, run["attempts"]):
            assert (got.x, got.q, got.k, got.m) == (want["x"], want["q"], want["k"], want["m"]), run["n"]
            assert got.outcome.kind == want["outcome"]["kind"]
            if want["candidate"]:
                assert got.candidate.p == want["candidate"]["p"]


def test_pipeline_q2_24_properties():
    # n=3127 seed 0 attempt 1: x=1991, r=116, k=825, c0=29, M=144631, m=578525
    s = qstate.Sampler(0)
    x = shor._draw_base(3127, s)
    assert x == 1991
    reg = qstate.entangle_modexp(qstate.init_uniform(1 << 24), x, 3127)
    k, rc = qstate.measure_part2(reg, s)
    a = rc.amplitudes
    assert (k, a.a0, a.stride, a.m, a.length) == (825, 29, 116, 144631, 144631)
    spec = qft.transform(rc.amplitudes, "dense", qft.build_twiddles(1 << 24), qft.KernelPlan())
    assert abs(qstate.l2_norm(qstate.CompositeRegister(1 << 24, spec, None)) - 1.0) < 1e-9
    m = qstate.sample_part1(qstate.CompositeRegister(1 << 24, spec, None), s)
    assert m == 578525


def test_full_spectrum_q2_30_vs_cufft():
    """Whole q = 2^30 spectrum against an independent oracle (test-only):
    V_k = (1/sqrt q) sum_j e^{+2 pi i jk/q} V_j = sqrt(q) * ifft(V)[k] (cuFFT).
    A sparse comb (M = 1031) keeps the direct DFT at ~1e12 phase terms."""
    q = 1 << 30
    c0, r, M = 12345, 1_000_003, 1031
    amp = complex(1.0 / math.sqrt(M))
    out, prob, bsum = dev.dft_uniform(amp, M, c0, r, q, 0, q)
    state = torch.zeros(q, dtype=torch.complex128, device="cuda")
    state[c0: c0 + r * M: r] = amp
    ref = torch.fft.ifft(state) * math.sqrt(q)
    del state
    got = out.view(torch.complex128)
    assert float((got - ref).abs().max()) < 1e-12
    pr = ref.abs() ** 2
    assert float((prob - pr).abs().max() / pr.max()) < 1e-9
    assert abs(dev.dsum(bsum) - 1.0) < 1e-9
    # generic (TMA-staged) kernel on the same comb, output shard only
    amps = dev.fill_progression(None, M, c0, r, M, amp)
    part, _, _ = dev.dft(amps, M, c0, r, q, q // 2, 1 << 20)
    assert float((part.view(torch.complex128) - ref[q // 2: q // 2 + (1 << 20)]).abs().max()) < 1e-12


def test_cli_factor_and_bench_suite(capsys):
    from paper_1801_01434_b200 import cli
    assert cli.main(["factor", "--n", "77", "--kernel", "dense"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["factors"] == [7, 11] and 0.0 <= out["qft_fraction"] <= 1.0
    # SPEC acceptance 1 (cofactor multisets of Table 3), small suite, two engine names
    assert cli.main(["bench", "--suite", "table3-small", "--engines", "dense,fft", "--format", "csv"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    cof = {(ln.split(",")[0], ln.split(",")[2]): ln.split(",")[1] for ln in lines[1:]}
    assert cof[("77", "dense")] == "7x11" and cof[("231", "fft")] == "3x7x11" and cof[("255", "dense")] == "3x5x17"


@pytest.mark.parametrize("world", [2, 3, 8])
def test_exponent_shards_reassemble_bitwise(world):
    """What each rank of distributed.sharded_attempt computes on its a-slice:
    residues, accumulated class counts and offset compactions reassemble to the
    single-GPU results exactly."""
    from paper_1801_01434_b200 import distributed as D
    x, n, q = 8477, 32399, 1 << 22
    full = dev.modexp(x, n, q)
    counts_full = dev.class_counts(full, n)
    k = int(full[12345].item()) & 0xFFFFFFFF
    sup_full = dev.compact_eq(full, k)
    counts = torch.zeros(n, dtype=torch.int64, device="cuda")
    sups = []
    for g in range(world):
        lo, hi = D.shard(q, g, world)
        res = dev.modexp(x, n, hi - lo, a_begin=lo)
        assert torch.equal(res, full[lo:hi])
        dev.class_counts(res, n, out=counts)  # accumulates, like the all_reduce
        sups.append(dev.compact_eq(res, k, a_begin=lo))
    assert torch.equal(counts, counts_full)
    assert torch.equal(torch.cat(sups), sup_full)
    assert dev.support_progression(torch.cat(sups)) == dev.support_progression(sup_full)


def test_fp32_pipeline_end_to_end():
    # the FP32 fast path through the public API: same k, m and factors as FP64
    res64 = shor.run_shor(shor.ShorConfig(n=3127, seed=0, kernel="dense", max_width=32))
    res32 = shor.run_shor(shor.ShorConfig(n=3127, seed=0, kernel="dense", max_width=32,
                                          plan=qft.KernelPlan(precision="fp32")))
    assert res32.factors == res64.factors == [53, 59]
    assert [(a.k, a.m) for a in res32.attempts] == [(a.k, a.m) for a in res64.attempts]


def _two_rank_worker(rank, world, port, ret):
    import os
    import torch.distributed as dist
    from paper_1801_01434_b200 import distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = qstate.Sampler(0)
        x = shor._draw_base(3127, s)
        rec = D.sharded_attempt(3127, x, 1 << 24, s, rank=rank, world=world, keep_spectrum=True)
        out, _ = rec.spectrum
        lo, hi = D.shard(1 << 24, rank, world)
        rows = torch.tensor([0, 1, 144631, 578525, 12345678], device="cuda")
        rows = rows[(rows >= lo) & (rows < hi)] - lo
        ret[rank] = {"x": x, "k": rec.k, "m": rec.m, "M": rec.M, "r": rec.r, "c0": rec.c0,
                     "rows": (rows + lo).tolist(),
                     "vals": out.view(torch.complex128)[rows].cpu().numpy().view(np.float64).tolist()}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_attempt_ranks_on_device(world):
    """distributed.sharded_attempt with the real device kernels, 2 ranks on one
    GPU (gloo collectives: host-staged; the kernels never wait on each other).
    Same k, m, support and bitwise-identical spectrum rows as 1 rank."""
    import socket

    import torch.multiprocessing as mp
    from paper_1801_01434_b200 import distributed as D
    s = qstate.Sampler(0)
    x = shor._draw_base(3127, s)
    one = D.sharded_attempt(3127, x, 1 << 24, s, keep_spectrum=True)
    full, _ = one.spectrum
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    ret = ctx.Manager().dict()
    procs = [ctx.Process(target=_two_rank_worker, args=(r, world, port, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    for r in range(world):
        g = ret[r]
        assert (g["k"], g["m"], g["M"], g["r"], g["c0"]) == (one.k, one.m, one.M, one.r, one.c0) == \
            (825, 578525, 144631, 116, 29)
        ref = full.view(torch.complex128)[torch.tensor(g["rows"], dtype=torch.int64, device="cuda")].cpu().numpy().view(np.float64)
        assert np.array_equal(np.asarray(g["vals"]), ref)


def test_edge_cases_vs_oracle():
    rng = np.random.default_rng(11)
    # smallest register, basis and random states
    for st in ([1, 0], [0, 1], [0.6, 0.8j]):
        z = np.asarray(st, dtype=np.complex128)
        got = qft.dense_dft(z, qft.build_twiddles(2), qft.KernelPlan())
        assert np.max(np.abs(got - oracle.dense_dft(z))) < 1e-15
    # all-zero state -> zeros; single element at the last index (progression length 1)
    q = 1 << 12
    assert not np.any(qft.dense_dft(np.zeros(q, complex), qft.build_twiddles(q), qft.KernelPlan()))
    z = np.zeros(q, complex)
    z[q - 1] = 1j
    assert np.max(np.abs(qft.dense_dft(z, qft.build_twiddles(q), qft.KernelPlan()) - oracle.dense_dft(z))) < 1e-14
    # support with holes (gcd stride 3, one zero slot) -> generic kernel
    z = np.zeros(q, complex)
    z[[1, 4, 10, 4000]] = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    for tiles in (1, 2, 16, q):
        plan = qft.KernelPlan(tiles=tiles)
        fn = qft.dense_dft if tiles == 1 else qft.tiled_dft
        ref = oracle.dense_dft(z) if tiles == 1 else oracle.tiled_dft(z, tiles)
        assert np.max(np.abs(fn(z, qft.build_twiddles(q), plan) - ref)) < 1e-13, tiles
    # ragged output ranges on both kernels (partial CTAs)
    sup = torch.arange(100, dtype=torch.int64, device="cuda") * 7 + 3
    amps = dev.fill_progression(sup, 100, 3, 7, 100, 0.1 + 0.2j)
    for lo, cnt in [(0, 1), (5, 1023), (999, 1025), (q - 3, 3)]:
        out, _, _ = dev.dft(amps, 100, 3, 7, q, lo, cnt)
        ou, _, _ = dev.dft_uniform(0.1 + 0.2j, 100, 3, 7, q, lo, cnt)
        ref = oracle.dft_rows(3 + 7 * np.arange(100, dtype=np.uint64), np.full(100, 0.1 + 0.2j), q,
                              np.arange(lo, lo + cnt, dtype=np.uint64))
        assert np.max(np.abs(out.cpu().numpy().view(np.complex128) - ref)) < 1e-14
        assert np.max(np.abs(ou.cpu().numpy().view(np.complex128) - ref)) < 1e-14


def test_modexp_edge_bases():
    # x >= n reduces mod n; x = 1 gives all ones; n = 2 (every residue 1)
    assert np.array_equal(dev.modexp(15 + 7, 15, 64).cpu().numpy(), oracle.modexp_residues(7, 15, 64).view(np.int32))
    assert np.all(dev.modexp(1, 15, 100).cpu().numpy() == 1)
    assert np.all(dev.modexp(3, 2, 50).cpu().numpy() == 1)
    reg = qstate.entangle_modexp(qstate.init_uniform(8), 1, 15)
    k, rc = qstate.measure_part2(reg, Forced([0.5]))
    assert k == 1 and rc.amplitudes.m == 8 and abs(qstate.l2_norm(rc) - 1) < 1e-15


@pytest.mark.parametrize("tag,n,attempt,q", [("n3127", 3127, 1, 1 << 24), ("n221", 221, 2, 1 << 16)])
def test_sampled_m_matches_reference_over_1000_draws(golden_dir, tag, n, attempt, q):
    """m over 1000 random draws equals the reference's m on the reference's own
    spectrum (fft engine at 2^24, dense at 2^16): our spectrum differs at ~1e-13
    and our cumsum is the exact sequential emulation, so no draw flips.  The 60
    adversarial draws placed within one ulp of peak CDF boundaries are reported."""
    d = np.load(golden_dir / "sampling_sweep.npz")
    s = qstate.Sampler(0)
    for a in range(attempt):
        x = shor._draw_base(n, s)
        reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
        k, rc = qstate.measure_part2(reg, s)
        if a < attempt - 1:
            s.uniform()
    assert (x, k) == (int(d[f"{tag}_x"]), int(d[f"{tag}_k"]))
    spec = qft.transform(rc.amplitudes, "dense", qft.build_twiddles(q), qft.KernelPlan())
    p = spec.probabilities()
    us, ms = d[f"{tag}_u"], d[f"{tag}_m"]
    got = np.array([min(dev.sample_index(p, float(u))[0], q - 1) for u in us])
    assert np.array_equal(got[:1000], ms[:1000])
    boundary_flips = int(np.sum(got[1000:] != ms[1000:]))
    print(f"{tag}: 1000/1000 random draws equal; boundary-adversarial flips {boundary_flips}/{len(us) - 1000}")
    assert boundary_flips <= len(us) - 1000


def test_qft_fourth_power_is_identity_on_device():
    """F^2 reverses indices (c -> -c mod q) and F^4 = I, with every
    intermediate staying on the device (DeviceSpectrum -> dense progression)."""
    q = 1 << 12
    rng = np.random.default_rng(4)
    z = rng.standard_normal(q) + 1j * rng.standard_normal(q)
    z /= np.linalg.norm(z)
    t = torch.from_numpy(z.view(np.float64)).cuda()
    st = dev.DeviceSpectrum(q, t)
    tw, plan = qft.build_twiddles(q), qft.KernelPlan()
    f2 = qft.dense_dft(qft.dense_dft(st, tw, plan), tw, plan)
    assert isinstance(f2, dev.DeviceSpectrum)
    assert np.max(np.abs(np.asarray(f2) - z[(-np.arange(q)) % q])) < 1e-12
    f4 = qft.dense_dft(qft.dense_dft(f2, tw, plan), tw, plan)
    assert np.max(np.abs(np.asarray(f4) - z)) < 1e-12
    assert abs(qstate.l2_norm(qstate.CompositeRegister(q, f4, None)) - 1.0) < 1e-12


def test_c_abi_demo_program(tmp_path):
    import subprocess
    from conftest import build_c_demo
    exe = build_c_demo(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "row64 = 8" in r.stdout


@pytest.mark.parametrize("engine,real_form", [("vector", "1"), ("mma", "0"), ("mma", "1"), ("i8", "1")])
def test_both_fp64_engines_vs_oracle(engine, real_form, monkeypatch):
    """The FP64 DFT kernels for tiles == 1: the vector Horner kernel, the DMMA
    (FP64 tensor-core) GEMM-factored kernel in a complex-A and a real-A form
    (2 DMMAs per k-step; uniform combs and real amplitudes), and the int8
    tensor-core engine of the uniform comb (8-digit exact split of G, FP64
    folds; under "i8" the generic/real calls still take DMMA).  All against
    the oracle on ragged sizes, output shards and the uniform / generic / real
    amplitude paths."""
    monkeypatch.setenv("SHB_DFT_ENGINE", engine)
    monkeypatch.setenv("SHB_MMA_REAL", real_form)
    rng = np.random.default_rng(21)
    for q, c0, r, M in [(2, 1, 1, 1), (8, 3, 2, 3), (1 << 10, 5, 3, 1), (1 << 10, 5, 3, 255), (1 << 12, 1, 7, 585),
                        (1 << 16, 11, 12, 5461)]:
        supp = c0 + r * np.arange(M, dtype=np.uint64)
        amps_h = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        amps = torch.from_numpy(amps_h.view(np.float64)).cuda()
        for lo, cnt in ([(0, q), (77, 129), (q - 130, 130)] if q > 256 else [(0, q), (1, q - 1)]):
            rows = np.arange(lo, lo + cnt, dtype=np.uint64)
            out, prob, bs = dev.dft(amps, M, c0, r, q, lo, cnt)
            ref = oracle.dft_rows(supp, amps_h, q, rows)
            assert np.max(np.abs(out.cpu().numpy().view(np.complex128) - ref)) < 1e-12 * max(1, np.abs(ref).max())
            assert abs(dev.dsum(bs) - float(prob.sum())) <= 1e-9 * float(prob.sum())
            ou, pu, bu = dev.dft_uniform(0.3 - 0.1j, M, c0, r, q, lo, cnt)
            refu = oracle.dft_rows(supp, np.full(M, 0.3 - 0.1j), q, rows)
            assert np.max(np.abs(ou.cpu().numpy().view(np.complex128) - refu)) < 1e-12 * max(1, np.abs(refu).max())
            re_h = rng.standard_normal(M) + 0j
            re_d = torch.from_numpy(re_h.view(np.float64)).cuda()
            orl, prl, brl = dev.dft(re_d, M, c0, r, q, lo, cnt, real=True)
            refr = oracle.dft_rows(supp, re_h, q, rows)
            assert np.max(np.abs(orl.cpu().numpy().view(np.complex128) - refr)) < 1e-12 * max(1, np.abs(refr).max())
            assert abs(dev.dsum(brl) - float(prl.sum())) <= 1e-9 * float(prl.sum())


# KCH = 6 (24576 per super-block) unless KCH = 8 (32768) needs fewer super-blocks:
# 24577, 2 * 24576 + 97, 65536, 2 * 32768 + 7 * 4096 + 5 and 100003 run at KCH = 8
@pytest.mark.parametrize("M", [1, 31, 4095, 4096, 4097, 24575, 24576, 24577, 2 * 24576 + 97, 3 * 24576 - 1, 32768,
                               65536, 65537, 2 * 32768 + 7 * 4096 + 5, 100003])
def test_i8_engine_superblock_edges_vs_oracle(M, monkeypatch):
    """The int8 tensor-core FP64 engine around its K-chunk (128 row-blocks x
    32 = 4096 amplitudes) and super-block (6 chunks = 24576, or 8 = 32768)
    sizes: full,
    one-past and ragged last chunks (masked weights in TMEM, dead chunks
    skipped), against the oracle on sampled rows and on an output shard that
    is not a multiple of the 24-output tile, which must also be bitwise
    identical to the same rows of the full transform."""
    monkeypatch.setenv("SHB_DFT_ENGINE", "i8")
    q, c0, r = 1 << 21, 7, 13
    assert c0 + (M - 1) * r < q
    rng = np.random.default_rng(M)
    supp = c0 + r * np.arange(M, dtype=np.uint64)
    amp = complex(1 / np.sqrt(M))
    full, pf, bf = dev.dft_uniform(amp, M, c0, r, q, 0, q)
    rows = np.unique(np.concatenate([rng.integers(0, q, 300, dtype=np.uint64),
                                     np.array([0, 1, q - 1, q // 2, q // r], dtype=np.uint64)]))
    ref = oracle.dft_rows(supp, np.full(M, amp), q, rows)
    got = full.cpu().numpy().view(np.complex128)[rows.astype(np.int64)]
    assert np.max(np.abs(got - ref)) < 1e-12 * max(1.0, np.abs(ref).max())
    exact = oracle.comb_rows_exact(q, r, c0, M, amp, rows)
    assert np.max(np.abs(got - exact)) < 1e-13 * max(1.0, np.abs(exact).max())
    assert abs(dev.dsum(bf) - 1.0) < 1e-9
    for lo, cnt in [(1000, 777), (5, 23), (q - 25, 25)]:
        sh, _, _ = dev.dft_uniform(amp, M, c0, r, q, lo, cnt)
        assert torch.equal(sh, full[2 * lo: 2 * (lo + cnt)])


def test_dense_dft_selects_real_form_for_real_states():
    """qft.dense_dft on a real non-uniform state takes shb_dft_real (the data
    decides, as it does for the uniform comb) and matches the oracle."""
    rng = np.random.default_rng(5)
    q = 1 << 14
    st = np.zeros(q, complex)
    supp = np.arange(3, q, 9, dtype=np.uint64)
    st[supp.astype(np.int64)] = rng.standard_normal(supp.size)
    st /= np.linalg.norm(st)
    amps, length, a0, stride, host, real = qft._support_of(st, q)
    assert real and not isinstance(amps, complex) and (a0, stride, length) == (3, 9, supp.size)
    out = np.asarray(qft.dense_dft(st, qft.build_twiddles(q), qft.KernelPlan()))
    rows = np.arange(q, dtype=np.uint64)
    ref = oracle.dft_rows(supp, st[supp.astype(np.int64)], q, rows)
    assert np.max(np.abs(out - ref)) < 1e-12
    st[5] = 1e-3j  # one complex amplitude: the complex form
    assert not qft._support_of(st, q)[5]


# ------------------------------------------------------------ SPEC acceptance
# SPEC.md:467-478, the reference's own acceptance contract, on the B200 path.

TABLE3 = {77: [7, 11], 143: [11, 13], 323: [17, 19], 551: [19, 29], 589: [19, 31],
          231: [3, 7, 11], 255: [3, 5, 17], 399: [3, 7, 19], 423: [3, 3, 47], 539: [7, 7, 11]}


def test_spec_acceptance_1_table3_full_cofactors():
    for n, cof in TABLE3.items():
        res = shor.run_shor(shor.ShorConfig(n=n, seed=0, kernel="fft"))
        assert res.succeeded and res.factors == cof, n


def test_spec_acceptance_2_dense_fft_same_m():
    for n in (77, 143):
        a = shor.run_shor(shor.ShorConfig(n=n, seed=3, kernel="dense"))
        b = shor.run_shor(shor.ShorConfig(n=n, seed=3, kernel="fft"))
        assert a.factors == b.factors and [t.m for t in a.attempts] == [t.m for t in b.attempts]


def test_spec_acceptance_8_qft_dominates_at_scale():
    # the paper's "97% of the runtime": on the GPU the QFT share
    # grows with q; at q = 2^24 it dominates the attempt
    res = shor.run_shor(shor.ShorConfig(n=3127, seed=0, kernel="dense", max_width=24))
    assert shor.profile_phases(res)["qft"] > 0.9


def test_spec_acceptance_9_worker_invariance():
    a = shor.run_shor(shor.ShorConfig(n=323, seed=42, kernel="dense", plan=qft.KernelPlan(workers=1)))
    b = shor.run_shor(shor.ShorConfig(n=323, seed=42, kernel="dense", plan=qft.KernelPlan(workers=8)))
    assert a.factors == b.factors == [17, 19]
    assert [(t.x, t.k, t.m) for t in a.attempts] == [(t.x, t.k, t.m) for t in b.attempts]


def test_spec_acceptance_10_period_recovery_rate():
    """SPEC.md:478 asks for >= 90% exact-period recovery over 200 seeded draws on
    n in {15, 21, 33, 35}.  The reference code itself recovers 78 of the 106
    draws that reach the quantum path (73.6%; computed in the build container by
    running shorsim on this very loop) -- the B200 path must reproduce that
    count exactly, accept only verified periods and retry-classify the rest."""
    ok = total = 0
    for n in (15, 21, 33, 35):
        for seed in range(50):
            s = qstate.Sampler(seed)
            x = shor._draw_base(n, s)
            if math.gcd(x, n) > 1:
                continue
            q = nt.choose_register_width(n).q
            reg = qstate.entangle_modexp(qstate.init_uniform(q), x, n)
            k, rc = qstate.measure_part2(reg, s)
            spec = qft.transform(rc.amplitudes, "dense", qft.build_twiddles(q), qft.KernelPlan())
            m = qstate.sample_part1(qstate.CompositeRegister(q, spec, None), s)
            est = nt.extract_period(m, q, n, x)
            total += 1
            if isinstance(est, nt.PeriodCandidate):
                assert nt.modpow(x, est.p, n) == 1  # every acceptance is a true period multiple
                ok += est.p == nt.classical_period(x, n)
            else:
                assert est.kind == "retry"  # failures are retry-classified
    assert (ok, total) == (78, 106)  # the reference's own outcome on the same draws


def test_fp64_peak_probes():
    """The bench's FP64 roofline probes (DFMA chains and DMMA chains) report a
    throughput near the nominal 148 SM x 64 FMA/clk x 2 flops (37 TF/s at
    1.965 GHz): a sanity bound on the denominators the bench prints."""
    import ctypes
    lib = nat.load()
    for fn in (lib.shb_fp64_peak, lib.shb_fp64_dmma_peak):
        tf = ctypes.c_double()
        nat.check(fn(0.2, ctypes.byref(tf), None), "probe")
        assert 15.0 < tf.value < 45.0, tf.value


def test_chained_device_cumsum_matches_whole_vector(golden_dir):
    """The device halves of the sharded Born-rule read: shb_cumsum_total_from /
    shb_cumsum_search_from chained over 2..8 shards of a probability vector
    give the same total (bitwise) and the same m as shb_sample_index on the
    whole vector, on the reference's draws and on adversarial vectors (tie
    storms, long zero runs, subnormals)."""
    d = np.load(golden_dir / "sampling.npz")
    rng = np.random.default_rng(17)
    vecs = [(oracle.probabilities(d["state"]), [float(u) for u, _ in d["draws"]])]
    ties = np.full(1 << 16, 2.0 ** -20)
    ties[::3] = 2.0 ** -53
    zeros = rng.random(1 << 18) * (rng.random(1 << 18) < 0.1)
    sub = np.concatenate([np.full(1000, 5e-324), rng.random(50000)])
    vecs += [(v, list(rng.random(40))) for v in (ties, zeros, sub)]
    for p_h, us in vecs:
        p = torch.from_numpy(np.ascontiguousarray(p_h)).cuda()
        n = p_h.size
        for world in (2, 3, 8):
            cuts = [0] + sorted(rng.choice(np.arange(1, n), world - 1, replace=False).tolist()) + [n]
            bounds, s = [], 0.0
            for g in range(world):
                s_out = dev.cumsum_total_from(p[cuts[g]:cuts[g + 1]], s)
                bounds.append((s, s_out))
                s = s_out
            m_all, tot = dev.sample_index(p, 0.5)
            assert s == tot == float(np.cumsum(p_h)[-1])
            for u in us:
                target = u * s
                owner = next((g for g in range(world) if bounds[g][1] > target), None)
                got = n if owner is None else cuts[owner] + dev.cumsum_search_from(
                    p[cuts[owner]:cuts[owner + 1]], bounds[owner][0], target)
                assert got == dev.sample_index(p, u)[0]


@pytest.mark.parametrize("hint_kind", ["approx", "zero", "wrong"])
def test_split_cumsum_records_walk_find(golden_dir, hint_kind):
    """The split sequential cumsum of the sharded read (distributed._sharded_sample,
    shb_sample): per-shard records from a hint (the all-gathered approximate
    shard sums, or a useless 0 / wildly wrong hint), the exact walk chained
    shard to shard, and the search in the owning shard -- same total (bitwise)
    and same m as shb_sample_index on the whole vector, whatever the hint."""
    d = np.load(golden_dir / "sampling.npz")
    rng = np.random.default_rng(29)
    ties = np.full(1 << 16, 2.0 ** -20)
    ties[::3] = 2.0 ** -53
    zeros = rng.random(1 << 18) * (rng.random(1 << 18) < 0.1)
    big = rng.random(3 << 20)
    vecs = [oracle.probabilities(d["state"]), ties, zeros, big / big.sum()]
    for p_h in vecs:
        p = torch.from_numpy(np.ascontiguousarray(p_h)).cuda()
        n = p_h.size
        for world in (2, 5):
            cuts = [0] + sorted(rng.choice(np.arange(1, n), world - 1, replace=False).tolist()) + [n]
            shards = [p[cuts[g]:cuts[g + 1]] for g in range(world)]
            approx = [dev.dsum(sh) for sh in shards]
            plans = []
            for g, sh in enumerate(shards):
                hint = {"approx": float(sum(approx[:g])), "zero": 0.0, "wrong": 1e6 * (g + 1)}[hint_kind]
                plans.append(dev.cumsum_plan(sh, hint))
            bounds, s = [], 0.0
            for g, sh in enumerate(shards):
                s_out = dev.cumsum_walk(sh, plans[g], s)
                bounds.append((s, s_out))
                s = s_out
            assert s == dev.sample_index(p, 0.5)[1] == float(np.cumsum(p_h)[-1])
            for u in list(rng.random(25)) + [0.0, float(np.nextafter(1.0, 0.0))]:
                target = u * s
                owner = next((g for g in range(world) if bounds[g][1] > target), None)
                got = n if owner is None else cuts[owner] + dev.cumsum_find(
                    shards[owner], plans[owner], bounds[owner][1], target)
                assert got == dev.sample_index(p, u)[0], (hint_kind, world, u)
