"""Pin the CPU oracle against golden vectors produced by the reference itself.

These run without a GPU.  If any of them fails, the oracle is not a trustworthy
checker and every GPU parity test downstream is meaningless.
"""

import json
import math

import numpy as np
import pytest

from oracle import oracle


@pytest.fixture(scope="module")
def kats(golden_dir):
    return json.loads((golden_dir / "kats.json").read_text())


def _load_spec(golden_dir, tag):
    d = np.load(golden_dir / f"spectrum_{tag}.npz")
    return {k: d[k] for k in d.files}


def test_root_table_bitwise(kats):
    for q, vals in kats["twiddles"].items():
        q = int(q)
        got = oracle.roots(q, np.arange(q))
        ref = np.array([complex(a, b) for a, b in vals])
        assert np.array_equal(got.view(np.float64), ref.view(np.float64))
    # wide tables: compare with numpy's own expression (qft.py:79) on samples
    for w in (16, 24, 30, 32):
        q = 1 << w
        idx = np.random.default_rng(w).integers(0, q, 20000, dtype=np.uint64)
        ref = np.exp((2j * np.pi / q) * idx.astype(np.int64))
        assert np.array_equal(oracle.roots(q, idx).view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("tag", ["n15", "n15x2", "n221a1", "n221a2", "n3127"])
def test_dft_rows_bitwise_vs_reference(golden_dir, tag):
    d = _load_spec(golden_dir, tag)
    info = json.loads(str(d["info"]))
    q = int(d["q"])
    M, c0, r = info["M"], info["c0"], info["r"]
    amp = complex(np.uint64(int(info["amp_re_bits"], 16)).view(np.float64),
                  np.uint64(int(info["amp_im_bits"], 16)).view(np.float64))
    supp = c0 + r * np.arange(M, dtype=np.uint64)
    amps = np.full(M, amp, dtype=np.complex128)
    got = oracle.dft_rows(supp, amps, q, d["rows"])
    # bitwise, signed zeros included
    assert np.array_equal(got.view(np.uint64), d["V"].view(np.uint64))


def test_literal_rows_match_support_rows(golden_dir):
    d = _load_spec(golden_dir, "n221a2")
    info = json.loads(str(d["info"]))
    q = int(d["q"])
    amp = np.uint64(int(info["amp_re_bits"], 16)).view(np.float64)
    state = np.zeros(q, dtype=np.complex128)
    state[info["c0"]::info["r"]] = amp
    rows = d["rows"][:64]
    lit = oracle.dense_rows_literal(state, rows) * (1.0 / math.sqrt(q))
    assert np.array_equal(lit.view(np.uint64), d["V"][:64].view(np.uint64))


def test_collapse_facts(golden_dir):
    # n=15, x=2 forced k=1: support {0,4,...,252}, amplitude 1/8
    d = _load_spec(golden_dir, "n15x2")
    info = json.loads(str(d["info"]))
    assert (info["k"], info["M"], info["c0"], info["r"]) == (1, 64, 0, 4)
    p = np.abs(d["V"]) ** 2
    # exact peak law
    assert set(np.flatnonzero(p > 1e-20).tolist()) == {0, 64, 128, 192}
    assert np.allclose(p[[0, 64, 128, 192]], 0.25, atol=1e-10)


def test_random_states_dense_and_tiled(golden_dir):
    d = np.load(golden_dir / "random_states.npz")
    for key in ("16", "256", "1024", "4096", "sparse2048"):
        z = d[f"{key}_state"]
        ref_dense = d[f"{key}_dense"]
        got = oracle.dense_dft(z)
        assert np.array_equal(got.view(np.uint64), ref_dense.view(np.uint64)), key
        got_t = oracle.tiled_dft(z, 8)
        assert np.array_equal(got_t.view(np.uint64), d[f"{key}_tiled8"].view(np.uint64)), key


def test_modexp_vs_reference_vectors(kats):
    for q, x, n, res in kats["entangle"]:
        assert oracle.modexp_residues(x, n, q).tolist() == res
        assert oracle.modexp_residues_cycle(x, n, q).tolist() == res
    # shard offsets agree with the full vector
    full = oracle.modexp_residues(20637, 32399, 1 << 14)
    assert np.array_equal(oracle.modexp_residues(20637, 32399, 4096, a_begin=8192), full[8192:12288])


def test_measure_sweep_vs_reference(kats):
    # k, support and amplitude bits for 1000+ draws including odd widths
    seen = 0
    for row in kats["measure_sweep"]:
        q, x, n, u = row["q"], row["x"], row["n"], row["u"]
        res = oracle.modexp_residues(x, n, q)
        amps = np.full(q, 1.0 / math.sqrt(q), dtype=np.complex128)
        k, out = oracle.measure_part2(amps, res, u)
        assert k == row["k"]
        supp = np.flatnonzero(out)
        assert supp.size == row["M"] and supp[0] == row["c0"]
        assert out[supp[0]].real.view(np.uint64) == np.uint64(int(row["amp_re_bits"], 16))
        seen += 1
    assert seen > 500


def test_sampling_vs_reference(golden_dir):
    d = np.load(golden_dir / "sampling.npz")
    p = oracle.probabilities(d["state"])
    for u, m in d["draws"]:
        assert oracle.sample_index(p, float(u)) == int(m)
        assert oracle.sample_index_numpy(p, float(u)) == int(m)


def test_closed_form_comb_vs_reference_rows(golden_dir):
    for tag in ("n221a1", "n221a2", "n3127"):
        d = _load_spec(golden_dir, tag)
        info = json.loads(str(d["info"]))
        q = int(d["q"])
        p_ref = np.abs(d["V"]) ** 2
        p_cf = oracle.comb_probabilities(q, info["r"], info["c0"], info["M"], d["rows"])
        # the reference dense rows themselves carry ~1e-11 accumulated rounding at 2^24
        assert np.max(np.abs(p_cf - p_ref)) / np.max(p_ref) < 1e-10


def test_chained_cumsum_reproduces_reference_sampling(golden_dir):
    """The sharded Born-rule read (distributed._sharded_sample) chains the
    sequential cumsum shard to shard.  On the reference's own draws, every
    split of the probability vector into 2..8 shards gives the reference's m:
    the running sum entering a shard is exactly the one leaving the last."""
    d = np.load(golden_dir / "sampling.npz")
    p = oracle.probabilities(d["state"])
    q = p.size
    rng = np.random.default_rng(3)
    for world in (2, 3, 4, 8):
        cuts = [0] + sorted(rng.choice(np.arange(1, q), world - 1, replace=False).tolist()) + [q]
        bounds, s = [], 0.0
        for g in range(world):
            s_out = oracle.cumsum_total_from(p[cuts[g]:cuts[g + 1]], s)
            bounds.append((s, s_out))
            s = s_out
        assert s == np.cumsum(p)[-1]
        for u, m in d["draws"]:
            target = float(u) * s
            owner = next(g for g in range(world) if bounds[g][1] > target)
            got = cuts[owner] + oracle.cumsum_search_from(p[cuts[owner]:cuts[owner + 1]], bounds[owner][0], target)
            assert min(got, q - 1) == int(m)


@pytest.mark.parametrize("tag,n", [("n221a1", 221), ("n3127", 3127)])
def test_attempt_register_vs_reference_golden(golden_dir, tag, n):
    """oracle.attempt_register (the --impl reference arm's register) against the
    collapse the reference itself produced (attempt 1, seed 0), amplitude bits included."""
    d = np.load(golden_dir / f"spectrum_{tag}.npz")
    info = json.loads(str(d["info"]))
    got = oracle.attempt_register(n, 0)
    assert (got["q"], got["x"]) == (int(d["q"]), int(d["x"]))
    assert (got["k"], got["M"], got["c0"], got["r"]) == (info["k"], info["M"], info["c0"], info["r"])
    assert np.float64(got["amp"].real).view(np.uint64) == np.uint64(int(info["amp_re_bits"], 16))
    assert got["amp"].imag == 0.0


def test_attempt_register_baseline_traces():
    """SURVEY.md 8(d) attempt-1 registers at q = 2^30 / 2^32 (x, r, k, c0, M)."""
    want = {(32399, 8): (10594, 16020, 31897, 10943, 67025), (32399, 2): (8477, 5340, 9557, 4828, 201075),
            (32399, 0): (20637, 4005, 8440, 1347, 268100), (46927, 0): (29890, 23240, 12551, 11799, 184809)}
    for (n, seed), tr in want.items():
        g = oracle.attempt_register(n, seed)
        assert (g["x"], g["r"], g["k"], g["c0"], g["M"]) == tr


@pytest.mark.parametrize("tag", ["n15", "n221a1", "n221a2", "n3127"])
def test_comb_rows_exact_vs_reference_golden(golden_dir, tag):
    """The long-double closed form (accuracy reference) against the reference's
    own dense_dft rows: they differ by no more than the reference's sequential
    rounding bound 2 M 2^-53 max|V|."""
    d = np.load(golden_dir / f"spectrum_{tag}.npz")
    info = json.loads(str(d["info"]))
    if not info.get("comb"):
        pytest.skip("not a comb")
    amp = complex(np.uint64(int(info["amp_re_bits"], 16)).view(np.float64),
                  np.uint64(int(info["amp_im_bits"], 16)).view(np.float64))
    rows = d["rows"] if "rows" in d.files else np.arange(int(d["q"]))
    V = d["V"] if "V" in d.files else d["spectrum"]
    ex = oracle.comb_rows_exact(int(d["q"]), info["r"], info["c0"], info["M"], amp, rows)
    err = np.abs(ex - V).max() / np.abs(ex).max()
    assert err <= 2 * info["M"] * 2.0 ** -53, err
