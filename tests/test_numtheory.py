"""Host integer math against the reference golden vectors and SPEC invariants (CPU)."""

import json
import math

import pytest

from paper_1801_01434_b200 import numtheory as nt


@pytest.fixture(scope="module")
def kats(golden_dir):
    return json.loads((golden_dir / "kats.json").read_text())


def test_kats(kats):
    for b, e, m, want in kats["modpow"]:
        assert nt.modpow(b, e, m) == want
    for a, b, want in kats["gcd"]:
        assert nt.gcd(a, b) == want
    for n, q, w in kats["register_width"]:
        assert nt.choose_register_width(n, 32) == nt.RegisterWidth(q=q, w=w)
    for x, n, p in kats["classical_period"]:
        assert nt.classical_period(x, n) == p
    for m, q, conv in kats["convergents"]:
        assert [list(c) for c in nt.convergents(m, q)] == conv
    for m, q, n, x, want in kats["extract_period"]:
        got = nt.extract_period(m, q, n, x)
        if "p" in want:
            assert (got.p, list(got.source_convergent), got.multiplier) == (
                want["p"], want["source_convergent"], want["multiplier"])
        else:
            assert (got.kind, got.reason) == (want["kind"], want["reason"])
    for n, x, p, want in kats["derive_factors"]:
        got = nt.derive_factors(n, x, p)
        assert got.kind == want["kind"] and got.reason == want["reason"]
        assert (list(got.factors) if got.factors else None) == want["factors"]


def test_guards():
    with pytest.raises(ValueError):
        nt.choose_register_width(32399)  # default max_width 24 (numtheory.py:166)
    with pytest.raises(nt.NothingToFactor):
        nt.pre_checks(46927 * 0 + 101)
    assert nt.pre_checks(15) is None
    assert nt.pre_checks(16).factors == (2, 8)
    assert nt.pre_checks(49).factors == (7, 7)
    with pytest.raises(ValueError):
        nt.gcd(0, 0)
    with pytest.raises(ValueError):
        nt.modpow(2, 3, 1)
    with pytest.raises(ValueError):
        nt.convergents(5, 5)
    with pytest.raises(ValueError):
        nt.FactorOutcome.retry("nope")


def test_spec_invariants():
    for n in range(3, 3000):
        rw = nt.choose_register_width(n, 32)
        assert n * n <= rw.q < 2 * n * n and rw.q == 1 << rw.w
    for n in range(3, 300):
        for x in range(2, n):
            if math.gcd(x, n) != 1:
                continue
            out = nt.derive_factors(n, x, nt.classical_period(x, n))
            if out.kind == "factors":
                f1, f2 = out.factors
                assert f1 * f2 == n and 1 < f1 <= f2 < n
    for m in range(1, 512):
        cs = nt.convergents(m, 512)
        assert cs[-1][0] * 512 == m * cs[-1][1] or cs[-1] == (m // math.gcd(m, 512), 512 // math.gcd(m, 512))
        assert all(math.gcd(a, b) == 1 for a, b in cs)
        assert all(cs[i][1] < cs[i + 1][1] for i in range(1, len(cs) - 1))
    for b in range(0, 20):
        for e in range(0, 20):
            for m in range(2, 30):
                assert nt.modpow(b, e, m) == (b ** e) % m
    for n in range(2, 5000):
        assert nt.is_prime(n) == (n > 1 and all(n % d for d in range(2, int(n ** 0.5) + 1)))
