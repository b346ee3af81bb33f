"""Pins for the oracle's key schedule (§3.1, Eqs.2-7).

Each test checks the oracle against something other than itself: SPEC's worked
examples (tests/golden/spec_examples.json), the paper's printed ranges
(tests/golden/paper_constants.json), exact integer / rational arithmetic,
invertibility, or hashlib.
"""
import hashlib
import json
import math
import os
import random
from fractions import Fraction

import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
PAPER = json.load(open(os.path.join(GOLD, "paper_constants.json")))


# ------------------------------------------------------------ Eqs.2-4 packing
def test_pack_spec_examples(ref):
    for ex in SPEC["pack"]:
        a = ref.pack(ex["pw"].encode())
        if "a" in ex:
            assert list(a) == ex["a"], ex["cite"]
        else:
            assert a[1] == ex["a2"], ex["cite"]


def _unpack(a, n):
    """Invert Eqs.2-4 (positional base-256 digits) back to the password bytes."""
    L, rem = n // 3, n % 3
    a1, a2, a3 = a
    pw = [None] * n
    if rem == 0:
        for i in range(L):
            pw[i] = (a1 >> (8 * i)) & 0xFF
    else:
        pw[3 * L] = a1 & 0xFF
        for i in range(L):
            pw[i] = (a1 >> (8 * (i + 1))) & 0xFF
    if rem == 2:
        pw[3 * L + 1] = a2 & 0xFF
        for i in range(L):
            pw[L + i] = (a2 >> (8 * (i + 1))) & 0xFF
    else:
        for i in range(L):
            pw[L + i] = (a2 >> (8 * i)) & 0xFF
    for i in range(L):
        pw[2 * L + i] = (a3 >> (8 * i)) & 0xFF
    # high bytes beyond the packed digits must be zero
    top = [8 * (L + (rem != 0)), 8 * (L + (rem == 2)), 8 * L]
    for ai, t in zip(a, top):
        assert ai >> t == 0
    return bytes(pw)


def test_pack_is_invertible_every_length(ref):
    """Injectivity at every length: unpacking recovers the password."""
    rng = random.Random(7)
    for n in range(3, 24):
        for _ in range(200):
            pw = bytes(rng.getrandbits(8) for _ in range(n))
            assert _unpack(ref.pack(pw), n) == pw


def test_pack_length_limits(ref):
    for n in (0, 1, 2, 24, 40):
        with pytest.raises(ref.OracleError):
            ref.pack(b"x" * n)


def test_pack_fits_u64_at_max_length(ref):
    a = ref.pack(b"\xff" * 23)
    assert all(0 <= x < 2 ** 64 for x in a)
    assert a[0] == 2 ** 64 - 1  # n=23: L=7, rem 2 -> eight 0xff digits


# ------------------------------------------------------------ g
def test_norm_exponent_closed_form(ref):
    for L in range(1, 8):
        k = 8 * (L + 1)
        assert ref.norm_exponent(L) == len(str(2 ** k))  # ceil(log10 2^k) = #digits(2^k)


def test_normalize_spec_examples(ref):
    for ex in SPEC["normalize"]:
        ap = ref.normalize(ex["a"], ex["L"])
        assert list(ap) == ex["ap"], ex["cite"]
        if "divisor_exp" in ex:
            assert ref.norm_exponent(ex["L"]) == ex["divisor_exp"]


def test_normalize_correctly_rounded_and_in_unit_interval(ref):
    rng = random.Random(11)
    for n in range(3, 24):
        pw = bytes(rng.getrandbits(8) for _ in range(n))
        a = ref.pack(pw)
        L = n // 3
        ap = ref.normalize(a, L)
        d = len(str(2 ** (8 * (L + 1))))
        for ai, v in zip(a, ap):
            # RN(RN(a)/10^d): a < 2^53 for L <= 6 so RN(a) = a and one rounding
            exact = Fraction(float(ai)) / 10 ** d
            assert v == float(exact)
            assert PAPER["a_prime_range"]["lo"] <= v <= PAPER["a_prime_range"]["hi"]


# ------------------------------------------------------------ lambda (Eq.5)
def test_lambda_in_paper_ranges_and_near_exact(ref):
    lo, hi = PAPER["lambda_ranges"]["lo"], PAPER["lambda_ranges"]["hi"]
    rng = random.Random(5)
    for _ in range(300):
        n = rng.randrange(3, 24)
        a = ref.pack(bytes(rng.getrandbits(8) for _ in range(n)))
        lam = ref.lam(a)
        for i in range(3):
            assert lo[i] < lam[i] < hi[i]
            msg = b"\x4c" + b"".join(x.to_bytes(8, "big") for x in a) + bytes([i + 1])
            h = int.from_bytes(hashlib.sha256(msg).digest()[:8], "big")
            exact = Fraction(lo[i]) + Fraction(h, 2 ** 64) * (Fraction(hi[i]) - Fraction(lo[i]))
            # three roundings of magnitude <= 64 each -> error well below 1e-13
            assert abs(Fraction(lam[i]) - exact) < Fraction(1, 10 ** 13)


def test_lambda_distinct_for_distinct_passwords(ref):
    rng = random.Random(9)
    seen = set()
    for _ in range(1000):
        a = ref.pack(bytes(rng.getrandbits(8) for _ in range(16)))
        seen.add(ref.lam(a))
    assert len(seen) == 1000


# ------------------------------------------------------------ mu
def test_mu_spec_examples(ref):
    for ex in SPEC["mu"]:
        assert list(ref.mu(ex["a"])) == ex["mu"], ex["cite"]


def test_mu_big_integer_brute_force(ref):
    rng = random.Random(3)
    for _ in range(2000):
        a = [rng.getrandbits(64) for _ in range(3)]
        want = [(a[0] + a[1] + a[2]) % 3, (a[0] * a[1] + a[2]) % 3, (a[0] + a[1] * a[2]) % 3]
        assert list(ref.mu(a)) == want


# ------------------------------------------------------------ k, Omega (Eq.7)
def test_k_omega_ranges_and_hash(ref):
    xi = PAPER["xi"]["value"]
    nu = math.floor(math.log10(2 ** (xi - 6)))
    kmax = (xi - 14) // 8
    rng = random.Random(4)
    for _ in range(500):
        n = rng.randrange(3, 24)
        pw = bytes(rng.getrandbits(8) for _ in range(n))
        a = ref.pack(pw)
        k, k3, om = ref.k_omega(pw, a)
        H = hashlib.sha256(pw).digest()
        for i in range(3):
            assert 2 < k[i] <= kmax
            assert k[i] == 3 + H[i] % 2                  # reading Q12
            msg = b"".join(((i + 1) * x % 2 ** 64).to_bytes(8, "big") for x in a)
            assert om[i] == int.from_bytes(hashlib.sha256(msg).digest()[:8], "big") % k[i]
        assert 0 < k3 < nu - 2 and k3 <= 6
        assert k3 == 1 + H[3] % 6


def test_nu_is_13():
    assert math.floor(math.log10(2 ** (PAPER["xi"]["value"] - 6))) == 13


# ------------------------------------------------------------ password normalisation / sub-keys
def test_normalize_password(ref):
    assert ref.normalize_password(b"abc") == b"abc"
    pw = b"0123456789abcdefghijklm"  # 23 bytes: kept
    assert ref.normalize_password(pw) == pw
    long = pw + b"n"
    assert ref.normalize_password(long) == hashlib.sha256(long).digest()[:18]
    with pytest.raises(ref.OracleError):
        ref.normalize_password(b"ab")


def test_subpassword(ref):
    rng = random.Random(2)
    for _ in range(100):
        pw = bytes(rng.getrandbits(8) for _ in range(rng.randrange(3, 100)))
        b = rng.getrandbits(32)
        assert ref.subpassword(pw, b) == hashlib.sha256(pw + b.to_bytes(4, "big")).digest()[:18]


def test_keymaterial_composition(ref):
    """r0 = a' + lambda (Eq.5); alpha0 = r0[mu] (Eq.6, n = 0); determinism."""
    km = ref.keymaterial(b"abc").as_dict()
    assert km["a"] == (97, 98, 99) and km["mu"] == (0, 2, 1)
    for i in range(3):
        assert km["r0"][i] == km["ap"][i] + km["lam"][i]
        assert km["alpha"][i] == km["r0"][km["mu"][i]]
    assert ref.keymaterial(b"abc").as_dict() == km
    # Fig.2's slightly different passwords give different key material
    k1, k2 = ref.keymaterial(b"123456").as_dict(), ref.keymaterial(b"123457").as_dict()
    assert k1["r0"] != k2["r0"]


def test_keymaterial_matches_independent_python(ref):
    import pyref
    rng = random.Random(21)
    for _ in range(300):
        n = rng.randrange(3, 24)
        pw = bytes(rng.getrandbits(8) for _ in range(n))
        km = ref.keymaterial(pw).as_dict()
        py = pyref.key_material(pw)
        assert list(km["a"]) == py["a"]
        assert list(km["ap"]) == py["ap"]
        assert list(km["r0"]) == py["r0"]
        assert list(km["mu"]) == py["mu"]
        assert list(km["k"]) == py["k"] and km["k3chain"] == py["k3c"]
        assert list(km["omega"]) == py["omega"]
