"""Pins for the oracle's SHA-256 (the hash of Eq.7; SHA-256 per reading Q11).

Pinned to FIPS 180-4 / NIST known-answer vectors (an external standard) and to
Python's hashlib (an independent library implementation) on random inputs.
"""
import hashlib
import random


KATS = [
    (b"", "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"),
    (b"abc", "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"),
    (b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq",
     "248d6a61d20638b8e5c026930c3e60 39a33ce45964ff2167f6ecedd419db06c1".replace(" ", "")),
    (b"abcdefghbcdefghicdefghijdefghijkefghijklfghijklmghijklmnhijklmnoijklmnopjklmnopqklmnopqrlmnopqrsmnopqrstnopqrstu",
     "cf5b16a778af8380036ce59e7b0492370b249b11e8f07a51afac45037afee9d1"),
]


def test_fips_kats(ref):
    for msg, hexd in KATS:
        assert ref.sha256(msg).hex() == hexd


def test_million_a(ref):
    assert ref.sha256(b"a" * 1_000_000).hex() == \
        "cdc76e5c9914fb9281a1c7e284d73e67f1809a48a497200e046d39ccc7112cd0"


def test_random_vs_hashlib(ref):
    rng = random.Random(1201)
    # every length across the one/two padding-block boundary, then random lengths
    lengths = list(range(0, 200)) + [rng.randrange(0, 5000) for _ in range(300)]
    for n in lengths:
        msg = bytes(rng.getrandbits(8) for _ in range(n))
        assert ref.sha256(msg) == hashlib.sha256(msg).digest(), n
