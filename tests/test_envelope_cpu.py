"""Envelope header (NEXT-2): the C-ABI's host-only header functions
against the oracle's struct-packed header and SPEC's worked framing examples. No GPU."""
import random

import pytest


@pytest.fixture(scope="module")
def L():
    from paper_1201_3114_b200 import build, lorenz
    build.build()
    lorenz.lib()
    return lorenz


def test_header_matches_oracle(L, ref):
    from oracle import envelope
    rng = random.Random(24)
    for _ in range(200):
        mode = rng.choice([L.FAST, L.STRONG])
        kw = dict(mode=mode, n_it=rng.choice([0, 1, 100, 3000, 77]), dt_code=rng.randrange(4),
                  block_size=rng.choice([0, 1024, 1040, 65536]), integrator=rng.randrange(3),
                  variant=rng.choice([0, 0, 1, 2, 4, 5, 6]))
        key = L.lorenz_keysetup(b"envelope-pw", **kw)
        n = rng.choice([0, 5, 1024, 10 ** 6, 1 << 33])
        hdr = L.lorenz_envelope_write(key, n)
        assert hdr == envelope.header(ref.params(**kw), n)
        p, n2, ctl = L.lorenz_envelope_read(hdr)
        eff = key.params
        assert (p.mode, p.n_it, p.dt_code, p.block_size, p.integrator, p.variant) == \
            (eff.mode, eff.n_it, eff.dt_code, eff.block_size, eff.integrator, eff.variant)
        if kw["integrator"] == 0 and kw["variant"] == 0:
            assert hdr[6] == 0  # SPEC's reserved flags byte for the default cipher
        assert n2 == n and ctl == key.ct_len(n)
        assert envelope.parse(hdr)["n"] == n


def test_spec_framing_examples(L):
    # strong mode, 5-byte plaintext -> file length 24 + 5 + 16 = 45
    k = L.lorenz_keysetup(b"abc", mode=L.STRONG)
    assert L.ENVELOPE_BYTES + k.ct_len(5) == 45
    # fast mode, 100 KiB, 64 KiB chunks -> body = 100*1024 + 32
    k = L.lorenz_keysetup(b"abc", mode=L.FAST, block_size=65536)
    assert k.ct_len(100 * 1024) == 100 * 1024 + 32
    _, _, ctl = L.lorenz_envelope_read(L.lorenz_envelope_write(k, 100 * 1024))
    assert ctl == 100 * 1024 + 32


def test_header_errors(L):
    k = L.lorenz_keysetup(b"abcdef", mode=L.FAST)
    good = L.lorenz_envelope_write(k, 1000)
    cases = [(b"LZX2" + good[4:], L.E_FORMAT), (good[:4] + b"\x02" + good[5:], L.E_FORMAT),
             (good[:5] + b"\x02" + good[6:], L.E_FORMAT), (good[:6] + b"\x07" + good[7:], L.E_FORMAT),
             (good[:7] + b"\x04" + good[8:], L.E_FORMAT), (good[:23], L.E_LENGTH),
             (good[:12] + (1000).to_bytes(4, "little") + good[16:], L.E_FORMAT)]
    for hdr, st in cases:
        with pytest.raises(L.LorenzError) as e:
            L.lorenz_envelope_read(hdr)
        assert e.value.status == st


def test_untrusted_payload_length_does_not_wrap(L):
    """A header whose payload length would make the file exceed 2^64 bytes is malformed
    (E_FORMAT), not a wrapped ciphertext length."""
    import struct
    key = L.lorenz_keysetup(b"envelope-pw", mode=L.FAST)
    hdr = bytearray(L.lorenz_envelope_write(key, 5))
    for bad in (2 ** 64 - 16, 2 ** 64 - 1, 2 ** 64 - 24 - 16 * (2 ** 64 // 1040)):
        hdr[16:24] = struct.pack("<Q", bad)
        with pytest.raises(L.LorenzError) as e:
            L.lorenz_envelope_read(bytes(hdr))
        assert e.value.status == L.E_FORMAT
    # the largest representable payload is still accepted
    big = (2 ** 64 - 1 - 24) // 1040 * 1024
    hdr[16:24] = struct.pack("<Q", big)
    p, n, ctl = L.lorenz_envelope_read(bytes(hdr))
    assert n == big and ctl == big + 16 * (big // 1024)
    sk = L.lorenz_keysetup(b"envelope-pw", mode=L.STRONG)
    hdr = bytearray(L.lorenz_envelope_write(sk, 5))
    hdr[16:24] = struct.pack("<Q", 2 ** 64 - 40)
    with pytest.raises(L.LorenzError):
        L.lorenz_envelope_read(bytes(hdr))
