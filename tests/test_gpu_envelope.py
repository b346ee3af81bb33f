"""NEXT-2 on the GPU: the streaming file path (envelope + chunked H2D/kernel/D2H pipeline)
against the oracle's envelope bytes, byte for byte, plus round trip, tamper and truncation."""
import os

import numpy as np
import pytest

import oracle
from oracle import envelope
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu


def _write(path, data):
    with open(path, "wb") as f:
        f.write(bytes(data))


@pytest.mark.parametrize("n,chunk,mode,n_it", [
    (0, 0, L.FAST, 9), (1, 0, L.FAST, 9), (50 * 1024 + 7, 4096, L.FAST, 9), (50 * 1024 + 7, 0, L.FAST, 9),
    (3 * 1024, 1024, L.FAST, 9), (777, 0, L.STRONG, 15), (0, 0, L.STRONG, 15)])
def test_file_round_trip_matches_oracle(tmp_path, n, chunk, mode, n_it):
    pw = inputs.password()
    data = inputs.message(n, seed=n + 11)
    src, enc, dec = tmp_path / "in.bin", tmp_path / "out.lzx", tmp_path / "back.bin"
    _write(src, data)
    tag = L.lorenz_encrypt_file(str(src), str(enc), pw, mode=mode, n_it=n_it, chunk_bytes=chunk)
    want = envelope.encrypt_file_bytes(pw, data, oracle.params(mode=mode, n_it=n_it))
    got = enc.read_bytes()
    assert got == want
    _, want_tag = oracle.encrypt(pw, data, oracle.params(mode=mode, n_it=n_it))
    assert tag == want_tag
    st, fb = L.lorenz_decrypt_file(str(enc), str(dec), pw, chunk_bytes=chunk)
    assert st == L.OK and fb == -1
    assert dec.read_bytes() == data.tobytes()
    assert not os.path.exists(str(enc) + ".partial") and not os.path.exists(str(dec) + ".partial")


def test_file_tamper_wrong_password_truncation(tmp_path):
    pw = inputs.password()
    n = 20 * 1024 + 100
    data = inputs.message(n)
    src, enc, dec = tmp_path / "in.bin", tmp_path / "out.lzx", tmp_path / "back.bin"
    _write(src, data)
    L.lorenz_encrypt_file(str(src), str(enc), pw, n_it=7, chunk_bytes=3 * 1024)
    blob = bytearray(enc.read_bytes())
    bad = bytearray(blob)
    pos = 24 + 13 * 1040 + 500
    bad[pos] ^= 0x10
    _write(tmp_path / "bad.lzx", bad)
    st, fb = L.lorenz_decrypt_file(str(tmp_path / "bad.lzx"), str(dec), pw, chunk_bytes=3 * 1024)
    assert st == L.E_INTEGRITY and fb == 13
    assert not dec.exists() and not os.path.exists(str(dec) + ".partial")  # nothing released
    st, fb = L.lorenz_decrypt_file(str(enc), str(dec), b"not-the-password")
    assert st == L.E_INTEGRITY and fb == 0 and not dec.exists()
    _write(tmp_path / "short.lzx", blob[:-1])
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_decrypt_file(str(tmp_path / "short.lzx"), str(dec), pw)
    assert e.value.status == L.E_LENGTH
    _write(tmp_path / "magic.lzx", b"XXXX" + bytes(blob[4:]))
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_decrypt_file(str(tmp_path / "magic.lzx"), str(dec), pw)
    assert e.value.status == L.E_FORMAT
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_encrypt_file(str(tmp_path / "missing.bin"), str(enc), pw)
    assert e.value.status == L.E_IO


def test_file_large_multichunk_sampled(tmp_path):
    """A 96 MiB file in 32 MiB chunks (three chunks in flight): sampled oracle parity."""
    pw = inputs.password()
    n = 96 << 20
    data = inputs.message(n)
    src, enc, dec = tmp_path / "in.bin", tmp_path / "out.lzx", tmp_path / "back.bin"
    data.tofile(src)
    tag = L.lorenz_encrypt_file(str(src), str(enc), pw, chunk_bytes=32 << 20)
    ct = np.fromfile(enc, dtype=np.uint8)
    assert ct.size == 24 + n + 16 * (n // 1024)
    prm = oracle.params(mode=oracle.FAST, n_it=100)
    for b in [0, 1, 32767, 32768, 65535, 65536, 98303]:
        want = oracle.encrypt_block(pw, n, b, data[b * 1024:(b + 1) * 1024], prm)
        assert np.array_equal(ct[24 + b * 1040: 24 + (b + 1) * 1040], want), b
    tags = ct[24:].reshape(-1, 1040)[:, 1024:]
    assert np.bitwise_xor.reduce(tags, axis=0).tobytes() == tag
    st, fb = L.lorenz_decrypt_file(str(enc), str(dec), pw, chunk_bytes=32 << 20)
    assert st == L.OK and np.array_equal(np.fromfile(dec, dtype=np.uint8), data)
