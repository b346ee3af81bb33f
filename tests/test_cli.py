"""The `lorenz` command (NEXT-2; SPEC cli S:510-548): usage / exit codes on CPU, and the
encrypt -> decrypt round trip against the oracle's envelope bytes on the GPU."""
import json
import os
import subprocess

import pytest


@pytest.fixture(scope="module")
def cli():
    from paper_1201_3114_b200 import build
    build.build()
    return build.CLI


def run(cli, *args, env=None, pw=None):
    e = dict(os.environ)
    e.pop("LZX_PASSWORD", None)
    if pw is not None:
        e["LZX_PASSWORD"] = pw
    return subprocess.run([cli, *args], capture_output=True, text=True, env=e)


def test_usage_and_exit_codes(cli, tmp_path):
    assert run(cli).returncode == 2
    assert run(cli, "frobnicate", "a", "b").returncode == 2
    assert run(cli, "encrypt", "a", "b", "--mode", "medium").returncode == 2
    src = tmp_path / "x.bin"
    src.write_bytes(b"hello")
    r = run(cli, "encrypt", str(src), str(tmp_path / "y.lzx"))
    assert r.returncode == 2 and "password" in r.stderr  # no password given
    assert run(cli, "info", str(tmp_path / "missing.lzx")).returncode == 3


def test_info_prints_the_header(cli, tmp_path):
    from paper_1201_3114_b200 import lorenz as L
    key = L.lorenz_keysetup(b"abcdef", mode=L.FAST, n_it=77, block_size=2048)
    f = tmp_path / "h.lzx"
    f.write_bytes(L.lorenz_envelope_write(key, 5000))
    r = run(cli, "info", str(f))
    assert r.returncode == 0
    d = json.loads(r.stdout)
    assert d == {"mode": "fast", "n_it": 77, "dt_code": 0, "block_size": 2048, "integrator": 0, "variant": 0,
                 "payload_len": 5000, "ciphertext_len": 5000 + 16 * 3}
    f.write_bytes(b"NOPE" + bytes(20))
    assert run(cli, "info", str(f)).returncode == 3


@pytest.mark.gpu
def test_cli_round_trip_matches_oracle(cli, tmp_path):
    import oracle
    from oracle import envelope
    from paper_1201_3114_b200 import inputs
    data = inputs.message(70 * 1024 + 3)
    src, enc, dec = tmp_path / "in.bin", tmp_path / "out.lzx", tmp_path / "back.bin"
    src.write_bytes(data.tobytes())
    pwf = tmp_path / "pw.txt"
    pwf.write_bytes(b"cli-password\n")
    r = run(cli, "encrypt", str(src), str(enc), "--nit", "9", "--password-file", str(pwf), "--stream-bytes", "16384")
    assert r.returncode == 0, r.stderr
    assert enc.read_bytes() == envelope.encrypt_file_bytes(b"cli-password", data, oracle.params(n_it=9))
    r = run(cli, "decrypt", str(enc), str(dec), pw="cli-password")
    assert r.returncode == 0 and dec.read_bytes() == data.tobytes()
    bad = bytearray(enc.read_bytes())
    bad[24 + 5 * 1040 + 9] ^= 1
    (tmp_path / "bad.lzx").write_bytes(bytes(bad))
    r = run(cli, "decrypt", str(tmp_path / "bad.lzx"), str(tmp_path / "bad.out"), pw="cli-password")
    assert r.returncode == 1 and "block 5" in r.stderr and not (tmp_path / "bad.out").exists()
    r = run(cli, "encrypt", str(src), str(tmp_path / "s.lzx"), "--mode", "strong", "--nit", "3", pw="ab")
    assert r.returncode == 1  # password shorter than 3 bytes
