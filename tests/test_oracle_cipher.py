"""Pins for the oracle's quantiser, encode/decode and chain (Eqs.8-10, Steps 1-3)
and its message framing (§5).

Pinned to SPEC's worked examples, exhaustive inverse checks, the method's
invariants (round trip, tamper detection, pattern destruction, chain symmetry,
worker invariance, FAST-equals-STRONG special case), and bit-exact agreement
with an independently written pure-Python reading (tests/pyref.py).
"""
import hashlib
import json
import os
import random
import struct

import numpy as np
import pytest

import pyref

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
SURV = json.load(open(os.path.join(GOLD, "survey_vectors.json")))


# ------------------------------------------------------------ Eq.8 R_nu
def test_R_spec_examples(ref):
    for ex in SPEC["R"]:
        assert ref.R(ex["alpha"], ex["omega"]) == ex["R"], ex["cite"]


def test_R_is_byte_omega_of_floor_product(ref):
    """R = byte Omega of floor(|alpha| 1e13); the 16-byte remark of
    P:270 is garbled (Q7): |alpha| <= 100 keeps the integer below 2^53."""
    rng = random.Random(1)
    for _ in range(20000):
        a = rng.uniform(-100, 100)
        om = rng.randrange(0, 6)
        m = int(abs(a) * 1e13)  # Python float product is the same IEEE RN product
        assert m < 2 ** 53
        assert ref.R(a, om) == m.to_bytes(8, "little")[om]
        assert ref.R(a, om) == ref.R(-a, om)


def test_theta_spec_examples(ref):
    for ex in SPEC["perturb_theta"]:
        assert ref.theta(ex["p"], ex["omega3"]) == ex["theta"], ex["cite"]
    for p in range(256):
        for e in range(6):
            assert ref.theta(p, e) <= 0.255  # 0 <= m_i <= 0.255
            assert ref.theta(p, e) == p / 10 ** (3 + e)  # Python '/' of ints is correctly rounded


# ------------------------------------------------------------ Eqs.9-10
def test_encode_spec_examples(ref):
    for ex in SPEC["encode"]:
        assert ref.encode(ex["p"], ex["ksum"]) == ex["c"], ex["cite"]
        assert ref.decode(ex["c"], ex["ksum"]) == ex["p"], ex["cite"]


def test_encode_decode_inverse_exhaustive(ref):
    for ks in range(0, 511):
        cs = [ref.encode(p, ks) for p in range(256)]
        assert sorted(cs) == list(range(256))  # a bijection on bytes
        assert [ref.decode(c, ks) for c in cs] == list(range(256))


# ------------------------------------------------------------ the whole pipeline
def _P(mode, n_it, B=0, dt_code=0, integ=0):
    import oracle
    return oracle.params(mode=mode, n_it=n_it, block_size=B, dt_code=dt_code, integrator=integ)


def test_survey_cross_check_vectors(ref):
    s = (1.0, 1.0, 1.0)
    for n, want in SURV["rk4_from_111_h001"].items():
        got = ref.iterate(s, int(n))
        assert [struct.pack(">d", v).hex() for v in got] == want
    km = ref.keymaterial(b"abc").as_dict()
    assert [struct.pack(">d", v).hex() for v in km["ap"]] == SURV["key_abc"]["ap"]
    assert list(km["r0"]) == SURV["key_abc"]["r0"]
    assert list(km["omega"]) == SURV["key_abc"]["omega0"]
    assert [km["k"][0], km["k"][1], km["k3chain"]] == SURV["key_abc"]["k1_k2_k3chain"]
    c10 = ref.encrypt_stream(ref.keymaterial(b"abc"), b"Lorenz", _P(ref.STRONG, 10))
    assert c10.hex() == SURV["strong_abc_Lorenz"]["n_it_10"]
    ct, _ = ref.encrypt(b"abc", b"Lorenz", _P(ref.STRONG, 3000))
    assert ct.tobytes().hex() == SURV["strong_abc_Lorenz"]["n_it_3000"]
    v = SURV["fast_0123456789abcdef_block0"]
    assert ref.subpassword(b"0123456789abcdef", 0).hex() == v["subpassword"]
    ct, _ = ref.encrypt(b"0123456789abcdef", bytes.fromhex(v["pt_hex"]), _P(ref.FAST, v["n_it"]))
    assert ct.tobytes().hex() == v["ct_hex"]


@pytest.mark.parametrize("mode", ["strong", "fast"])
def test_matches_independent_python_reading(ref, mode):
    """Two independently written CPU readings agree bit for bit (SURVEY c.3 last row)."""
    rng = random.Random(77)
    fast = mode == "fast"
    for trial in range(12):
        pw = bytes(rng.getrandbits(8) for _ in range(rng.randrange(3, 30)))
        n = rng.randrange(0, 65)
        pt = bytes(rng.getrandbits(8) for _ in range(n))
        n_it = rng.choice([1, 7, 20])
        dt_code = rng.randrange(4)
        prm = _P(ref.FAST if fast else ref.STRONG, n_it, dt_code=dt_code)
        ct, _ = ref.encrypt(pw, pt, prm)
        want = pyref.encrypt_message(pw, pt, fast, n_it, dt_code=dt_code)
        assert ct.tobytes() == want, (trial, pw, n, n_it)
        st, back, fb = ref.decrypt(pw, ct, prm)
        assert st == ref.OK and back.tobytes() == pt


def test_matches_python_reading_multiblock_and_euler(ref):
    rng = random.Random(78)
    pw = b"multi-block-pw"
    pt = bytes(rng.getrandbits(8) for _ in range(1024 + 40))
    ct, _ = ref.encrypt(pw, pt, _P(ref.FAST, 3))
    assert ct.tobytes() == pyref.encrypt_message(pw, pt, True, 3)
    ct, _ = ref.encrypt(pw, pt[:50], _P(ref.STRONG, 9, integ=ref.EULER))
    assert ct.tobytes() == pyref.run_stream(pyref.key_material(pw), pt[:50], 9, integrator="euler")


def test_round_trip_random(ref):
    """D(E(P)) = P (SPEC acceptance #1): 1000 messages of length 0..4096."""
    rng = random.Random(1000)
    for t in range(1000):
        fast = t % 2 == 0
        n_it = 200 if t % 10 == 0 else 20
        n = rng.randrange(0, 4097)
        pt = rng.randbytes(n)
        pw = rng.randbytes(rng.randrange(3, 40))
        prm = _P(ref.FAST if fast else ref.STRONG, n_it)
        ct, _ = ref.encrypt(pw, pt, prm, threads=1)
        assert len(ct) == ref.ct_len(prm, n)
        st, back, fb = ref.decrypt(pw, ct, prm, threads=1)
        assert st == ref.OK and fb == -1 and back.tobytes() == pt


def test_length_contract(ref):
    for ex in SPEC["lengths"]:
        prm = _P(ref.FAST if ex["mode"] == "fast" else ref.STRONG, 5, B=ex.get("B", 0))
        assert ref.ct_len(prm, ex["n"]) == ex["ct_len"], ex["cite"]
        assert ref.pt_len(prm, ex["ct_len"]) == ex["n"]
    for ex in SPEC["plan_chunks"]:
        assert ref.num_blocks(_P(ref.FAST, 5, B=ex["B"]), ex["n"]) == ex["blocks"], ex["cite"]
    prm = _P(ref.FAST, 5)
    for n in [0, 1, 15, 16, 1023, 1024, 1025, 4096, 5000]:
        assert ref.pt_len(prm, ref.ct_len(prm, n)) == n
    for bad in [0, 15, 1041, 1040 + 16]:
        with pytest.raises(ref.OracleError):
            ref.pt_len(prm, bad)
    ct, _ = ref.encrypt(b"pw0", b"", prm)
    assert len(ct) == 16


def test_tamper_detection_two_blocks(ref):
    """a changed C_i changes the trajectory; 100 single-byte flips are all
    caught with the right block index, >= 95% of later bytes garble, the other block
    decrypts intact (SPEC acceptance #6)."""
    rng = random.Random(6)
    pw = b"tamper-test-pw"
    prm = _P(ref.FAST, 20)
    pt = rng.randbytes(2048)
    ct, _ = ref.encrypt(pw, pt, prm)
    garbled = []
    for _ in range(100):
        pos = rng.randrange(len(ct))
        bad = ct.copy()
        bad[pos] ^= rng.randrange(1, 256)
        st, back, fb, ok = ref.decrypt(pw, bad, prm, per_block=True)
        blk = pos // 1040
        assert st == ref.E_INTEGRITY and fb == blk
        assert list(ok) == [int(b != blk) for b in range(2)]
        other = 1 - blk
        assert back.tobytes()[other * 1024:(other + 1) * 1024] == pt[other * 1024:(other + 1) * 1024]
        assert not back[blk * 1024:(blk + 1) * 1024].any()  # failing block zero-filled
        # garbling: decrypt the tampered block without the zero-fill
        km = ref.keymaterial(ref.subpassword(pw, blk))
        rec, good = ref.decrypt_stream(km, bad[blk * 1040:(blk + 1) * 1040].tobytes(), prm)
        off = pos - blk * 1040
        if off + 1 < 1024:
            post = np.frombuffer(rec[off + 1:], np.uint8)
            orig = np.frombuffer(pt[blk * 1024 + off + 1:(blk + 1) * 1024], np.uint8)
            garbled.append(float(np.mean(post != orig)))
        # whole-range zero-fill without per-block verdicts
        st2, back2, fb2 = ref.decrypt(pw, bad, prm)
        assert st2 == ref.E_INTEGRITY and fb2 == blk and not back2.any()
    assert np.mean(garbled) >= 0.95


def test_wrong_password_rejected(ref):
    rng = random.Random(12)
    prm = _P(ref.STRONG, 20)
    pt = rng.randbytes(64)
    ct, _ = ref.encrypt(b"the-right-one", pt, prm)
    for _ in range(100):
        wrong = rng.randbytes(rng.randrange(3, 24))
        st, back, fb = ref.decrypt(wrong, ct, prm)
        assert st == ref.E_INTEGRITY and fb == 0 and not back.any()


def test_pattern_destruction(ref):
    """P:120 / P:145: similar plaintext blocks give different ciphertext (SPEC #7)."""
    blk = random.Random(3).randbytes(64)
    ct, _ = ref.encrypt(b"pattern-pw", blk * 16, _P(ref.STRONG, 20))
    chunks = {ct[i * 64:(i + 1) * 64].tobytes() for i in range(16)}
    assert len(chunks) == 16


def test_chain_symmetry(ref):
    """Encrypt-side and decrypt-side chains stay bit-identical."""
    km = ref.keymaterial(b"symmetry")
    pt = random.Random(4).randbytes(10_000)
    prm = _P(ref.STRONG, 3)
    ct, tr_e = ref.encrypt_stream(km, pt, prm, trace=True)
    back, ok, tr_d = ref.decrypt_stream(km, ct, prm, trace=True)
    assert ok and back == pt
    assert np.array_equal(tr_e.view(np.uint64), tr_d.view(np.uint64))


def test_thread_invariance_and_ranges(ref):
    """Worker-count invariance and block-range slicing."""
    rng = random.Random(5)
    pt = rng.randbytes(10 * 1024 + 77)
    prm = _P(ref.FAST, 10)
    c1, t1 = ref.encrypt(b"invariance", pt, prm, threads=1)
    c8, t8 = ref.encrypt(b"invariance", pt, prm, threads=8)
    assert np.array_equal(c1, c8) and t1 == t8
    # slices [0,4) ∪ [4,11) reproduce the whole; tags XOR together
    ca, ta = ref.encrypt(b"invariance", pt, prm, b0=0, b1=4)
    cb, tb = ref.encrypt(b"invariance", pt, prm, b0=4, b1=11)
    assert np.array_equal(ca[:4 * 1040], c1[:4 * 1040]) and np.array_equal(cb[4 * 1040:], c1[4 * 1040:])
    assert bytes(x ^ y for x, y in zip(ta, tb)) == t1
    tags = [c1[b * 1040 + min(1024, len(pt) - b * 1024): b * 1040 + min(1024, len(pt) - b * 1024) + 16]
            for b in range(11)]
    x = np.bitwise_xor.reduce(np.stack(tags), axis=0)
    assert x.tobytes() == t1


def test_encrypt_block_equals_message_slice(ref):
    """encrypt_block (used for sampled GPU parity at full size) reproduces the block's slice
    of the whole-message ciphertext, including the ragged last block."""
    rng = random.Random(15)
    pt = rng.randbytes(5 * 1024 + 300)
    prm = _P(ref.FAST, 12)
    whole, _ = ref.encrypt(b"block-pw", pt, prm)
    for b in range(6):
        blk = np.frombuffer(pt[b * 1024:(b + 1) * 1024], np.uint8)
        got = ref.encrypt_block(b"block-pw", len(pt), b, blk, prm)
        assert np.array_equal(got, whole[b * 1040: b * 1040 + len(blk) + 16])


def test_fast_single_block_equals_strong_under_subkey(ref):
    """a single-block FAST message equals STRONG encryption under the block-0
    sub-password with the FAST n_it."""
    pw = b"special-case"
    pt = random.Random(9).randbytes(700)
    cf, _ = ref.encrypt(pw, pt, _P(ref.FAST, 100))
    sub = ref.subpassword(pw, 0)
    cs, _ = ref.encrypt(sub, pt, _P(ref.STRONG, 100))
    assert np.array_equal(cf, cs)
    assert sub == hashlib.sha256(pw + b"\0\0\0\0").digest()[:18]


def test_lock_in_characterisation(ref):
    """Property of Step 3 as printed (P:320-323 under reading Q13): once
    (mu1,Omega1) = (mu2,Omega2) with k1 = k2 the two keystream terms coincide, so the
    keystream is even and ciphertext LSB = plaintext LSB; never when k1 != k2."""
    pw = b"lock-in-study"
    prm = _P(ref.FAST, 100)
    nb = 48
    pt = np.frombuffer(random.Random(10).randbytes(nb * 1024), np.uint8)
    ct, _ = ref.encrypt(pw, pt, prm)
    locked = 0
    for b in range(nb):
        body = ct[b * 1040: b * 1040 + 1024]
        same_lsb = ((body ^ pt[b * 1024:(b + 1) * 1024]) & 1) == 0
        km = ref.keymaterial(ref.subpassword(pw, b)).as_dict()
        if same_lsb[256:].all():
            locked += 1
            assert km["k"][0] == km["k"][1]
        if km["k"][0] != km["k"][1]:
            assert not same_lsb[256:].all()
    assert 0.1 <= locked / nb <= 0.6


def test_guard_reports_divergence(ref):
    """Reading Q18: the guard is a status. Forward Euler at the paper's largest step
    (h = 0.027) is unstable and leaves the box; RK4 at the same step does not."""
    from paper_1201_3114_b200 import inputs
    pw, msg = inputs.password(), inputs.message(3 * 1024 + 5, seed=3)
    with pytest.raises(ref.OracleError) as e:
        ref.encrypt(pw, msg, _P(ref.FAST, 13, dt_code=3, integ=ref.EULER))
    assert e.value.status == ref.E_DIVERGENCE
    ref.encrypt(pw, msg, _P(ref.FAST, 13, dt_code=3, integ=ref.RK4))


def test_strong_long_password_is_hashed(ref):
    long_pw = b"x" * 40
    pt = b"hello world"
    prm = _P(ref.STRONG, 10)
    ct, _ = ref.encrypt(long_pw, pt, prm)
    ct2, _ = ref.encrypt(hashlib.sha256(long_pw).digest()[:18], pt, prm)
    assert np.array_equal(ct, ct2)
    with pytest.raises(ref.OracleError):
        ref.encrypt(b"ab", pt, prm)
