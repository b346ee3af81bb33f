"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol that
include/lorenz.h declares, and its host-only helpers (key setup, length arithmetic,
argument validation) behave as documented. No compute call is made here.
"""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lorenz.h")


@pytest.fixture(scope="module")
def L():
    from paper_1201_3114_b200 import build, lorenz
    build.build()
    lorenz.lib()
    return lorenz


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lorenz_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 17
    so = C.CDLL(L.LIB_PATH)
    for s in syms:
        assert hasattr(so, s), s
    assert set(L.EXPORTS) == set(syms)
    assert L.lib().lorenz_abi_version() == 2


def test_keysetup_deterministic_and_validated(L):
    a = L.lorenz_keysetup(b"password123", mode=L.FAST)
    b = L.lorenz_keysetup(b"password123", mode=L.FAST)
    assert bytes(a.raw.opaque) == bytes(b.raw.opaque)
    p = a.params
    assert (p.mode, p.n_it, p.dt_code, p.block_size, p.integrator) == (L.FAST, 100, 0, 1024, L.RK4)
    s = L.lorenz_keysetup(b"password123", mode=L.STRONG)
    assert s.params.n_it == 3000
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_keysetup(b"ab")
    assert e.value.status == L.E_PASSWORD
    for bad in (dict(block_size=1000), dict(block_size=1032), dict(dt_code=4), dict(integrator=3),
                dict(mode=2)):
        with pytest.raises(L.LorenzError) as e:
            L.lorenz_keysetup(b"password", **bad)
        assert e.value.status == L.E_ARG


def test_length_arithmetic_matches_oracle(L, ref):
    for mode in (L.FAST, L.STRONG):
        for B in (1024, 2048):
            k = L.lorenz_keysetup(b"pw-lengths", mode=mode, block_size=B)
            prm = ref.params(mode=mode, block_size=B)
            for n in [0, 1, 15, 1023, 1024, 1025, 2047, 2048, 2049, 10 ** 6, 1 << 30]:
                assert k.num_blocks(n) == ref.num_blocks(prm, n)
                assert k.ct_len(n) == ref.ct_len(prm, n)
                assert L.lorenz_pt_len(k, k.ct_len(n)) == n
            for bad in [0, 15]:
                with pytest.raises(L.LorenzError) as e:
                    L.lorenz_pt_len(k, bad)
                assert e.value.status == L.E_LENGTH
    k = L.lorenz_keysetup(b"pw-lengths", mode=L.FAST)
    with pytest.raises(L.LorenzError):
        L.lorenz_pt_len(k, 1041)


def test_device_calls_reject_bad_ranges_before_launch(L):
    """Argument errors are returned before any launch (works without a GPU)."""
    k = L.lorenz_keysetup(b"password", mode=L.FAST)
    tag = (C.c_uint8 * 16)()
    lib = L.lib()
    # b1 > nb
    assert lib.lorenz_encrypt(C.byref(k.raw), 4096, 0, 9, 16, 4096 + 16 * 64, tag, None) == L.E_ARG
    # misaligned pointer
    assert lib.lorenz_encrypt(C.byref(k.raw), 4096, 0, 4, 17, 1 << 20, tag, None) == L.E_ARG
    # overlapping buffers
    assert lib.lorenz_encrypt(C.byref(k.raw), 4096, 0, 4, 1 << 20, (1 << 20) + 1024, tag, None) == L.E_ARG
    # invalid key
    bad = L.lorenz_key()
    assert lib.lorenz_encrypt(C.byref(bad), 4096, 0, 4, 16, 1 << 20, tag, None) == L.E_ARG
    # empty range: a no-op that succeeds without touching the device
    assert lib.lorenz_encrypt(C.byref(k.raw), 4096, 2, 2, 16, 1 << 20, tag, None) == L.OK
    # maximum size: block indices are BE32 in the sub-key (Q16), so nb > 2^32 is refused
    huge = (1 << 32) * 1024 + 1
    assert k.num_blocks(huge) == (1 << 32) + 1
    assert lib.lorenz_encrypt(C.byref(k.raw), huge, 0, 1, 16, 1 << 40, tag, None) == L.E_ARG


def test_product_never_imports_oracle():
    """The product package shares no code with the oracle and never imports it."""
    pkg = os.path.join(ROOT, "paper_1201_3114_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "lorenz_ref" not in txt, f


def test_launch_plan_rules(L, tune):
    """Host-side schedule choice, computed without a device (148 SMs): the
    balanced kernel for 2+ warps per SM sub-partition and under three waves unless the wave
    kernel's single wave splits evenly; the wave kernel otherwise; overrides honoured."""
    tune()
    key = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST)
    plan = lambda blocks: L.lorenz_launch_plan(key, blocks * 1024, 0, blocks)
    p = plan(65536)  # C3: 2,048 units, 3.46 warps per sub-partition in one wave
    assert p["kind"] == "balanced" and p["cta"] == 384 and p["grid"] == 148 and p["slots"] == 1776
    # skewed: 3 warp groups per CTA, the slots of group g hold 74 + g chunks (mean 75 = ceil(2048 x 65 / 1776))
    assert p["chunks_per_slot"] == 74 and p["chunks_skew"] == 1
    assert plan(131072)["kind"] == "balanced" and plan(131072)["cta"] == 512  # C4 per rank at N = 8
    assert plan(1 << 20)["kind"] == "balanced"       # C4 at N = 1 (RK4: every size from 2 warps/SMSP)
    assert plan(262144)["kind"] == "balanced"        # C4 per rank at N = 4
    eul = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST, integrator=L.EULER)
    assert L.lorenz_launch_plan(eul, 1 << 30, 0, 1 << 20)["kind"] == "wave"  # Euler: wave from 3 waves
    assert plan(75776)["kind"] == "wave"             # exactly 4 warps per sub-partition
    assert plan(37888)["kind"] == "wave"             # exactly 2 warps per sub-partition
    assert plan(1024)["kind"] == "wave" and plan(1024)["grid"] * plan(1024)["cta"] >= 1024  # C2
    assert L.lorenz_launch_plan(key, 0, 0, 1)["lanes"] == 1
    fma = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST, integrator=L.RK4_FMA)
    assert L.lorenz_launch_plan(fma, 65536 * 1024, 0, 65536)["kind"] == "balanced"
    for blocks, kind in ((131072, "balanced"), (262144, "balanced"), (524288, "wave"), (1 << 20, "wave")):
        assert L.lorenz_launch_plan(fma, blocks * 1024, 0, blocks)["kind"] == kind, blocks  # 3 x 20 warps/SM
    tune(schedule="wave")
    assert plan(65536)["kind"] == "wave"
    tune(schedule="seg", seg_slots=3)
    p = plan(160)
    assert p["kind"] == "balanced" and p["slots"] == 3 and p["chunks_per_slot"] == 109 and p["chunks_skew"] == 0
    with pytest.raises(L.LorenzError):
        L.lorenz_launch_plan(key, 1024, 0, 2)


def test_launch_plan_mcnaughton_invariants(L, tune):
    """For every balanced plan: slots <= units (else a slot would hold less than one unit),
    every slot holds >= Q = (B+16)/16 chunks (a cut unit's two pieces then never overlap in time;
    skewed plans keep Q/8 more), the slots cover the U * Q chunk line without a spare slot's worth,
    and the grid holds every slot."""
    tune()
    import random
    rng = random.Random(5)
    for B in (1024, 2048, 65536):
        key = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST, block_size=B)
        q = (B + 16 + 15) // 16
        sizes = [rng.randrange(1, 400_000) for _ in range(200)] + [37888, 37889, 65536, 75776, 113664, 113665]
        for blocks in sizes:
            n = blocks * B - rng.randrange(0, B)
            nb = key.num_blocks(n)
            b0 = rng.randrange(0, nb) if rng.random() < 0.3 else 0
            p = L.lorenz_launch_plan(key, n, b0, nb)
            assert p["lanes"] == nb - b0
            if p["kind"] == "wave":
                assert p["grid"] * p["cta"] >= p["lanes"]
                continue
            units = -(-p["lanes"] // 32)
            assert 2 * 592 <= p["slots"] <= units
            assert p["grid"] == 148 and p["cta"] * p["grid"] // 32 >= p["slots"]
            wpc = p["cta"] // 32
            caps = ([p["chunks_per_slot"] + (w // 4) * p["chunks_skew"] for w in range(wpc)] * p["grid"])[:p["slots"]]
            if p["chunks_skew"]:
                assert p["slots"] == wpc * p["grid"]
                assert p["chunks_per_slot"] >= q + q // 8  # slack: the pieces of a cut unit never meet
            assert min(caps) >= q
            assert sum(caps) >= units * q > sum(caps) - len(caps) - p["grid"] * wpc * p["chunks_skew"]


def test_set_tuning_validated(L):
    """lorenz_set_tuning (the library reads no environment variables): out-of-range fields are
    rejected and change nothing; NULL restores the defaults."""
    key = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST)
    default = L.lorenz_launch_plan(key, 65536 * 1024, 0, 65536)
    for bad in (dict(schedule=3), dict(cta=100), dict(seg_skew=-2), dict(seg_skew=1001)):
        with pytest.raises(L.LorenzError) as e:
            L.lorenz_set_tuning(**bad)
        assert e.value.status == L.E_ARG
    assert L.lorenz_launch_plan(key, 65536 * 1024, 0, 65536) == default
    with L.tuning(schedule=L.SCHED_WAVE, cta=512):
        p = L.lorenz_launch_plan(key, 65536 * 1024, 0, 65536)
        assert p["kind"] == "wave" and p["cta"] == 512
    assert L.lorenz_launch_plan(key, 65536 * 1024, 0, 65536) == default


def test_async_result_and_batch_tags_alignment(L):
    """The kernels update `res` and the batch tags with 64-bit atomics: a pointer that is not
    16-byte aligned is an argument error, reported before anything is enqueued (no device here)."""
    key = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST)
    lib, kp = L.lib(), C.byref(key.raw)
    pt, ct = 0x7F0000000000, 0x7F0010000000
    for res in (0x7F0020000008, 0x7F0020000001):
        assert lib.lorenz_encrypt_async(kp, 4096, 0, 4, pt, ct, res, None) == L.E_ARG
        assert lib.lorenz_decrypt_async(kp, 4096, 0, 4, ct, pt, None, res, None) == L.E_ARG
        assert lib.lorenz_verify_async(kp, 4096, 0, 4, ct, res, None) == L.E_ARG
        assert lib.lorenz_result_init_async(res, None) == L.E_ARG
    keys = (L.lorenz_key * 2)(key.raw, key.raw)
    assert lib.lorenz_encrypt_batch(keys, 2, 4096, pt, ct, 0x7F0020000008, None) == L.E_ARG


def test_ragged_overlap_not_hidden_by_an_empty_message(L):
    """Decrypt outputs A = [0, 4096), B = [16, 16) (a zero-length message), C = [1024, 2048):
    A and C overlap; the empty range sorted between them must not hide it."""
    import numpy as np
    key = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST)
    keys = (L.lorenz_key * 3)(key.raw, key.raw, key.raw)
    n = np.array([4096, 0, 1024], dtype=np.uint64)
    ct_off = np.array([0, 8192, 12288], dtype=np.uint64)
    pt_off = np.array([0, 16, 1024], dtype=np.uint64)
    fb = np.zeros(3, dtype=np.int64)
    st = L.lib().lorenz_decrypt_ragged(keys, 3, n.ctypes.data, ct_off.ctypes.data, pt_off.ctypes.data,
                                       0x7F0000000000, 0x7F0010000000, 0x7F0020000000, fb.ctypes.data, None)
    assert st == L.E_ARG
    assert b"overlap" in L.lib().lorenz_last_error()
