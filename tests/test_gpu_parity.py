"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, byte for byte.

Integer outputs, tolerance 0 (north star). Configs C1-C5 of BASELINE.json:
full element-by-element parity where the oracle finishes in seconds, sampled blocks
(recomputed one by one by the oracle) plus size-independent properties at the full
C3/C4 sizes in the launch configuration bench.py times.
"""
import hashlib
import random

import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def oparams(key: L.Key):
    p = key.params
    return oracle.params(mode=p.mode, n_it=p.n_it, dt_code=p.dt_code, block_size=p.block_size,
                         integrator=p.integrator, variant=p.variant)


def gpu_encrypt(key, msg: np.ndarray):
    pt = torch.from_numpy(msg).to(DEV) if len(msg) else None
    n = len(msg)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    tag = L.lorenz_encrypt(key, n, 0, key.num_blocks(n), pt, ct)
    return ct, tag


def check_full(pw, msg, **kw):
    key = L.lorenz_keysetup(pw, **kw)
    ct, tag = gpu_encrypt(key, msg)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    got = ct.cpu().numpy()
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{len(bad)} ciphertext bytes differ, first at {bad[0]} (block {bad[0] // 1040})")
    assert tag == want_tag
    n = len(msg)
    nb = key.num_blocks(n)
    st, fb, vtag = L.lorenz_verify(key, n, 0, nb, ct)
    assert st == L.OK and fb == -1 and vtag == tag
    back = torch.empty(max(n, 1), dtype=torch.uint8, device=DEV)
    st, fb = L.lorenz_decrypt(key, n, 0, nb, ct, back if n else None)
    assert st == L.OK and fb == -1
    assert np.array_equal(back[:n].cpu().numpy(), msg)
    return key, ct, tag


# ------------------------------------------------------------------ C1
def test_c1_strong_3000_single_block():
    """C1: 1 KB random plaintext, 16-byte password, one block, the paper's n_it = 3000."""
    check_full(inputs.password(), inputs.message(1024), mode=L.STRONG, n_it=3000)


def test_c1_fast_single_block():
    check_full(inputs.password(), inputs.message(1024), mode=L.FAST)


# ------------------------------------------------------------------ C2
@pytest.mark.parametrize("B", [1024, 65536])
def test_c2_one_mib_round_trip(B):
    """C2: 1 MiB split into blocks, full parity (ciphertext, tag, plaintext)."""
    check_full(inputs.password(), inputs.message(1 << 20), mode=L.FAST, block_size=B)


def test_c2_tamper_detection():
    """C2: 100 random single-byte flips -> the flipped block is reported, other blocks intact."""
    pw = inputs.password()
    n = 1 << 20
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST)
    ct, _ = gpu_encrypt(key, msg)
    nb = key.num_blocks(n)
    ok = torch.empty(nb, dtype=torch.uint8, device=DEV)
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    rng = random.Random(1201)
    msg_t = torch.from_numpy(msg).to(DEV)
    for _ in range(100):
        pos = rng.randrange(ct.numel())
        bad = ct.clone()
        bad[pos] ^= rng.randrange(1, 256)
        st, fb = L.lorenz_decrypt(key, n, 0, nb, bad, back, block_ok=ok)
        blk = pos // 1040
        assert st == L.E_INTEGRITY and fb == blk
        okh = ok.cpu().numpy()
        assert okh[blk] == 0 and okh.sum() == nb - 1
        keep = torch.ones(n, dtype=torch.bool, device=DEV)
        keep[blk * 1024:(blk + 1) * 1024] = False
        assert torch.equal(back[keep], msg_t[keep])
        assert not back[blk * 1024:(blk + 1) * 1024].any()
        st, fb, _ = L.lorenz_verify(key, n, 0, nb, bad)
        assert st == L.E_INTEGRITY and fb == blk
    # without per-block verdicts the whole slice is zero-filled
    bad = ct.clone()
    bad[5] ^= 1
    st, fb = L.lorenz_decrypt(key, n, 0, nb, bad, back)
    assert st == L.E_INTEGRITY and fb == 0 and not back.any()


# ------------------------------------------------------------------ edge cases, full parity
@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 1008, 1023, 1024, 1025, 2048, 3000, 5 * 1024 + 77])
def test_edge_lengths_fast(n):
    check_full(inputs.password(seed=n + 1), inputs.message(n, seed=n), mode=L.FAST, n_it=7)


@pytest.mark.parametrize("n", [0, 1, 16, 100, 2000])
def test_edge_lengths_strong(n):
    check_full(inputs.password(seed=n + 7), inputs.message(n, seed=n + 3), mode=L.STRONG, n_it=11)


@pytest.mark.parametrize("pw_len", [3, 4, 5, 17, 23, 24, 51, 52, 55, 56, 59, 60, 63, 64, 65, 130])
@pytest.mark.parametrize("mode", [L.FAST, L.STRONG])
def test_password_lengths(pw_len, mode):
    """Every packing case of Eqs.2-4, the >23 hashing rule, and every SHA-256 padding
    layout of the FAST sub-password (1- and 2-block final blocks, midstate)."""
    pw = bytes(random.Random(pw_len).getrandbits(8) for _ in range(pw_len))
    check_full(pw, inputs.message(2100, seed=pw_len), mode=mode, n_it=5)


@pytest.mark.parametrize("dt_code", [0, 1, 2, 3])
@pytest.mark.parametrize("integrator", [L.RK4, L.EULER])
def test_dt_codes_and_integrators(dt_code, integrator):
    """All step sizes of the paper's range with RK4 and Euler. Forward Euler at
    h = 0.027 can leave the guard box (Q18): then both sides must report DIVERGENCE."""
    pw, msg = inputs.password(), inputs.message(3 * 1024 + 5, seed=dt_code)
    kw = dict(mode=L.FAST, n_it=13, dt_code=dt_code, integrator=integrator)
    key = L.lorenz_keysetup(pw, **kw)
    try:
        oracle.encrypt(pw, msg, oparams(key))
    except oracle.OracleError as e:
        assert e.status == oracle.E_DIVERGENCE and integrator == L.EULER
        with pytest.raises(L.LorenzError) as g:
            gpu_encrypt(key, msg)
        assert g.value.status == L.E_DIVERGENCE
        return
    check_full(pw, msg, **kw)


@pytest.mark.parametrize("n,mode,dt_code", [(0, L.FAST, 0), (5 * 1024 + 77, L.FAST, 0), (3000, L.FAST, 3),
                                            (2000, L.STRONG, 1), (40 * 1024, L.FAST, 2)])
def test_rk4_fma_variant(n, mode, dt_code):
    """NEXT-3: the FMA-formulated RK4 (__fma_rn at the oracle's fma() sites) is bit-exact."""
    check_full(inputs.password(seed=n), inputs.message(n, seed=n + 5), mode=mode, n_it=17, dt_code=dt_code,
               integrator=L.RK4_FMA)


@pytest.mark.parametrize("variant", [1, 2, 4, 5, 6])
@pytest.mark.parametrize("mode,n", [(L.FAST, 5 * 1024 + 77), (L.STRONG, 700)])
def test_step3_variants(variant, mode, n):
    """NEXT-4: the Step-3 reading variants are bit-exact against the pinned oracle."""
    check_full(inputs.password(seed=variant), inputs.message(n, seed=variant), mode=mode, n_it=23,
               variant=variant)


def test_step3_variant_full_size_sampled():
    pw = inputs.password()
    n = 128 << 20
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, variant=L.V_CYCLIC | L.V_DISTINCT_K)
    ct, tag = gpu_encrypt(key, msg)
    _sampled_parity(pw, msg, key, ct, tag, 24, seed=46)


def test_rk4_fma_full_size_sampled():
    pw = inputs.password()
    n = 256 << 20
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, integrator=L.RK4_FMA)
    ct, tag = gpu_encrypt(key, msg)
    _sampled_parity(pw, msg, key, ct, tag, 24, seed=45)


@pytest.mark.parametrize("B", [1040, 4096, 1 << 20])
def test_block_sizes(B):
    check_full(inputs.password(), inputs.message(3 * B // 2 + 3), mode=L.FAST, n_it=3, block_size=B)


def test_block_range_slices_and_tag_combine():
    """Any split of [0,nb) into slices reproduces the whole ciphertext; tags XOR-combine
    (the multi-GPU partition of DESIGN.md §5, emulated on one GPU)."""
    pw = inputs.password()
    n = 40 * 1024 + 300
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=9)
    whole, tag = gpu_encrypt(key, msg)
    nb = key.num_blocks(n)
    pt = torch.from_numpy(msg).to(DEV)
    for W in (2, 3, 7):
        ct = torch.zeros_like(whole)
        acc = bytes(16)
        for r in range(W):
            b0, b1 = nb * r // W, nb * (r + 1) // W
            t = L.lorenz_encrypt(key, n, b0, b1, pt[b0 * 1024:], ct[b0 * 1040:])
            acc = bytes(a ^ b for a, b in zip(acc, t))
        assert torch.equal(ct, whole) and acc == tag


def test_async_api_and_result_slot():
    pw = inputs.password()
    n = 9000
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=4)
    pt = torch.from_numpy(msg).to(DEV)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    res = torch.empty(32, dtype=torch.uint8, device=DEV)
    L.lorenz_result_init_async(res)
    L.lorenz_encrypt_async(key, n, 0, key.num_blocks(n), pt, ct, res)
    torch.cuda.synchronize()
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    assert np.array_equal(ct.cpu().numpy(), want)
    r = res.cpu().numpy()
    assert r[:16].tobytes() == want_tag
    assert int(r[16:24].view(np.uint64)[0]) == 2 ** 64 - 1 and int(r[24:28].view(np.uint32)[0]) == 0


def test_async_calls_capture_into_a_cuda_graph():
    """The _async calls enqueue only stream-ordered work (kernels; the balanced kernel adds a pool
    allocation and a memset), no synchronisation: a whole
    init -> encrypt -> init -> decrypt sequence is captured once and replayed."""
    pw = inputs.password()
    n = 6 * 1024 + 3
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=5)
    nb = key.num_blocks(n)
    pt = torch.from_numpy(msg).to(DEV)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    res = torch.empty(64, dtype=torch.uint8, device=DEV)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        L.lorenz_result_init_async(res[:32], stream=s)
        L.lorenz_encrypt_async(key, n, 0, nb, pt, ct, res[:32], stream=s)
        L.lorenz_result_init_async(res[32:], stream=s)
        L.lorenz_decrypt_async(key, n, 0, nb, ct, back, res[32:], stream=s)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    for _ in range(2):
        ct.zero_()
        back.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(ct.cpu().numpy(), want)
        r = res.cpu().numpy()
        assert r[:16].tobytes() == want_tag
        assert int(r[48:56].view(np.uint64)[0]) == 2 ** 64 - 1  # no failing block
        assert torch.equal(back, pt)


def test_host_buffer_end_to_end():
    pw = inputs.password()
    n = 50 * 1024 + 9
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=6)
    pt_h = torch.from_numpy(msg).pin_memory()
    ct_h = torch.empty(key.ct_len(n), dtype=torch.uint8).pin_memory()
    nb = key.num_blocks(n)
    tag = L.lorenz_encrypt_host(key, n, 0, nb, pt_h, ct_h, n_chunks=5)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    assert np.array_equal(ct_h.numpy(), want) and tag == want_tag
    back = np.zeros(n, dtype=np.uint8)
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, ct_h.numpy(), back, n_chunks=3)
    assert st == L.OK and fb == -1 and np.array_equal(back, msg)
    # a rank-style slice [7, 30) end to end
    sl = np.zeros(23 * 1040, dtype=np.uint8)
    t2 = L.lorenz_encrypt_host(key, n, 7, 30, msg[7 * 1024:], sl)
    assert np.array_equal(sl, want[7 * 1040:30 * 1040])
    bad = ct_h.numpy().copy()
    bad[20 * 1040 + 3] ^= 0x40
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, bad, back)
    assert st == L.E_INTEGRITY and fb == 20 and not back.any()


@pytest.mark.parametrize("chunks", [9, 17, 51])
def test_host_buffer_ring_reuse(chunks):
    """More chunks than the 8 device slots: chunk c reuses slot c % 8's buffers after chunk c-8's
    D2H (stream order). Ragged chunks (51 blocks into 17 / 9), last block partial."""
    pw = inputs.password()
    n = 50 * 1024 + 777
    msg = inputs.message(n, seed=11)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=5)
    nb = key.num_blocks(n)
    ct_h = np.zeros(key.ct_len(n), dtype=np.uint8)
    tag = L.lorenz_encrypt_host(key, n, 0, nb, msg, ct_h, n_chunks=chunks)
    want, want_tag = oracle.encrypt(pw, msg, oparams(key))
    assert np.array_equal(ct_h, want) and tag == want_tag
    back = np.zeros(n, dtype=np.uint8)
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, ct_h, back, n_chunks=chunks)
    assert st == L.OK and fb == -1 and np.array_equal(back, msg)
    bad = ct_h.copy()
    bad[47 * 1040 + 1039] ^= 1  # a tag byte of block 47: a late lap of the ring
    bad[44 * 1040 + 5] ^= 0x80
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, bad, back, n_chunks=chunks)
    assert st == L.E_INTEGRITY and fb == 44 and not back.any()


def test_argument_errors():
    key = L.lorenz_keysetup(b"password", mode=L.FAST)
    n = 4096
    pt = torch.zeros(n + 16, dtype=torch.uint8, device=DEV)
    ct = torch.zeros(key.ct_len(n) + 16, dtype=torch.uint8, device=DEV)
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_encrypt(key, n, 0, 5, pt, ct)  # b1 > nb
    assert e.value.status == L.E_ARG
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_encrypt(key, n, 0, 4, pt[1:], ct)  # misaligned
    assert e.value.status == L.E_ARG
    assert L.lorenz_encrypt(key, n, 2, 2, pt, ct) == bytes(16)  # empty range is a no-op


# ------------------------------------------------------------------ C3 / C4 at full size (sampled)
def _sampled_parity(pw, msg, key, ct, tag, n_samples, seed):
    n = len(msg)
    nb = key.num_blocks(n)
    rng = random.Random(seed)
    blocks = sorted({0, nb - 1, *(rng.randrange(nb) for _ in range(n_samples))})
    prm = oparams(key)
    B = key.block_size
    assert n % B == 0
    for b in blocks:
        want = oracle.encrypt_block(pw, n, b, msg[b * B:(b + 1) * B], prm)
        got = ct[b * (B + 16):(b + 1) * (B + 16)].cpu().numpy()
        assert np.array_equal(got, want), f"block {b}"
    # tag combine at any size: XOR of the per-block tags read from the ciphertext
    tags = ct.view(nb, B + 16)[:, B:].cpu().numpy()
    assert np.bitwise_xor.reduce(tags, axis=0).tobytes() == tag


@pytest.mark.parametrize("n_it", [100, 3000])
def test_c3_64mib(n_it):
    """C3: 64 MiB message on 1 B200 (bench launch configuration): sampled oracle parity,
    round trip and tag combine over the whole message."""
    pw = inputs.password()
    n = 64 << 20
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=n_it)
    ct, tag = gpu_encrypt(key, msg)
    _sampled_parity(pw, msg, key, ct, tag, 96 if n_it == 100 else 12, seed=n_it)
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    st, fb = L.lorenz_decrypt(key, n, 0, key.num_blocks(n), ct, back)
    assert st == L.OK and torch.equal(back, torch.from_numpy(msg).to(DEV))


def test_c4_1gib_single_gpu():
    """C4 on one GPU: 1 GiB, sampled oracle parity and rank-slice invariance (W = 8)."""
    pw = inputs.password()
    n = 1 << 30
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST)
    ct, tag = gpu_encrypt(key, msg)
    _sampled_parity(pw, msg, key, ct, tag, 64, seed=4)
    nb = key.num_blocks(n)
    # rank boundary blocks of W = 8 recomputed as separate slices must match
    pt = torch.from_numpy(msg).to(DEV)
    for r in range(1, 8):
        b = nb * r // 8
        part = torch.empty(2 * 1040, dtype=torch.uint8, device=DEV)
        L.lorenz_encrypt(key, n, b - 1, b + 1, pt[(b - 1) * 1024:], part)
        assert torch.equal(part, ct[(b - 1) * 1040:(b + 1) * 1040])


# ------------------------------------------------------------------ C5 batch
def test_c5_batch_parity():
    S, n = 12, 8 * 1024
    pws = [inputs.password(seed=inputs.SEED_PW ^ t) for t in range(S)]
    msgs = [inputs.message(n, seed=inputs.SEED_MSG ^ t) for t in range(S)]
    keys = [L.lorenz_keysetup(pw, mode=L.FAST, n_it=17) for pw in pws]
    pts = torch.from_numpy(np.concatenate(msgs)).to(DEV)
    ctl = keys[0].ct_len(n)
    cts = torch.empty(S * ctl, dtype=torch.uint8, device=DEV)
    tags = torch.empty(S * 16, dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt_batch(keys, n, pts, cts, tags)
    prm = oparams(keys[0])
    for s in range(S):
        want, wtag = oracle.encrypt(pws[s], msgs[s], prm)
        assert np.array_equal(cts[s * ctl:(s + 1) * ctl].cpu().numpy(), want), s
        assert tags[16 * s:16 * (s + 1)].cpu().numpy().tobytes() == wtag


def test_survey_fast_vector_on_gpu():
    """SURVEY Appendix B FAST vector (independent scratch computation) reproduced on the GPU."""
    key = L.lorenz_keysetup(b"0123456789abcdef", mode=L.FAST, n_it=100)
    ct, _ = gpu_encrypt(key, np.arange(0x28, dtype=np.uint8))
    assert ct.cpu().numpy().tobytes().hex() == (
        "874cec92922a173db8bfcfdbd67d663332cd926519e2e727a31a848d4d90bc77b779c3b5e39072eb848205f7d570d3c642503d2b05b153b1")
    assert hashlib.sha256(b"0123456789abcdef\0\0\0\0").digest()[:18].hex() == "3453b940792df16f962c01f9a3ddc38e1d9e"


@pytest.mark.parametrize("blocks", [50, 40000])
def test_host_direct_streaming(blocks):
    """Pinned (mapped) host buffers with n_chunks = 0 take the direct path: ONE chain launch reads the
    plaintext and writes the ciphertext over PCIe (lorenz.h). 50 blocks (wave kernel) and 40,000
    (balanced kernel, cut units); ragged last block; a rank-style slice of pinned views; decrypt round
    trip; a tampered block fails with its index and the whole host slice zero-filled. Against the
    oracle (sampled at 40,000 blocks) and against the staged pipeline on the same buffers."""
    pw = inputs.password(seed=blocks)
    n = blocks * 1024 - 999
    msg = inputs.message(n, seed=blocks)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=4)
    nb = key.num_blocks(n)
    pt_h = torch.from_numpy(msg).pin_memory()
    ct_h = torch.zeros(key.ct_len(n), dtype=torch.uint8).pin_memory()
    tag = L.lorenz_encrypt_host(key, n, 0, nb, pt_h, ct_h)
    staged = torch.zeros_like(ct_h)
    assert L.lorenz_encrypt_host(key, n, 0, nb, pt_h, staged, n_chunks=3) == tag
    assert torch.equal(ct_h, staged)
    prm = oparams(key)
    if blocks <= 1000:
        want, want_tag = oracle.encrypt(pw, msg, prm)
        assert np.array_equal(ct_h.numpy(), want) and tag == want_tag
    else:
        for b in (0, 1, 777, nb // 2, nb - 2, nb - 1):
            blk = msg[b * 1024:min(n, (b + 1) * 1024)]
            got = ct_h.numpy()[b * 1040:b * 1040 + len(blk) + 16]
            assert np.array_equal(got, oracle.encrypt_block(pw, n, b, blk, prm)), b
    back_h = torch.zeros(n, dtype=torch.uint8).pin_memory()
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, ct_h, back_h)
    assert st == L.OK and fb == -1 and torch.equal(back_h, pt_h)
    b0, b1 = 7, nb - 3  # pinned views at 16-byte aligned offsets
    sl = torch.zeros((b1 - b0) * 1040, dtype=torch.uint8).pin_memory()
    L.lorenz_encrypt_host(key, n, b0, b1, pt_h[b0 * 1024:], sl)
    assert torch.equal(sl, ct_h[b0 * 1040:b1 * 1040])
    bad = ct_h.clone().pin_memory()
    bad[(nb // 3) * 1040 + 5] ^= 0x10
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, bad, back_h)
    assert st == L.E_INTEGRITY and fb == nb // 3 and not back_h.any()


def test_device_calls_refuse_pageable_host_memory():
    """A pageable host buffer passed where a device pointer belongs is refused with E_ARG before any
    launch (it would fault inside the kernel and kill the context); mapped pinned host memory is
    device-accessible and works (the kernel reads it over PCIe), equal to the device result."""
    pw = inputs.password()
    n = 40 * 1024 + 48
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=3)
    nb = key.num_blocks(n)
    pageable = np.zeros(key.ct_len(n) + 64, dtype=np.uint8)
    pg = pageable.ctypes.data + (-pageable.ctypes.data % 16)  # 16-byte aligned, still pageable
    ct_d = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    pt_d = torch.from_numpy(msg).to(DEV)
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_encrypt(key, n, 0, nb, pt_d, pg)
    assert e.value.status == L.E_ARG
    with pytest.raises(L.LorenzError) as e:
        L.lorenz_verify(key, n, 0, nb, pg)
    assert e.value.status == L.E_ARG
    tag = L.lorenz_encrypt(key, n, 0, nb, pt_d, ct_d)  # the context survived
    pt_pin = torch.from_numpy(msg).pin_memory()
    ct_pin = torch.zeros(key.ct_len(n), dtype=torch.uint8).pin_memory()
    assert L.lorenz_encrypt(key, n, 0, nb, pt_pin, ct_pin) == tag
    assert torch.equal(ct_pin, ct_d.cpu())
