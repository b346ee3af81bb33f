"""Oracle parity at the stated sizes of BASELINE.json's configs, in the launch configuration
bench.py times (SURVEY.md §8(d) parity column; north star "bit-exact vs the CPU oracle on all
five configs"). Byte-for-byte, tolerance 0:

  C3  64 MiB, n_it = 100:  the whole message (encrypt, tag, GPU decrypt of the ORACLE's
                           ciphertext, verify), default launch plan (balanced kernel);
  C3  64 MiB, n_it = 3000: 4,096 random blocks + the first and last, recomputed one by one;
  C4  1 GiB, n_it = 100:   the whole message in the bench's single-GPU launch (the skewed
                           balanced plan), decrypt of the oracle's ciphertext, and every
                           rank's slice of the N = 2 / 4 / 8 partitions launched on its own
                           (the per-rank plans of the driver's scaling runs);
  C5  the bench's batch (128 trials x 3 x 1 MiB streams, one lorenz_encrypt_batch launch via
      sweep.Batch): 16 trials spread over the launch, all three streams and tags each.

The oracle runs on every host core (oracle/lorenz_ref.c, static block partition); C4 costs
about 3.5 minutes of the 16-core box's time.
"""
import json
import os
import random
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import dist as D
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L
from paper_1201_3114_b200 import sweep

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
B = 1024


def oparams(key: L.Key):
    p = key.params
    return oracle.params(mode=p.mode, n_it=p.n_it, dt_code=p.dt_code, block_size=p.block_size,
                         integrator=p.integrator, variant=p.variant)


def first_diff(got: np.ndarray, want: np.ndarray) -> str:
    bad = np.nonzero(got != want)[0]
    return f"{len(bad)} bytes differ, first at {bad[0]} (block {bad[0] // (B + 16)})"


def full_message_parity(n: int, n_it: int):
    """Whole-message encrypt against the oracle, then the GPU decrypts and verifies the
    oracle's own ciphertext. Returns (key, msg, ciphertext, tag)."""
    pw = inputs.password()
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=n_it, block_size=B)
    nb = key.num_blocks(n)
    plan = L.lorenz_launch_plan(key, n, 0, nb)
    assert plan["kind"] == "balanced"  # the bench launch at these sizes
    pt = torch.from_numpy(msg).to(DEV)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    tag = L.lorenz_encrypt(key, n, 0, nb, pt, ct)
    got = ct.cpu().numpy()
    want, want_tag = oracle.encrypt(pw, msg, oparams(key), threads=0)
    assert np.array_equal(got, want), first_diff(got, want)
    assert tag == want_tag
    # decrypt / verify of the oracle's ciphertext (independent of the GPU encrypt)
    ct_o = torch.from_numpy(want).to(DEV)
    back = torch.empty(n, dtype=torch.uint8, device=DEV)
    st, fb = L.lorenz_decrypt(key, n, 0, nb, ct_o, back)
    assert st == L.OK and fb == -1
    assert torch.equal(back, pt)
    st, fb, vtag = L.lorenz_verify(key, n, 0, nb, ct_o)
    assert st == L.OK and fb == -1 and vtag == want_tag
    return key, pw, msg, want, want_tag


def test_c3_full_message_n100():
    full_message_parity(64 << 20, 100)


def test_c3_n3000_4096_blocks():
    """C3 at the paper's n_it = 3000: 4,096 random blocks + first and last, one by one."""
    n, n_it = 64 << 20, 3000
    pw = inputs.password()
    msg = inputs.message(n)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=n_it, block_size=B)
    nb = key.num_blocks(n)
    assert L.lorenz_launch_plan(key, n, 0, nb)["kind"] == "balanced"
    pt = torch.from_numpy(msg).to(DEV)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt(key, n, 0, nb, pt, ct)
    got = ct.cpu().numpy().reshape(nb, B + 16)
    rng = random.Random(3000)
    blocks = sorted({0, nb - 1} | set(rng.sample(range(nb), 4096)))
    assert len(blocks) >= 4096
    prm = oparams(key)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:  # ctypes releases the GIL
        wants = list(ex.map(lambda b: oracle.encrypt_block(pw, n, b, msg[b * B:(b + 1) * B], prm), blocks))
    for b, want in zip(blocks, wants):
        assert np.array_equal(got[b], want), f"block {b}"


def test_c4_full_message_and_rank_slices():
    n = 1 << 30
    key, pw, msg, want, want_tag = full_message_parity(n, 100)
    nb = key.num_blocks(n)
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_tags.json")))
    assert want_tag.hex() == golden["c4/n_it=100/rk4"]  # what bench.py checks at every rank count
    pt = torch.from_numpy(msg).to(DEV)
    wv = want.reshape(nb, B + 16)
    # the driver's scaling runs: each rank launches its own slice (its own balanced plan)
    for world in (2, 4, 8):
        tags = []
        for r in range(world):
            b0, b1 = D.block_range(nb, r, world)
            sl = D.slice_of(n, B, b0, b1)
            ct = torch.empty(sl.ct_bytes, dtype=torch.uint8, device=DEV)
            tags.append(L.lorenz_encrypt(key, n, b0, b1, pt[sl.pt_off:sl.pt_off + sl.pt_bytes], ct))
            got = ct.cpu().numpy().reshape(b1 - b0, B + 16)
            assert np.array_equal(got, wv[b0:b1]), (world, r, first_diff(got.ravel(), wv[b0:b1].ravel()))
        comb = bytes(np.bitwise_xor.reduce(np.frombuffer(b"".join(tags), dtype=np.uint8).reshape(world, 16)))
        assert comb == want_tag, world
    # tamper at full size in the bench's launch: the lowest failing block is reported, the plaintext
    # is zero-filled, verify agrees; blocks at both ends of slots and in the middle of units
    ct_o = torch.from_numpy(want).to(DEV)
    rng = random.Random(44)
    for flips in ([nb - 1], [rng.randrange(nb) for _ in range(3)], [0, nb // 2]):
        bad = ct_o.clone()
        for b in flips:
            bad[b * (B + 16) + rng.randrange(B + 16)] ^= 1 << rng.randrange(8)
        back = torch.ones(n, dtype=torch.uint8, device=DEV)
        st, fb = L.lorenz_decrypt(key, n, 0, nb, bad, back)
        assert st == L.E_INTEGRITY and fb == min(flips) and not back.any(), (flips, st, fb)
        st, fb, _ = L.lorenz_verify(key, n, 0, nb, bad)
        assert st == L.E_INTEGRITY and fb == min(flips)


def test_c5_bench_batch_16_trials():
    """The bench's C5 step (sweep.Batch of 128 trials, one batched launch) against the oracle on
    16 trials spread over the launch: base, password-flip and plaintext-flip streams and tags."""
    n, T, n_it = 1 << 20, 128, 100
    bt = sweep.Batch(0, T, n, n_it, B, DEV)
    lanes = 3 * T * (n // B)
    assert L.lorenz_launch_plan(bt.keys[0], lanes * B, 0, lanes)["kind"] == "balanced"
    bt.encrypt()
    cts = bt.cts.cpu().numpy()
    tags = bt.tags.cpu().numpy()
    prm = oparams(bt.keys[0])
    ctl = bt.ctl
    for i in range(0, T, T // 16):
        pw, pwf, msg, msgf, _ = sweep.trial_inputs(i, n)
        for k, (p, m) in enumerate([(pw, msg), (pwf, msg), (pw, msgf)]):
            want, wtag = oracle.encrypt(p, m, prm, threads=0)
            got = cts[(3 * i + k) * ctl:(3 * i + k + 1) * ctl]
            assert np.array_equal(got, want), (i, k, first_diff(got, want))
            assert tags[16 * (3 * i + k):16 * (3 * i + k + 1)].tobytes() == wtag, (i, k)
