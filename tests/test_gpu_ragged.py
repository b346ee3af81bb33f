"""Ragged batches (serving): many FAST messages of different lengths and keys in one launch,
each byte equal to the oracle's single-message encryption; decrypt round trip; per-message
verdicts and zero-fill for tampered messages only; argument errors."""
import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def layout(lengths, key):
    """16-byte aligned back-to-back offsets for plaintexts and ciphertexts."""
    up = lambda x: (x + 15) // 16 * 16
    pt_off, ct_off, p, c = [], [], 0, 0
    for n in lengths:
        pt_off.append(p)
        ct_off.append(c)
        p += up(n)
        c += up(key.ct_len(n))
    return pt_off, ct_off, p, c


@pytest.mark.parametrize("count,seed", [(1, 1), (37, 2), (300, 3)])
def test_ragged_matches_oracle(count, seed):
    rng = np.random.default_rng(seed)
    lengths = [int(x) for x in rng.choice([0, 1, 15, 16, 1023, 1024, 1025, 3000, 5 * 1024 + 7], size=count)]
    pws = [inputs.password(seed=1000 * seed + s) for s in range(count)]
    keys = [L.lorenz_keysetup(pw, mode=L.FAST, n_it=6) for pw in pws]
    pt_off, ct_off, ptot, ctot = layout(lengths, keys[0])
    host_pt = np.zeros(max(ptot, 16), dtype=np.uint8)
    msgs = []
    for s, n in enumerate(lengths):
        m = inputs.message(n, seed=77 * seed + s)
        host_pt[pt_off[s]:pt_off[s] + n] = m
        msgs.append(m)
    pts = torch.from_numpy(host_pt).to(DEV)
    cts = torch.zeros(max(ctot, 16), dtype=torch.uint8, device=DEV)
    tags = torch.empty(16 * count, dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt_ragged(keys, lengths, pt_off, ct_off, pts, cts, tags)
    ct_h, tags_h = cts.cpu().numpy(), tags.cpu().numpy()
    prm = oracle.params(mode=oracle.FAST, n_it=6)
    for s, n in enumerate(lengths):
        want, want_tag = oracle.encrypt(pws[s], msgs[s], prm)
        assert np.array_equal(ct_h[ct_off[s]:ct_off[s] + len(want)], want), f"message {s} (n={n})"
        assert tags_h[16 * s:16 * s + 16].tobytes() == want_tag
    back = torch.zeros_like(pts)
    tags2 = torch.empty_like(tags)
    st, fb = L.lorenz_decrypt_ragged(keys, lengths, ct_off, pt_off, cts, back, tags2)
    assert st == L.OK and fb == [-1] * count
    assert torch.equal(back, pts) and torch.equal(tags2, tags)


def test_ragged_tamper_is_per_message():
    lengths = [4000, 1024, 0, 2500, 3000]
    pws = [inputs.password(seed=s) for s in range(len(lengths))]
    keys = [L.lorenz_keysetup(pw, mode=L.FAST, n_it=4) for pw in pws]
    pt_off, ct_off, ptot, ctot = layout(lengths, keys[0])
    pts = torch.from_numpy(inputs.message(ptot, seed=5)).to(DEV)
    cts = torch.zeros(ctot, dtype=torch.uint8, device=DEV)
    tags = torch.empty(16 * len(lengths), dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt_ragged(keys, lengths, pt_off, ct_off, pts, cts, tags)
    cts[ct_off[0] + 2 * 1040 + 9] ^= 1   # message 0, block 2
    cts[ct_off[3] + 1040 + 1050 - 1040] ^= 4  # message 3, block 1
    back = torch.full_like(pts, 0x5A)
    st, fb = L.lorenz_decrypt_ragged(keys, lengths, ct_off, pt_off, cts, back, torch.empty_like(tags))
    assert st == L.E_INTEGRITY and fb == [2, -1, -1, 1, -1]
    for s, n in enumerate(lengths):
        got = back[pt_off[s]:pt_off[s] + n]
        if fb[s] >= 0:
            assert not got.any()  # the whole failing message is withheld
        else:
            assert torch.equal(got, pts[pt_off[s]:pt_off[s] + n])


def test_ragged_argument_errors():
    keys = [L.lorenz_keysetup(b"abcdef", mode=L.FAST), L.lorenz_keysetup(b"ghijkl", mode=L.FAST, n_it=7)]
    buf = torch.zeros(1 << 16, dtype=torch.uint8, device=DEV)
    out = torch.zeros(1 << 16, dtype=torch.uint8, device=DEV)
    tags = torch.zeros(32, dtype=torch.uint8, device=DEV)
    with pytest.raises(L.LorenzError):  # different params
        L.lorenz_encrypt_ragged(keys, [10, 10], [0, 16], [0, 32], buf, out, tags)
    k2 = [keys[0], L.lorenz_keysetup(b"ghijkl", mode=L.FAST)]
    with pytest.raises(L.LorenzError):  # unaligned offset
        L.lorenz_encrypt_ragged(k2, [10, 10], [0, 8], [0, 32], buf, out, tags)
    with pytest.raises(L.LorenzError):  # overlapping outputs
        L.lorenz_encrypt_ragged(k2, [100, 100], [0, 112], [0, 16], buf, out, tags)
    with pytest.raises(L.LorenzError):  # STRONG keys are not batched
        s = [L.lorenz_keysetup(b"abcdef", mode=L.STRONG)] * 2
        L.lorenz_encrypt_ragged(s, [10, 10], [0, 16], [0, 32], buf, out, tags)
