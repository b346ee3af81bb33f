"""GPU parity past 32-bit offsets: a 4.5 GiB + ragged message (4.7 M blocks, ciphertext offsets
beyond 2^32), so every byte / block index on the device path must be 64-bit.

Blocks around the 2^32 plaintext and ciphertext offsets and the ragged last block are recomputed
one by one by the oracle (`encrypt_block`); the rest is checked by properties that hold at any
size: the tag equals the XOR of the per-block tags read back from the ciphertext, decrypt
inverts encrypt, and a flipped byte past 4 GiB is reported in the right block.
The message bytes come from torch's generator (plumbing, not the path under test); n_it = 2
keeps the launch to a fraction of a second.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
B = 1024


def test_message_beyond_4gib():
    n = (9 << 29) + 123  # 4.5 GiB + 123 bytes
    free, _ = torch.cuda.mem_get_info()
    if free < 3 * n + (1 << 30):
        pytest.skip("needs ~14 GB of free device memory")
    pw = inputs.password(seed=44)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=2)
    nb = key.num_blocks(n)
    assert nb == (n + B - 1) // B
    g = torch.Generator(device=DEV)
    g.manual_seed(20120114)
    pt = torch.randint(0, 256, (n,), dtype=torch.uint8, device=DEV, generator=g)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    tag = L.lorenz_encrypt(key, n, 0, nb, pt, ct)

    prm = oracle.params(mode=oracle.FAST, n_it=2, block_size=B)
    b_pt32 = (1 << 32) // B                      # first block at plaintext offset 2^32
    b_ct32 = (1 << 32) // (B + 16)               # the block whose ciphertext crosses 2^32
    for b in sorted({0, b_ct32 - 1, b_ct32, b_ct32 + 1, b_pt32 - 1, b_pt32, b_pt32 + 1, nb - 2, nb - 1}):
        lo = b * B
        blk = pt[lo:min(n, lo + B)].cpu().numpy()
        want = oracle.encrypt_block(pw, n, b, blk, prm)
        got = ct[b * (B + 16):b * (B + 16) + len(blk) + 16].cpu().numpy()
        assert np.array_equal(got, want), f"block {b}"

    # tag = XOR of every block's last 16 ciphertext bytes (full blocks + the ragged last one)
    full = ct[:(nb - 1) * (B + 16)].view(nb - 1, B + 16)[:, B:]
    x = full.contiguous().view(torch.int64).view(nb - 1, 2)
    acc = torch.zeros(2, dtype=torch.int64, device=DEV)
    for col in range(2):
        v = x[:, col]
        while v.numel() > 1:  # pairwise XOR reduction on the device
            if v.numel() % 2:
                v = torch.cat([v, torch.zeros(1, dtype=torch.int64, device=DEV)])
            v = torch.bitwise_xor(v[0::2], v[1::2])
        acc[col] = v[0]
    last = ct[-16:].cpu().numpy().view(np.int64)
    want_tag = (acc.cpu().numpy() ^ last).view(np.uint8).tobytes()
    assert tag == want_tag

    back = torch.empty_like(pt)
    st, fb = L.lorenz_decrypt(key, n, 0, nb, ct, back)
    assert st == L.OK and fb == -1
    assert torch.equal(back, pt)
    del back
    bad_b = b_pt32 + 7
    ct[bad_b * (B + 16) + 100] ^= 0x20
    st, fb, _ = L.lorenz_verify(key, n, 0, nb, ct)
    assert st == L.E_INTEGRITY and fb == bad_b


def test_host_api_bounded_device_memory():
    """lorenz_encrypt_host / lorenz_decrypt_host on a 6 GiB + ragged HOST message: host offsets
    past 2^32, and the device footprint stays at the 8-slot chunk ring (~2 GB), not the slice size
    (the ring is what lets messages larger than HBM stream through)."""
    n = (3 << 31) + 77  # 6 GiB + 77 bytes
    pw = inputs.password(seed=45)
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=2)
    nb = key.num_blocks(n)
    rng = np.random.default_rng(7)
    pt = rng.integers(0, 256, n, dtype=np.uint8)
    ct = np.empty(key.ct_len(n), dtype=np.uint8)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    tag = L.lorenz_encrypt_host(key, n, 0, nb, pt, ct)
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < (3 << 30), f"device footprint {(free0 - free1) / 2**30:.2f} GiB"  # pool keeps the ring cached
    prm = oracle.params(mode=oracle.FAST, n_it=2, block_size=B)
    b32 = (1 << 32) // (B + 16)
    for b in (0, b32 - 1, b32, b32 + 1, (1 << 32) // B, nb - 1):
        lo = b * B
        blk = pt[lo:min(n, lo + B)]
        want = oracle.encrypt_block(pw, n, b, blk, prm)
        assert np.array_equal(ct[b * (B + 16):b * (B + 16) + len(blk) + 16], want), f"block {b}"
    tags = ct[:(nb - 1) * (B + 16)].reshape(nb - 1, B + 16)[:, B:]
    want_tag = np.bitwise_xor.reduce(tags, axis=0) ^ ct[-16:]
    assert tag == want_tag.tobytes()
    back = np.empty(n, dtype=np.uint8)
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, ct, back)
    assert st == L.OK and fb == -1 and np.array_equal(back, pt)
