"""Randomised GPU-vs-oracle parity over the whole parameter space (300 seeded configurations):
mode, message length, password length, n_it, dt code, integrator, Step-3 variant, block
size, and a random block range. Integer outputs, tolerance 0."""
import random

import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _config(rng):
    mode = rng.choice([L.FAST, L.FAST, L.STRONG])
    B = rng.choice([1024, 1040, 1024 + 16 * rng.randrange(1, 200)])
    n = rng.choice([0, rng.randrange(1, 64), rng.randrange(64, 6000), B * rng.randrange(1, 4)])
    if mode == L.STRONG:
        n = min(n, 900)
    integ = rng.choice([L.RK4, L.RK4, L.EULER, L.RK4_FMA])
    dt = rng.randrange(3) if integ == L.EULER else rng.randrange(4)  # Euler at h = 0.027 may diverge
    return dict(mode=mode, n_it=rng.randrange(1, 25), dt_code=dt, block_size=B, integrator=integ,
                variant=rng.choice([0, 0, 1, 2, 4, 5, 6])), n


@pytest.mark.parametrize("seed", range(6))
def test_random_configurations(seed):
    rng = random.Random(9000 + seed)
    for _ in range(50):
        kw, n = _config(rng)
        pw = rng.randbytes(rng.randrange(3, 90))
        msg = np.frombuffer(rng.randbytes(n), np.uint8) if n else np.zeros(0, np.uint8)
        key = L.lorenz_keysetup(pw, **kw)
        p = key.params
        prm = oracle.params(mode=p.mode, n_it=p.n_it, dt_code=p.dt_code, block_size=p.block_size,
                            integrator=p.integrator, variant=p.variant)
        want, _ = oracle.encrypt(pw, msg, prm)
        nb = key.num_blocks(n)
        b0 = rng.randrange(nb)
        b1 = rng.randrange(b0, nb) + 1
        B = p.block_size if p.mode == L.FAST else n
        lo, hi = (b0 * B, min(n, b1 * B)) if p.mode == L.FAST else (0, n)
        pt = torch.from_numpy(msg[lo:hi].copy()).to(DEV) if hi > lo else None
        ct = torch.empty(hi - lo + 16 * (b1 - b0), dtype=torch.uint8, device=DEV)
        tag = L.lorenz_encrypt(key, n, b0, b1, pt, ct)
        clo = lo + 16 * b0
        got = ct.cpu().numpy()
        assert np.array_equal(got, want[clo:clo + got.size]), (kw, n, b0, b1)
        tags = [want[min(n, (b + 1) * B) + 16 * b: min(n, (b + 1) * B) + 16 * b + 16] if p.mode == L.FAST
                else want[n:n + 16] for b in range(b0, b1)]
        assert np.bitwise_xor.reduce(np.stack(tags), axis=0).tobytes() == tag
        back = torch.empty(max(hi - lo, 1), dtype=torch.uint8, device=DEV)
        st, fb = L.lorenz_decrypt(key, n, b0, b1, ct, back if hi > lo else None)
        assert st == L.OK and fb == -1
        if hi > lo:
            assert np.array_equal(back[:hi - lo].cpu().numpy(), msg[lo:hi])


@pytest.mark.parametrize("seed", range(3))
def test_random_configurations_balanced_kernel(seed, tune):
    """The same parity through the balanced kernel, forced onto a random number of warp slots
    (so units are cut at random chunk positions): FAST messages of 33-420 blocks, random block
    sizes, block ranges, integrators, step sizes and Step-3 variants."""
    tune(schedule="seg")
    rng = random.Random(7000 + seed)
    for _ in range(25):
        B = rng.choice([1024, 1040, 1024 + 16 * rng.randrange(1, 64)])
        blocks = rng.randrange(33, 420)
        n = blocks * B - rng.choice([0, 0, rng.randrange(1, B)])
        integ = rng.choice([L.RK4, L.RK4, L.EULER, L.RK4_FMA])
        kw = dict(mode=L.FAST, n_it=rng.randrange(1, 9), dt_code=rng.randrange(3) if integ == L.EULER
                  else rng.randrange(4), block_size=B, integrator=integ, variant=rng.choice([0, 0, 1, 2, 4, 5]))
        pw = rng.randbytes(rng.randrange(3, 40))
        msg = np.frombuffer(rng.randbytes(n), np.uint8)
        key = L.lorenz_keysetup(pw, **kw)
        nb = key.num_blocks(n)
        b0 = rng.choice([0, rng.randrange(nb // 2)])
        b1 = nb if rng.random() < 0.5 else rng.randrange(b0 + 1, nb + 1)
        units = -(-(b1 - b0) // 32)
        tune(seg_slots=rng.randrange(1, units + 1))
        p = key.params
        prm = oracle.params(mode=p.mode, n_it=p.n_it, dt_code=p.dt_code, block_size=p.block_size,
                            integrator=p.integrator, variant=p.variant)
        want, _ = oracle.encrypt(pw, msg, prm, b0=b0, b1=b1)
        lo, hi = b0 * B, min(n, b1 * B)
        pt = torch.from_numpy(msg[lo:hi].copy()).to(DEV)
        ct = torch.empty(hi - lo + 16 * (b1 - b0), dtype=torch.uint8, device=DEV)
        assert L.lorenz_launch_plan(key, n, b0, b1)["kind"] == "balanced"
        tag = L.lorenz_encrypt(key, n, b0, b1, pt, ct)
        clo = lo + 16 * b0
        got = ct.cpu().numpy()
        assert np.array_equal(got, want[clo:clo + got.size]), (kw, n, b0, b1)
        tags = [want[min(n, (b + 1) * B) + 16 * b: min(n, (b + 1) * B) + 16 * b + 16] for b in range(b0, b1)]
        assert np.bitwise_xor.reduce(np.stack(tags), axis=0).tobytes() == tag
        back = torch.empty(hi - lo, dtype=torch.uint8, device=DEV)
        st, fb = L.lorenz_decrypt(key, n, b0, b1, ct, back)
        assert st == L.OK and fb == -1
        assert np.array_equal(back.cpu().numpy(), msg[lo:hi])
