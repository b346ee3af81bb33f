"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Exercises every kernel of liblorenz.so on small, ragged inputs: encrypt / verify / decrypt
(FAST ragged multi-block, STRONG, all integrators), tamper path with and without per-block
verdicts, the batch launch, the statistics kernels and the host-buffer pipeline.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    pw = inputs.password()
    for integ in (L.RK4, L.EULER, L.RK4_FMA):
        for mode, n in ((L.FAST, 5 * 1024 + 77), (L.FAST, 0), (L.STRONG, 300)):
            key = L.lorenz_keysetup(pw, mode=mode, n_it=3, integrator=integ)
            msg = inputs.message(n)
            pt = torch.from_numpy(msg).to(dev) if n else torch.empty(16, dtype=torch.uint8, device=dev)
            ct, tag = L.encrypt(key, pt[:n])
            st, fb, vt = L.lorenz_verify(key, n, 0, key.num_blocks(n), ct)
            assert st == L.OK and vt == tag
            back, st, fb = L.decrypt(key, ct)
            assert st == L.OK and torch.equal(back, pt[:n])
    key = L.lorenz_keysetup(pw, mode=L.FAST, n_it=3)
    n = 4 * 1024 + 5
    msg = torch.from_numpy(inputs.message(n)).to(dev)
    ct, tag = L.encrypt(key, msg)
    ct[1040 + 3] ^= 1
    ok = torch.empty(key.num_blocks(n), dtype=torch.uint8, device=dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    st, fb = L.lorenz_decrypt(key, n, 0, key.num_blocks(n), ct, out, block_ok=ok)
    assert st == L.E_INTEGRITY and fb == 1
    st, fb = L.lorenz_decrypt(key, n, 0, key.num_blocks(n), ct, out)
    assert st == L.E_INTEGRITY and not out.any()
    # batch + statistics
    S, m = 5, 3 * 1024
    keys = [L.lorenz_keysetup(inputs.password(seed=s), mode=L.FAST, n_it=3) for s in range(S)]
    pts = torch.from_numpy(np.concatenate([inputs.message(m, seed=s) for s in range(S)])).to(dev)
    ctl = keys[0].ct_len(m)
    cts = torch.empty(S * ctl, dtype=torch.uint8, device=dev)
    tags = torch.empty(S * 16, dtype=torch.uint8, device=dev)
    L.lorenz_encrypt_batch(keys, m, pts, cts, tags)
    outc = torch.empty(3 * 2, dtype=torch.int64, device=dev)
    L.lorenz_compare_spans(cts, cts, [(0, ctl, ctl), (5, ctl + 7, 100)], outc)
    hist = torch.empty(256 * 2, dtype=torch.int64, device=dev)
    L.lorenz_histograms(cts, [(0, 0, ctl), (3, 0, 1000)], hist)
    torch.cuda.synchronize()
    assert int(hist[:256].sum()) == ctl
    # host pipeline
    h_pt = torch.from_numpy(inputs.message(9 * 1024 + 1)).pin_memory()
    k2 = L.lorenz_keysetup(pw, mode=L.FAST, n_it=2)
    h_ct = torch.empty(k2.ct_len(h_pt.numel()), dtype=torch.uint8).pin_memory()
    L.lorenz_encrypt_host(k2, h_pt.numel(), 0, k2.num_blocks(h_pt.numel()), h_pt, h_ct, n_chunks=4)
    print("sanitize case ok")


if __name__ == "__main__":
    main()
