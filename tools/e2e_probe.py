"""End-to-end cost of the host-buffer API against the device-only kernel time (1 GPU).

For each message size: the device call (lorenz_encrypt on resident tensors, CUDA events), the
host-buffer call in its automatic mode (direct streaming over PCIe from mapped pinned memory)
and in the staged copy pipeline (n_chunks > 0), encrypt and decrypt; every output is checked
against the device ciphertext / the plaintext.

Usage: python tools/e2e_probe.py [--mib 64 128 1024] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def wall(fn, reps):
    fn()  # warm: pool, streams, host path
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return sum(ts) / len(ts) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, nargs="+", default=[64, 128, 1024])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--staged-chunks", type=int, nargs="+", default=[4])
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    key = L.lorenz_keysetup(inputs.password(), mode=L.FAST)
    for mib in a.mib:
        n = mib << 20
        nb = key.num_blocks(n)
        msg = inputs.message(n)
        pt_d = torch.from_numpy(msg).to(dev)
        ct_d = torch.empty(key.ct_len(n), dtype=torch.uint8, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        L.lorenz_encrypt(key, n, 0, nb, pt_d, ct_d)
        dev_ms = []
        for _ in range(a.reps):
            e0.record()
            L.lorenz_encrypt(key, n, 0, nb, pt_d, ct_d)
            e1.record()
            torch.cuda.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
        dms = sum(dev_ms) / len(dev_ms)
        pt_h = torch.from_numpy(msg).pin_memory()
        ct_h = torch.empty(key.ct_len(n), dtype=torch.uint8).pin_memory()
        back_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        row = {"mib": mib, "device_ms": round(dms, 3)}
        for label, chunks in [("direct", 0)] + [(f"staged{c}", c) for c in a.staged_chunks]:
            ct_h.zero_()
            ms = wall(lambda: L.lorenz_encrypt_host(key, n, 0, nb, pt_h, ct_h, n_chunks=chunks), a.reps)
            ok = bool(torch.equal(ct_h.to(dev), ct_d))
            back_h.zero_()
            dms_dec = wall(lambda: L.lorenz_decrypt_host(key, n, 0, nb, ct_h, back_h, n_chunks=chunks), a.reps)
            ok_dec = bool(torch.equal(back_h, pt_h))
            row[label] = {"enc_ms": round(ms, 3), "enc_frac_of_device": round(dms / ms, 4), "enc_ok": ok,
                          "dec_ms": round(dms_dec, 3), "dec_ok": ok_dec}
        print(json.dumps(row), flush=True)
        del pt_h, ct_h, back_h, pt_d, ct_d


if __name__ == "__main__":
    main()
