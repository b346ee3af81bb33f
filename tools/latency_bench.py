"""C1 / C2 timings: the latency-bound configurations (one lane / 1,024 lanes), GPU vs the CPU oracle.

C1: 1 KiB, 16-byte password, STRONG (one block), n_it = 3000 (the paper's value):
    encrypt + decrypt + verify.
C2: 1 MiB, FAST, n_it = 100, B = 1024 (1,024 blocks) and B = 65,536 (16 blocks).
Each chain is sequential, so these sizes cannot fill 148 SMs; the numbers show the
per-lane latency regime (≈ 19 dependent FP64 operations x 8.8 cycles per RK4 step).
Usage: python tools/latency_bench.py
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (timing baseline only)
from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def gpu_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def main():
    dev = torch.device("cuda:0")
    pw = inputs.password()
    out = []
    for name, n, kw in [("C1 STRONG n_it=3000", 1024, dict(mode=L.STRONG, n_it=3000)),
                        ("C2 FAST B=1024", 1 << 20, dict(mode=L.FAST, n_it=100)),
                        ("C2 FAST B=65536", 1 << 20, dict(mode=L.FAST, n_it=100, block_size=65536))]:
        key = L.lorenz_keysetup(pw, **kw)
        msg = inputs.message(n)
        pt = torch.from_numpy(msg).to(dev)
        nb = key.num_blocks(n)
        ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=dev)
        back = torch.empty(n, dtype=torch.uint8, device=dev)
        res = torch.empty(32, dtype=torch.uint8, device=dev)

        def enc():
            L.lorenz_result_init_async(res)
            L.lorenz_encrypt_async(key, n, 0, nb, pt, ct, res)

        def dec():
            L.lorenz_result_init_async(res)
            L.lorenz_decrypt_async(key, n, 0, nb, ct, back, res)

        def ver():
            L.lorenz_result_init_async(res)
            L.lorenz_verify_async(key, n, 0, nb, ct, res)
        te, td, tv = gpu_time(enc), gpu_time(dec), gpu_time(ver)
        assert torch.equal(back, pt)
        p = key.params
        prm = oracle.params(mode=p.mode, n_it=p.n_it, block_size=p.block_size)
        threads = 1 if p.mode == L.STRONG else len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        want, _ = oracle.encrypt(pw, msg, prm, threads=threads)
        tc = time.perf_counter() - t0
        assert np.array_equal(ct.cpu().numpy(), want)
        out.append({"config": name, "bytes": n, "lanes": nb, "gpu_encrypt_s": round(te, 5),
                    "gpu_decrypt_s": round(td, 5), "gpu_verify_s": round(tv, 5),
                    "gpu_encrypt_MBps": round(n / te / 1e6, 3), "oracle_encrypt_s": round(tc, 4),
                    "oracle_threads": threads, "parity": True})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
