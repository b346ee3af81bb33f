"""Per-call wall time of the host-buffer API (lorenz_encrypt_host) on C3 (64 MiB), automatic and
fixed chunk counts, 4 calls each (1 GPU). Shows the first-call cost and the chunking trade-off.

Usage: python tools/e2e_probe.py [--mib 64]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=64)
    a = ap.parse_args()
    n = a.mib << 20
    key = L.lorenz_keysetup(inputs.password(), mode=L.FAST)
    pt_h = torch.from_numpy(inputs.message(n)).pin_memory()
    ct_h = torch.empty(key.ct_len(n), dtype=torch.uint8).pin_memory()
    nb = key.num_blocks(n)
    for chunks in [0, 0, 0, 1, 2, 4]:
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            L.lorenz_encrypt_host(key, n, 0, nb, pt_h, ct_h, n_chunks=chunks)
            ts.append(time.perf_counter() - t0)
        print(json.dumps({"mib": a.mib, "chunks": chunks, "ms": [round(t * 1e3, 2) for t in ts]}), flush=True)


if __name__ == "__main__":
    main()
