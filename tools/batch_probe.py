"""Time lorenz_encrypt_batch alone (C5 launch shape: 384 streams x 1 MiB) with CUDA events and
wall clock, for the CTA-size dispatch study. Usage: [PROBE_CTA=128|256] python tools/batch_probe.py"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import fp64_ops  # noqa: E402
from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def main():
    S, n = int(os.environ.get("PROBE_STREAMS", "384")), 1 << 20
    dev = torch.device("cuda:0")
    if os.environ.get("PROBE_CTA"):
        L.lorenz_set_tuning(cta=int(os.environ["PROBE_CTA"]))
    keys = [L.lorenz_keysetup(inputs.password(seed=s), mode=L.FAST) for s in range(S)]
    pts = torch.from_numpy(np.tile(inputs.message(n), S)).to(dev)
    ctl = keys[0].ct_len(n)
    cts = torch.empty(S * ctl, dtype=torch.uint8, device=dev)
    tags = torch.empty(S * 16, dtype=torch.uint8, device=dev)
    L.lorenz_encrypt_batch(keys, n, pts, cts, tags)
    out = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        L.lorenz_encrypt_batch(keys, n, pts, cts, tags)
        e1.record()
        torch.cuda.synchronize()
        out.append((e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0))
    ev = min(o[0] for o in out)
    ops = S * fp64_ops(n, 1024, 0, n // 1024, 100)
    print(json.dumps({"cta_env": os.environ.get("PROBE_CTA"), "streams": S, "event_s": round(ev, 4),
                      "wall_s": round(min(o[1] for o in out), 4), "frac": round(ops / ev / (148 * 64 * 1965e6), 4)}))


if __name__ == "__main__":
    main()
