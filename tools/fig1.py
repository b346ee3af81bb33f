"""NEXT-4 measurement: the paper's Fig.1 on the GPU at scale.

Usage: python tools/fig1.py [--lanes 262144] [--skip 1000] [--samples 200] [--stride 10]
Prints one JSON line: time, FP64-pipe fraction (RK4 ops only), and per coordinate the
integer-part range and the chi-square (99 dof) of the digit pairs 1-2, 3-4, 5-6.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lanes", type=int, default=262144)
    ap.add_argument("--skip", type=int, default=1000)
    ap.add_argument("--samples", type=int, default=200)
    ap.add_argument("--stride", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    ic = torch.from_numpy(inputs.initial_states(a.lanes)).to(dev)
    hist = torch.empty(3 * 4 * 128, dtype=torch.int64, device=dev)
    L.lorenz_digit_histograms(ic, min(a.lanes, 1024), 10, 10, 1, hist)  # warm up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.lorenz_digit_histograms(ic, a.lanes, a.skip, a.samples, a.stride, hist)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3
    ops = a.lanes * (a.skip + a.samples * a.stride) * 75
    digit_ops = a.lanes * a.samples * 9  # |v| 10^2, 10^4, 10^6 for 3 coordinates per sample (DMUL)
    h = hist.cpu().numpy().reshape(3, 4, 128)
    out = {"what": "Fig.1 digit histograms (NEXT-4)", "lanes": a.lanes, "skip": a.skip, "samples": a.samples,
           "stride": a.stride, "seconds": round(sec, 4),
           "fp64_pipe_frac": round(ops / sec / (148 * 64 * 1965e6), 4),
           "fp64_pipe_frac_incl_digit_products": round((ops + digit_ops) / sec / (148 * 64 * 1965e6), 4), "coords": {}}
    for c, name in enumerate("xyz"):
        nz = np.nonzero(h[c, 0])[0] - 64
        chis = []
        for k in (1, 2, 3):
            e = h[c, k, :100].sum() / 100
            chis.append(round(float((((h[c, k, :100] - e) ** 2) / e).sum()), 1))
        out["coords"][name] = {"int_part_range": [int(nz.min()), int(nz.max())],
                               "chi2_digits_12_34_56": chis, "chi2_p99_99dof": 135.8}
    # the CPU oracle beside it: the same recipe on a bounded sample of trajectories, one core
    import time

    import oracle
    lanes_cpu = min(a.lanes, 512)
    t0 = time.perf_counter()
    oracle.digit_hist(inputs.initial_states(lanes_cpu), a.skip, a.samples, a.stride)
    cpu_s = time.perf_counter() - t0
    steps = a.skip + a.samples * a.stride
    out["cpu_oracle"] = {"lanes": lanes_cpu, "seconds": round(cpu_s, 3), "cores": 1,
                         "rk4_steps_per_s": round(lanes_cpu * steps / cpu_s, 1),
                         "gpu_rk4_steps_per_s": round(a.lanes * steps / sec, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
