"""NEXT-4 measurement: the paper's Figs. 3 and 4 on the GPU.

Usage: python tools/spectra.py [--sizes 256 1024 4096] [--reps 10] [--fig 1024]
Prints JSON lines:
  * timing of lorenz_power_spectrum / lorenz_autocorrelation per size (CUDA events, warm,
    L2-resident only below 126 MB) with the HBM bytes of DESIGN.md §4 (N = H W): the
    unavoidable 9 N (bytes in, float64 out) and the implemented pipeline's 25 N (spectrum:
    R2C rows + half-spectrum columns) / 58 N (autocorrelation: byte sum, R2C rows, fused
    transform-|.|^2-transform columns, C2R rows, normalisation) -> GB/s;
  * the CPU oracle (plain O(N^2) sums, one core) timed beside the GPU at --oracle-side (128);
  * the Fig.3 / Fig.4 experiment at --fig x --fig (0: skipped): a synthetic plain image, its ciphertext
    (FAST, the first N ciphertext bytes) and white noise -> byte entropy, spectral flatness,
    r(1,0), r(0,1), max off-origin |r|.
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402

DEV = torch.device("cuda:0")


def plain_image(h, w):
    i, j = np.indices((h, w))
    g = 60 + 100 * i / h + 40 * j / w
    g += 50 * (((i - h / 2) ** 2 + (j - w / 3) ** 2) < (min(h, w) / 4) ** 2)
    g += 20 * ((j // 4) % 2)
    return np.clip(g, 0, 255).astype(np.uint8)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def entropy(x):
    c = np.bincount(x.ravel(), minlength=256).astype(np.float64)
    p = c[c > 0] / c.sum()
    return float(-(p * np.log2(p)).sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[256, 1024, 4096])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fig", type=int, default=1024)
    ap.add_argument("--oracle-side", type=int, default=128)
    a = ap.parse_args()
    for s in a.sizes:
        n = s * s
        x = torch.from_numpy(inputs.message(n, seed=2)).to(DEV).view(s, s)
        p = torch.empty((s, s), dtype=torch.float64, device=DEV)
        f = torch.empty(1, dtype=torch.float64, device=DEV)
        r = torch.empty((s, s), dtype=torch.float64, device=DEV)
        tp = timed(lambda: L.lorenz_power_spectrum(x, p, f), a.reps)
        ta = timed(lambda: L.lorenz_autocorrelation(x, r), a.reps)
        print(json.dumps({"what": "NEXT-4 spectra timing", "side": s, "spectrum_ms": round(tp * 1e3, 4),
                          "spectrum_gbs_pipeline": round(25 * n / tp / 1e9, 1),
                          "spectrum_gbs_in_out": round(9 * n / tp / 1e9, 1), "autocorr_ms": round(ta * 1e3, 4),
                          "autocorr_gbs_pipeline": round(58 * n / ta / 1e9, 1),
                          "autocorr_gbs_in_out": round(9 * n / ta / 1e9, 1)}))
    if a.oracle_side:
        import time

        import oracle
        s = a.oracle_side
        img = inputs.message(s * s, seed=2).reshape(s, s)
        t0 = time.perf_counter()
        oracle.power_spectrum(img)
        cp = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.autocorr(img)
        ca = time.perf_counter() - t0
        x = torch.from_numpy(img).to(DEV)
        p = torch.empty((s, s), dtype=torch.float64, device=DEV)
        f = torch.empty(1, dtype=torch.float64, device=DEV)
        r = torch.empty((s, s), dtype=torch.float64, device=DEV)
        tp = timed(lambda: L.lorenz_power_spectrum(x, p, f), a.reps)
        ta = timed(lambda: L.lorenz_autocorrelation(x, r), a.reps)
        print(json.dumps({"what": "CPU oracle beside the GPU (plain O(N^2) definitions, 1 core)", "side": s,
                          "oracle_spectrum_s": round(cp, 3), "gpu_spectrum_ms": round(tp * 1e3, 4),
                          "oracle_autocorr_s": round(ca, 3), "gpu_autocorr_ms": round(ta * 1e3, 4)}))
    if not a.fig:
        return
    s = a.fig
    n = s * s
    plain = plain_image(s, s)
    key = L.lorenz_keysetup(inputs.password(), mode=L.FAST)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt(key, n, 0, key.num_blocks(n), torch.from_numpy(plain.ravel()).to(DEV), ct)
    images = {"plain": plain, "cipher": ct[:n].cpu().numpy().reshape(s, s),
              "noise": inputs.message(n, seed=99).reshape(s, s)}
    out = {"what": "Fig.3/Fig.4 experiment (synthetic plain image, FAST n_it=100)", "side": s,
           "flatness_white_noise_expected": round(math.exp(-0.5772156649015329), 4)}
    for name, img in images.items():
        xd = torch.from_numpy(np.ascontiguousarray(img)).to(DEV)
        p = torch.empty((s, s), dtype=torch.float64, device=DEV)
        f = torch.empty(1, dtype=torch.float64, device=DEV)
        r = torch.empty((s, s), dtype=torch.float64, device=DEV)
        L.lorenz_power_spectrum(xd, p, f)
        L.lorenz_autocorrelation(xd, r)
        rc = r.cpu().numpy()
        out[name] = {"entropy_bits": round(entropy(img), 5), "flatness": round(float(f.item()), 5),
                     "r10": round(float(rc[1, 0]), 5), "r01": round(float(rc[0, 1]), 5),
                     "max_off_origin_abs_r": round(float(np.abs(rc.ravel()[1:]).max()), 5)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
