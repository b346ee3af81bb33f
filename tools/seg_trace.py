"""Timeline of the balanced (McNaughton) chain kernel, one row per warp slot (1 GPU).

Builds nothing itself: run it with LORENZ_LIB pointing at a tuning build of the library,
`python paper_1201_3114_b200/build.py -D LZ_SEG_TRACE --out tools/variants/liblorenz_trace.so`.
For one encrypt launch of each size it prints the slot count, the kernel time, how long slots
waited for their cut unit's first piece, and when slots finished relative to the kernel's end
(the tail), per SM sub-partition.

Usage: LORENZ_LIB=tools/variants/liblorenz_trace.so python tools/seg_trace.py --kib 65536 100000
"""
import argparse
import ctypes as C
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
    ap.add_argument("--kib", type=int, nargs="+", default=[65536, 100000, 131072])
    ap.add_argument("--n-it", type=int, default=100)
    ap.add_argument("--dump", default=None, help="write the raw per-slot rows (npz) here")
    ap.add_argument("--integrator", choices=["rk4", "euler", "rk4fma"], default="rk4")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    lib = L.lib()
    lib.lorenz_debug_seg_trace.argtypes = [C.c_void_p]
    key = L.lorenz_keysetup(inputs.password(), mode=L.FAST, n_it=a.n_it,
                            integrator={"rk4": L.RK4, "euler": L.EULER, "rk4fma": L.RK4_FMA}[a.integrator])
    big = max(a.kib) << 10
    msg = torch.from_numpy(inputs.message(big)).to(dev)
    ct = torch.empty(key.ct_len(big), dtype=torch.uint8, device=dev)
    res = torch.empty(32, dtype=torch.uint8, device=dev)
    raw = {}
    for kib in a.kib:
        n = kib << 10
        nb = key.num_blocks(n)
        L.lorenz_result_init_async(res)
        L.lorenz_encrypt_async(key, n, 0, nb, msg, ct, res)  # warm
        torch.cuda.synchronize()
        tr = np.zeros(4096 * 8, dtype=np.uint64)
        lib.lorenz_debug_seg_trace(tr.ctypes.data)  # read-and-clear: drop the warm-up launch's rows
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.lorenz_encrypt_async(key, n, 0, nb, msg, ct, res)
        e1.record()
        torch.cuda.synchronize()
        lib.lorenz_debug_seg_trace(tr.ctypes.data)
        tr = tr.reshape(4096, 8).astype(np.int64)
        used = tr[:, 0] > 0
        t0 = tr[used, 0].min()
        rows = tr[used]
        start, first, arrive, go, fin = (rows[:, i] - t0 for i in range(5))
        waited = (rows[:, 2] > 0)
        wait = np.where(waited, rows[:, 3] - rows[:, 2], 0)
        sm = rows[:, 6] >> 32
        wid = rows[:, 6] & 0xFFFFFFFF
        end = fin.max()
        raw[kib] = rows
        print(json.dumps({
            "kib": kib, "slots": int(used.sum()), "kernel_ms": round(e0.elapsed_time(e1), 3),
            "span_ms": round(end / 1e6, 3), "start_spread_us": round((start.max() - start.min()) / 1e3, 1),
            "slots_waiting": int((wait > 1000).sum()), "wait_ms_max": round(wait.max() / 1e6, 3),
            "wait_ms_mean": round(wait.mean() / 1e6, 4),
            "finish_ms_p0_p50_p100": [round(float(np.percentile(fin, q)) / 1e6, 3) for q in (0, 50, 100)],
            "first_piece_done_ms_p50_p100": [round(float(np.percentile(first[first > -t0], q)) / 1e6, 3)
                                             for q in (50, 100)] if (rows[:, 1] > 0).any() else None,
            "warpid_mod4_counts": np.bincount((wid % 4).astype(np.int64), minlength=4).tolist(),
            # mean finish time per warp index within the CTA (t = start order): rate differences
            "finish_ms_by_warp_in_cta": [round(float(fin[(rows[:, 7] % (int(used.sum()) // 148)) == w].mean()) / 1e6, 3)
                                         for w in range(int(used.sum()) // 148)],
            "sms": int(len(np.unique(sm))),
        }), flush=True)
    if a.dump:
        np.savez(a.dump, **{str(k): v for k, v in raw.items()})


if __name__ == "__main__":
    main()
