"""Time the encrypt kernel of one liblorenz.so variant over several message sizes (1 GPU).

Usage: LORENZ_LIB=/path/to/variant.so python tools/tune.py --tag NAME [--mib 64 128 256 1024] [--n-it 100]
Prints one JSON line per size: MB/s and the FP64-pipe fraction (DESIGN.md §4 accounting).
The sizes model the per-rank slices of the C4 1 GiB message at N = 16, 8, 4, 1 GPUs.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import fp64_ops  # noqa: E402
from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default=os.environ.get("LORENZ_LIB", "default"))
    ap.add_argument("--mib", type=int, nargs="+", default=[64, 128, 256, 1024])
    ap.add_argument("--kib", type=int, nargs="+", default=None, help="sizes in KiB (= blocks at B = 1024)")
    ap.add_argument("--n-it", type=int, default=100)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--integrator", choices=["rk4", "euler", "rk4fma"], default="rk4")
    ap.add_argument("--sched", choices=["auto", "wave", "seg"], default="auto")
    ap.add_argument("--slots", type=int, default=0, help="balanced-kernel warp slots (0 = default)")
    ap.add_argument("--skew", type=int, default=-1, help="balanced-kernel skew per mille (-1 = default)")
    a = ap.parse_args()
    L.lorenz_set_tuning(schedule={"auto": L.SCHED_AUTO, "wave": L.SCHED_WAVE, "seg": L.SCHED_BALANCED}[a.sched],
                        seg_slots=a.slots, seg_skew=a.skew)
    dev = torch.device("cuda:0")
    integ = {"rk4": L.RK4, "euler": L.EULER, "rk4fma": L.RK4_FMA}[a.integrator]
    key = L.lorenz_keysetup(inputs.password(), mode=L.FAST, n_it=a.n_it, integrator=integ)
    sizes = [k << 10 for k in a.kib] if a.kib else [m << 20 for m in a.mib]
    big = max(sizes)
    msg = torch.from_numpy(inputs.message(big)).to(dev)
    ct = torch.empty(key.ct_len(big), dtype=torch.uint8, device=dev)
    res = torch.empty(32, dtype=torch.uint8, device=dev)
    peak = 148 * 64 * 1965e6
    for n in sizes:
        nb = key.num_blocks(n)
        L.lorenz_result_init_async(res)
        L.lorenz_encrypt_async(key, n, 0, nb, msg, ct, res)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.lorenz_encrypt_async(key, n, 0, nb, msg, ct, res)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = min(ts)
        ops = fp64_ops(n, 1024, 0, nb, a.n_it, a.integrator)
        print(json.dumps({"tag": a.tag, "integrator": a.integrator, "plan": L.lorenz_launch_plan(key, n, 0, nb), "mib": round(n / 2**20, 3), "blocks": nb, "ms": round(t * 1e3, 3),
                          "MBps": round(n / t / 1e6, 1), "frac": round(ops / t / peak, 4)}), flush=True)


if __name__ == "__main__":
    main()
