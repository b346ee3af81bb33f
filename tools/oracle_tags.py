"""Write tests/golden/oracle_tags.json: the message digest (XOR of the block tags, Q15) of the
bench workloads, computed by the CPU ORACLE alone (oracle/, all host cores) from the seeded
inputs of paper_1201_3114_b200/inputs.py. bench.py checks its combined tag against these at
every rank count (the driver's scaling runs) and tests/test_gpu_fullsize.py against the
oracle's own result. Nothing here touches the CUDA path.

Usage: python tools/oracle_tags.py [--skip-c4]     (C4 takes ~15 min on 8 cores)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1201_3114_b200 import inputs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_tags.json")
INTEG = {"rk4": oracle.RK4, "euler": oracle.EULER, "rk4fma": oracle.RK4_FMA}


def digest(n: int, n_it: int, integrator: str) -> str:
    msg = inputs.message(n)
    prm = oracle.params(mode=oracle.FAST, n_it=n_it, block_size=1024, integrator=INTEG[integrator])
    _, tag = oracle.encrypt(inputs.password(), msg, prm, threads=0)
    return tag.hex()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    a = ap.parse_args()
    cases = [("c3", 64 << 20, 100, "rk4"), ("c3", 64 << 20, 100, "euler"), ("c3", 64 << 20, 100, "rk4fma")]
    if not a.skip_c4:
        cases.append(("c4", 1 << 30, 100, "rk4"))
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out["_doc"] = ("tag XOR of the whole message of each bench workload (password inputs.password(), message "
                   "inputs.message(n), FAST, B = 1024, dt_code 0, variant 0), from oracle.encrypt only; "
                   "written by tools/oracle_tags.py")
    for wl, n, n_it, integ in cases:
        t0 = time.time()
        out[f"{wl}/n_it={n_it}/{integ}"] = digest(n, n_it, integ)
        print(wl, n_it, integ, out[f"{wl}/n_it={n_it}/{integ}"], f"{time.time() - t0:.0f} s", flush=True)
        json.dump(out, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
