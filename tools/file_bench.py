"""NEXT-2 measurement: end-to-end file encryption/decryption through lorenz_encrypt_file /
lorenz_decrypt_file (disk -> pinned -> HBM -> kernel -> HBM -> pinned -> disk, 3 chunks in flight).

Usage: python tools/file_bench.py [--mib 1024] [--chunk-mib 256] [--dir /dev/shm]
Prints one JSON line. The files live in --dir (tmpfs by default, so the disk is not the bound).
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--chunk-mib", type=int, default=32)
    ap.add_argument("--dir", default="/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir())
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    n = a.mib << 20
    d = tempfile.mkdtemp(dir=a.dir)
    src, enc, dec = (os.path.join(d, x) for x in ("in.bin", "out.lzx", "back.bin"))
    inputs.message(n).tofile(src)
    pw = inputs.password()
    L.lorenz_encrypt_file(src, enc, pw, chunk_bytes=a.chunk_mib << 20)  # warm up (CUDA context, pools)
    te, td = [], []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        tag = L.lorenz_encrypt_file(src, enc, pw, chunk_bytes=a.chunk_mib << 20)
        te.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        st, fb = L.lorenz_decrypt_file(enc, dec, pw, chunk_bytes=a.chunk_mib << 20)
        td.append(time.perf_counter() - t0)
        assert st == L.OK
    same = open(src, "rb").read() == open(dec, "rb").read()
    for p in (src, enc, dec):
        os.unlink(p)
    os.rmdir(d)
    print(json.dumps({"what": "lorenz_encrypt_file / lorenz_decrypt_file (NEXT-2)", "bytes": n,
                      "chunk_bytes": a.chunk_mib << 20, "dir": a.dir,
                      "encrypt_MBps": round(n / min(te) / 1e6, 1), "decrypt_MBps": round(n / min(td) / 1e6, 1),
                      "round_trip_ok": same, "tag": tag.hex()}))


if __name__ == "__main__":
    main()
