"""One host-buffer call in direct mode (pinned buffers, lorenz_encrypt_host / lorenz_decrypt_host), for
an ncu capture of the chain kernel's PCIe traffic: the plaintext / ciphertext cross PCIe inside the
kernel. Usage (under ncu):
  ncu --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum -k regex:lorenz_chain \
      python tools/pcie_probe.py --mib 256
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1201_3114_b200 import inputs  # noqa: E402
from paper_1201_3114_b200 import lorenz as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    a = ap.parse_args()
    n = a.mib << 20
    key = L.lorenz_keysetup(inputs.password(), mode=L.FAST)
    nb = key.num_blocks(n)
    pt_h = torch.from_numpy(inputs.message(n)).pin_memory()
    ct_h = torch.empty(key.ct_len(n), dtype=torch.uint8).pin_memory()
    back_h = torch.empty(n, dtype=torch.uint8).pin_memory()
    L.lorenz_encrypt_host(key, n, 0, nb, pt_h, ct_h)
    st, fb = L.lorenz_decrypt_host(key, n, 0, nb, ct_h, back_h)
    assert st == L.OK and torch.equal(back_h, pt_h)
    print({"mib": a.mib, "pt_bytes": n, "ct_bytes": key.ct_len(n)})


if __name__ == "__main__":
    main()
