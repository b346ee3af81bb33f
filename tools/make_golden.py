"""Write tests/golden/ regression fixtures. Calls ONLY the CPU oracle (oracle/).

Usage: python tools/make_golden.py
"""
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def main():
    s = (1.0, 1.0, 1.0)
    lines = ["# RK4 (canonical order, DESIGN.md §3 Q3) from (1,1,1), h = 0.01: states 1..100",
             "# one state per line: x y z as big-endian hex of IEEE binary64 (S:66, S:79)",
             "# written by tools/make_golden.py from oracle/ only"]
    for _ in range(100):
        s = oracle.rk4_step(s, 0.01)
        lines.append(" ".join(struct.pack(">d", v).hex() for v in s))
    with open(os.path.join(GOLD, "rk4_trajectory_h001.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
