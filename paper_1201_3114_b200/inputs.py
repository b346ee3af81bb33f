"""Seeded synthetic inputs (messages, passwords, flips) shared by tests, smoke and bench.

This module holds none of the cipher's arithmetic: it only draws bytes. It is the
one module both the oracle side and the CUDA side are fed from.

Recipe (SURVEY.md §8d "Synthetic inputs"):
* message byte i = byte (i mod 8), little-endian, of SplitMix64(seed XOR floor(i/8));
  counter-based, so any rank regenerates any slice [start, end) identically;
* password byte k = 0x21 + SplitMix64(seed_pw XOR k) mod 94 (printable ASCII), 16 bytes;
* trial t of the C5 sweep uses seeds XOR t; its flip position is
  SplitMix64(SEED_FLIP XOR t) mod (8 * length).
"""
from __future__ import annotations

import numpy as np

SEED_MSG = 0x12013114
SEED_PW = 0x5EED
SEED_FLIP = 0xF11B

_M64 = (1 << 64) - 1


def splitmix64(x):
    """SplitMix64 output for counter value(s) x (numpy uint64 array or int)."""
    if isinstance(x, (int, np.integer)):
        z = (int(x) + 0x9E3779B97F4A7C15) & _M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)
    z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def message(n: int, seed: int = SEED_MSG, start: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Bytes [start, start+n) of the message stream for `seed` (uint8 array)."""
    if n == 0:
        return np.zeros(0, dtype=np.uint8) if out is None else out[:0]
    w0, w1 = start // 8, (start + n + 7) // 8
    chunk = 1 << 24  # words per chunk: bounds temporary memory for GiB messages
    res = np.empty(n, dtype=np.uint8) if out is None else out
    pos = 0
    for c0 in range(w0, w1, chunk):
        c1 = min(w1, c0 + chunk)
        idx = np.arange(c0, c1, dtype=np.uint64) ^ np.uint64(seed)
        by = splitmix64(idx).view(np.uint8)  # little-endian bytes
        lo = max(start - 8 * c0, 0)
        hi = min(start + n - 8 * c0, by.size)
        seg = by[lo:hi]
        res[pos:pos + seg.size] = seg
        pos += seg.size
    assert pos == n
    return res


SEED_IC = 0xF161  # Fig.1 trajectories
# initial states uniform in the lambda box of P:216 widened by a' <= 1: where r0 lives
IC_LO = (-15.67, -11.28, 0.090)
IC_HI = (17.01, 17.01, 63.0)


def initial_states(lanes: int, seed: int = SEED_IC) -> np.ndarray:
    """(lanes, 3) float64: component c of lane l = lo_c + u (hi_c - lo_c), u = 53-bit uniform
    from SplitMix64(seed XOR (3 l + c))."""
    idx = np.arange(3 * lanes, dtype=np.uint64) ^ np.uint64(seed)
    u = (splitmix64(idx) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    lo, hi = np.array(IC_LO * lanes), np.array(IC_HI * lanes)
    return (lo + u * (hi - lo)).reshape(lanes, 3)


def password(seed: int = SEED_PW, length: int = 16) -> bytes:
    return bytes(0x21 + splitmix64(seed ^ k) % 94 for k in range(length))


def flip_position(t: int, length: int) -> int:
    return splitmix64(SEED_FLIP ^ t) % (8 * length)


def flip_bit(buf: bytes | np.ndarray, bitpos: int):
    """Copy of buf with bit `bitpos` (byte bitpos//8, bit bitpos%8) inverted."""
    b = bytearray(bytes(buf)) if not isinstance(buf, np.ndarray) else buf.copy()
    b[bitpos // 8] ^= 1 << (bitpos % 8)
    return bytes(b) if not isinstance(buf, np.ndarray) else b
