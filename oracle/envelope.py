"""CPU ORACLE for the envelope file format (SPEC envelope module).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Plain Python ``struct`` packing of the
24-byte header followed by the oracle's ciphertext; the GPU file path must reproduce
these bytes exactly.

Header, little-endian: magic "LZX1" | u8 version = 1 | u8 mode (0 strong, 1 fast) |
u8 flags (SPEC: reserved 0; here the integrator code, 0 = RK4) | u8 dt_code | u32 n_it |
u32 chunk_size (the block size B; 0 in strong mode) | u64 payload_len.
"""
from __future__ import annotations

import struct

from . import FAST, STRONG, Params, encrypt

HEADER = struct.Struct("<4sBBBBIIQ")
assert HEADER.size == 24


def effective(prm: Params) -> tuple:
    """(mode, n_it, dt_code, block_size, flags) with the defaults of S:33 / S:312; flags =
    integrator | variant << 2 (0 for the default cipher, as SPEC's reserved byte)."""
    n_it = prm.n_it or (100 if prm.mode == FAST else 3000)
    B = (prm.block_size or 1024) if prm.mode == FAST else 0
    return prm.mode, n_it, prm.dt_code, B, prm.integrator | (prm.variant << 2)


def header(prm: Params, n: int) -> bytes:
    mode, n_it, dt, B, flags = effective(prm)
    return HEADER.pack(b"LZX1", 1, mode, flags, dt, n_it, B, n)


def parse(hdr: bytes) -> dict:
    if len(hdr) < HEADER.size:
        raise ValueError("truncated header")
    magic, ver, mode, flags, dt, n_it, chunk, n = HEADER.unpack(hdr[:HEADER.size])
    if magic != b"LZX1" or ver != 1 or mode not in (STRONG, FAST):
        raise ValueError("bad magic/version/mode")
    return dict(mode=mode, integrator=flags & 3, variant=flags >> 2, dt_code=dt, n_it=n_it, block_size=chunk, n=n)


def encrypt_file_bytes(pw: bytes, data: bytes, prm: Params) -> bytes:
    ct, _ = encrypt(pw, data, prm)
    return header(prm, len(data)) + ct.tobytes()
