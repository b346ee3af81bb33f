"""An independent, tiny pure-Python reading of arXiv 1201.3114's chaotic operation mode.

Used only by tests, as a second implementation written separately from the C
oracle (it shares no code with ``oracle/`` or the CUDA path): Python binary64
floats (IEEE round-to-nearest, never fused), ``hashlib`` for SHA-256, Python
big integers for the packing. If the C oracle and this file agree bit for bit on
small inputs, a transcription slip in either is very unlikely.

Paper references: P:n = PAPER.md line n. Readings: DESIGN.md §3.
"""
from __future__ import annotations

import hashlib
import math

SENT = b"LORENZCHAOS-MAC1"
DTS = [0.01, 0.005, 0.02, 0.027]


def pack(pw: bytes):
    """Eqs.2-4, written with Python integers and 0-based slices."""
    n = len(pw)
    L = n // 3
    rem = n % 3
    lo, mid, hi = pw[0:L], pw[L:2 * L], pw[2 * L:3 * L]
    le = lambda bs: int.from_bytes(bytes(bs), "little")  # sum pi_i 2^{8(i-1)}
    a1 = le(lo) if rem == 0 else (le(lo) << 8) + pw[3 * L]
    a2 = (le(mid) << 8) + pw[3 * L + 1] if rem == 2 else le(mid)
    a3 = le(hi)
    return [a1, a2, a3], L


def key_material(pw: bytes, variant: int = 0):
    a, L = pack(pw)
    d = len(str(2 ** (8 * (L + 1))))          # ceil(log10 2^{8(L+1)})
    ap = [float(ai) / float(10 ** d) for ai in a]
    lo, hi = [-15.67, -11.28, 0.090], [16.01, 16.01, 62.000]
    lam = []
    for i in (1, 2, 3):
        msg = b"\x4c" + b"".join(x.to_bytes(8, "big") for x in a) + bytes([i])
        h = int.from_bytes(hashlib.sha256(msg).digest()[:8], "big")
        t = float(h) * 2.0 ** -64
        lam.append(lo[i - 1] + t * (hi[i - 1] - lo[i - 1]))
    r0 = [ap[i] + lam[i] for i in range(3)]
    mu = [(a[0] + a[1] + a[2]) % 3, (a[0] * a[1] + a[2]) % 3, (a[0] + a[1] * a[2]) % 3]
    H = hashlib.sha256(pw).digest()
    k = [3 + H[0] % 2, 3 + H[1] % 2, 3 + H[2] % 2]
    k3c = 1 + H[3] % 6
    hs = []
    for i in (1, 2, 3):
        msg = b"".join(((i * x) % 2 ** 64).to_bytes(8, "big") for x in a)
        hs.append(int.from_bytes(hashlib.sha256(msg).digest()[:8], "big"))
    if variant & 4:  # NEXT-4 "distinct k": k2 = 7 - k1
        k[1] = 7 - k[0]
    om = [hs[i] % k[i] for i in range(3)]
    return dict(a=a, ap=ap, r0=r0, mu=mu, k=k, k3c=k3c, omega=om)


def f(x, y, z):
    return 10.0 * (y - x), (28.0 * x - y) - x * z, x * y - (8.0 / 3.0) * z


def rk4(s, h):
    h2, h6 = h * 0.5, h / 6.0
    k1 = f(*s)
    k2 = f(*[s[c] + h2 * k1[c] for c in range(3)])
    k3 = f(*[s[c] + h2 * k2[c] for c in range(3)])
    k4 = f(*[s[c] + h * k3[c] for c in range(3)])
    return [s[c] + h6 * (((((k1[c] + k2[c]) + k2[c]) + k3[c]) + k3[c]) + k4[c]) for c in range(3)]


def euler(s, h):
    d = f(*s)
    return [s[c] + d[c] * h for c in range(3)]


def fma(a, b, c):
    """Correctly rounded a*b + c, computed exactly with fractions (Python 3.12 has no math.fma)."""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def f_fma(x, y, z):
    return 10.0 * (y - x), fma(-x, z, fma(28.0, x, -y)), fma(x, y, -((8.0 / 3.0) * z))


def rk4fma(s, h):
    h2, h6 = h * 0.5, h / 6.0
    k1 = f_fma(*s)
    k2 = f_fma(*[fma(h2, k1[c], s[c]) for c in range(3)])
    k3 = f_fma(*[fma(h2, k2[c], s[c]) for c in range(3)])
    k4 = f_fma(*[fma(h, k3[c], s[c]) for c in range(3)])
    return [fma(h6, fma(2.0, k3[c], fma(2.0, k2[c], k1[c])) + k4[c], s[c]) for c in range(3)]


def Rnu(alpha, omega):
    return (int(abs(alpha) * 1e13) >> (8 * omega)) & 0xFF


def run_stream(km, data: bytes, n_it: int, dt_code=0, decrypt=False, integrator="rk4", variant=0):
    """variant bits 0-1 (NEXT-4 Step-3 order): 0 adopted reading, 1 literal text order,
    2 cyclic index; bit 2 (distinct k) is applied in key_material."""
    h = DTS[dt_code]
    step = {"rk4": rk4, "euler": euler, "rk4fma": rk4fma}[integrator]
    r = list(km["r0"])
    mu, om = list(km["mu"]), list(km["omega"])
    k = [km["k"][0], km["k"][1], km["k3c"]]
    alpha = [r[mu[i]] for i in range(3)]
    src = bytes(data) if decrypt else bytes(data) + SENT
    out = bytearray()
    for j, x in enumerate(src):
        ks = Rnu(alpha[0], om[0]) + Rnu(alpha[1], om[1])
        y = (x - ks) % 256 if decrypt else (x + ks) % 256
        out.append(y)
        p = y if decrypt else x
        if j == len(src) - 1:
            break
        r[mu[2]] = r[mu[2]] + float(p) / float(10 ** (3 + om[2]))
        for _ in range(n_it):
            r = step(r, h)
        order = variant & 3
        if order == 1:  # mu from the previous alpha, then alpha from the new mu, then Omega
            mu = [(mu[i] + Rnu(alpha[i], om[i])) % 3 for i in range(3)]
            alpha = [r[mu[i]] for i in range(3)]
            om = [(om[i] + Rnu(alpha[i], om[i])) % k[i] for i in range(3)]
        else:
            alpha = [r[mu[i]] for i in range(3)]
            Rv = [Rnu(alpha[i], om[i]) for i in range(3)]
            mu = [(mu[i] + Rv[i]) % 3 for i in range(3)]
            if order == 2:
                om = [(om[i] + Rnu(alpha[(i + 1) % 3], om[i])) % k[i] for i in range(3)]
            else:
                om = [(om[i] + Rv[i]) % k[i] for i in range(3)]
        r = [r[i] + km["ap"][i] for i in range(3)]
    return bytes(out)


def norm_pw(pw: bytes) -> bytes:
    return hashlib.sha256(pw).digest()[:18] if len(pw) > 23 else pw


def encrypt_message(pw: bytes, pt: bytes, fast: bool, n_it: int, B=1024, dt_code=0):
    if not fast:
        return run_stream(key_material(norm_pw(pw)), pt, n_it, dt_code)
    nb = max(1, -(-len(pt) // B))
    out = b""
    for b in range(nb):
        sub = hashlib.sha256(pw + b.to_bytes(4, "big")).digest()[:18]
        out += run_stream(key_material(sub), pt[b * B:(b + 1) * B], n_it, dt_code)
    return out


def decrypt_message(pw: bytes, ct: bytes, fast: bool, n_it: int, B=1024, dt_code=0):
    """Returns (plaintext, list of per-block sentinel verdicts)."""
    if not fast:
        rec = run_stream(key_material(norm_pw(pw)), ct, n_it, dt_code, decrypt=True)
        return rec[:-16], [rec[-16:] == SENT]
    out, oks, pos, b = b"", [], 0, 0
    while pos < len(ct):
        seg = ct[pos:pos + B + 16]
        sub = hashlib.sha256(pw + b.to_bytes(4, "big")).digest()[:18]
        rec = run_stream(key_material(sub), seg, n_it, dt_code, decrypt=True)
        out += rec[:-16]
        oks.append(rec[-16:] == SENT)
        pos += len(seg)
        b += 1
    return out, oks


assert math.isclose(DTS[0], 0.01)
