"""CPU ORACLE for arXiv 1201.3114's per-block chaotic operation mode.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package. The product package ``paper_1201_3114_b200`` never imports it.

This module is argument marshalling over ``oracle/liblorenz_ref.so`` (plain C,
``lorenz_ref.c``); every function's arithmetic and its citation live there.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblorenz_ref.so")

OK, E_INTEGRITY, E_ARG, E_PASSWORD, E_LENGTH, E_DIVERGENCE = 0, 1, 2, 3, 4, 5
STRONG, FAST = 0, 1
RK4, EULER, RK4_FMA = 0, 1, 2
SENTINEL = b"LORENZCHAOS-MAC1"


V_LITERAL, V_CYCLIC, V_DISTINCT_K = 1, 2, 4  # NEXT-4 Step-3 reading variants


class Params(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("n_it", C.c_uint32), ("dt_code", C.c_uint32),
                ("block_size", C.c_uint32), ("integrator", C.c_uint32), ("variant", C.c_uint32)]


class KeyMaterial(C.Structure):
    _fields_ = [("a", C.c_uint64 * 3), ("L", C.c_int), ("d", C.c_int),
                ("ap", C.c_double * 3), ("lam", C.c_double * 3), ("r0", C.c_double * 3),
                ("mu", C.c_int * 3), ("k", C.c_int * 3), ("k3chain", C.c_int),
                ("omega", C.c_int * 3), ("alpha", C.c_double * 3), ("hom", C.c_uint64 * 3)]

    def as_dict(self):
        return {"a": tuple(self.a), "L": self.L, "d": self.d, "ap": tuple(self.ap),
                "lam": tuple(self.lam), "r0": tuple(self.r0), "mu": tuple(self.mu),
                "k": tuple(self.k), "k3chain": self.k3chain, "omega": tuple(self.omega),
                "alpha": tuple(self.alpha)}


def build(verbose: bool = False) -> str:
    """Compile liblorenz_ref.so (strict IEEE flags, no FMA contraction)."""
    import subprocess
    src = os.path.join(_HERE, "lorenz_ref.c")
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", "-Wall", "-Wextra", "-o", LIB_PATH, src, "-lm"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "lorenz_ref.c")
        if (not os.path.exists(LIB_PATH)
                or os.path.getmtime(LIB_PATH) < os.path.getmtime(src)
                or os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "lorenz_ref.h"))):
            build()
        L = C.CDLL(LIB_PATH)
        u8p, dp, u64p, ip = C.POINTER(C.c_uint8), C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.POINTER(C.c_int)
        L.lorenz_ref_sha256.argtypes = [C.c_char_p, C.c_size_t, u8p]
        L.lorenz_ref_pack.argtypes = [C.c_char_p, C.c_size_t, u64p]
        L.lorenz_ref_norm_exponent.argtypes = [C.c_int]
        L.lorenz_ref_normalize.argtypes = [u64p, C.c_int, dp]
        L.lorenz_ref_lambda.argtypes = [u64p, dp]
        L.lorenz_ref_mu.argtypes = [u64p, ip]
        L.lorenz_ref_k_omega.argtypes = [C.c_char_p, C.c_size_t, u64p, ip, ip, ip]
        L.lorenz_ref_R.argtypes = [C.c_double, C.c_int]
        L.lorenz_ref_theta.argtypes = [C.c_int, C.c_int]
        L.lorenz_ref_theta.restype = C.c_double
        L.lorenz_ref_encode.argtypes = [C.c_int, C.c_int]
        L.lorenz_ref_decode.argtypes = [C.c_int, C.c_int]
        L.lorenz_ref_rhs.argtypes = [dp, dp]
        L.lorenz_ref_rk4_step.argtypes = [dp, C.c_double]
        L.lorenz_ref_euler_step.argtypes = [dp, C.c_double]
        L.lorenz_ref_rk4fma_step.argtypes = [dp, C.c_double]
        L.lorenz_ref_iterate.argtypes = [dp, C.c_uint32, C.c_uint32, C.c_uint64]
        L.lorenz_ref_dt.argtypes = [C.c_uint32]
        L.lorenz_ref_dt.restype = C.c_double
        L.lorenz_ref_normalize_password.argtypes = [C.c_char_p, C.c_size_t, u8p, C.POINTER(C.c_size_t)]
        L.lorenz_ref_subpassword.argtypes = [C.c_char_p, C.c_size_t, C.c_uint32, u8p]
        L.lorenz_ref_keymaterial.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(KeyMaterial)]
        L.lorenz_ref_apply_variant.argtypes = [C.POINTER(KeyMaterial), C.c_uint32]
        L.lorenz_ref_encrypt_stream.argtypes = [C.POINTER(KeyMaterial), C.POINTER(Params), C.c_void_p,
                                                C.c_size_t, C.c_void_p, C.c_void_p]
        L.lorenz_ref_decrypt_stream.argtypes = [C.POINTER(KeyMaterial), C.POINTER(Params), C.c_void_p,
                                                C.c_size_t, C.c_void_p, ip, C.c_void_p]
        L.lorenz_ref_num_blocks.argtypes = [C.POINTER(Params), C.c_uint64]
        L.lorenz_ref_num_blocks.restype = C.c_uint64
        L.lorenz_ref_ct_len.argtypes = [C.POINTER(Params), C.c_uint64]
        L.lorenz_ref_ct_len.restype = C.c_uint64
        L.lorenz_ref_pt_len.argtypes = [C.POINTER(Params), C.c_uint64, u64p]
        L.lorenz_ref_encrypt.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(Params), C.c_uint64, C.c_uint64,
                                         C.c_uint64, C.c_void_p, C.c_void_p, u8p, C.c_int]
        L.lorenz_ref_digit_hist.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_uint32, C.c_void_p]
        u32 = C.c_uint32
        L.lorenz_ref_autocorr.argtypes = [C.c_void_p, u32, u32, C.c_void_p]
        L.lorenz_ref_autocorr_at.argtypes = [C.c_void_p, u32, u32, u32, u32]
        L.lorenz_ref_autocorr_at.restype = C.c_double
        L.lorenz_ref_power_spectrum.argtypes = [C.c_void_p, u32, u32, C.c_void_p]
        L.lorenz_ref_power_at.argtypes = [C.c_void_p, u32, u32, u32, u32]
        L.lorenz_ref_power_at.restype = C.c_double
        L.lorenz_ref_spectral_flatness.argtypes = [C.c_void_p, u32, u32]
        L.lorenz_ref_spectral_flatness.restype = C.c_double
        L.lorenz_ref_encrypt_block.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(Params), C.c_uint64,
                                               C.c_uint64, C.c_void_p, C.c_void_p]
        L.lorenz_ref_decrypt.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(Params), C.c_uint64, C.c_uint64,
                                         C.c_uint64, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                                         C.c_void_p, C.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"oracle status {status} {msg}")
        self.status = status


def params(mode=FAST, n_it=0, dt_code=0, block_size=0, integrator=RK4, variant=0) -> Params:
    return Params(mode, n_it, dt_code, block_size, integrator, variant)


# ---------------------------------------------------------------- components
def sha256(msg: bytes) -> bytes:
    out = (C.c_uint8 * 32)()
    lib().lorenz_ref_sha256(msg, len(msg), out)
    return bytes(out)


def pack(pw: bytes):
    a = (C.c_uint64 * 3)()
    st = lib().lorenz_ref_pack(pw, len(pw), a)
    if st:
        raise OracleError(st)
    return tuple(a)


def norm_exponent(L: int) -> int:
    return lib().lorenz_ref_norm_exponent(L)


def normalize(a, L):
    aa = (C.c_uint64 * 3)(*a)
    out = (C.c_double * 3)()
    lib().lorenz_ref_normalize(aa, L, out)
    return tuple(out)


def lam(a):
    aa = (C.c_uint64 * 3)(*a)
    out = (C.c_double * 3)()
    lib().lorenz_ref_lambda(aa, out)
    return tuple(out)


def mu(a):
    aa = (C.c_uint64 * 3)(*a)
    out = (C.c_int * 3)()
    lib().lorenz_ref_mu(aa, out)
    return tuple(out)


def k_omega(pw: bytes, a):
    aa = (C.c_uint64 * 3)(*a)
    k, om, k3 = (C.c_int * 3)(), (C.c_int * 3)(), C.c_int()
    lib().lorenz_ref_k_omega(pw, len(pw), aa, k, C.byref(k3), om)
    return tuple(k), k3.value, tuple(om)


def R(alpha: float, omega: int) -> int:
    return lib().lorenz_ref_R(alpha, omega)


def theta(p: int, omega3: int) -> float:
    return lib().lorenz_ref_theta(p, omega3)


def encode(p: int, ksum: int) -> int:
    return lib().lorenz_ref_encode(p, ksum)


def decode(c: int, ksum: int) -> int:
    return lib().lorenz_ref_decode(c, ksum)


def rhs(s):
    a = (C.c_double * 3)(*s)
    f = (C.c_double * 3)()
    lib().lorenz_ref_rhs(a, f)
    return tuple(f)


def rk4_step(s, h):
    a = (C.c_double * 3)(*s)
    lib().lorenz_ref_rk4_step(a, h)
    return tuple(a)


def rk4fma_step(s, h):
    a = (C.c_double * 3)(*s)
    lib().lorenz_ref_rk4fma_step(a, h)
    return tuple(a)


def euler_step(s, h):
    a = (C.c_double * 3)(*s)
    lib().lorenz_ref_euler_step(a, h)
    return tuple(a)


def iterate(s, n, dt_code=0, integrator=RK4):
    a = (C.c_double * 3)(*s)
    lib().lorenz_ref_iterate(a, dt_code, integrator, n)
    return tuple(a)


def dt(dt_code: int) -> float:
    return lib().lorenz_ref_dt(dt_code)


def normalize_password(pw: bytes) -> bytes:
    out = (C.c_uint8 * 23)()
    n = C.c_size_t()
    st = lib().lorenz_ref_normalize_password(pw, len(pw), out, C.byref(n))
    if st:
        raise OracleError(st)
    return bytes(out)[: n.value]


def subpassword(pw: bytes, b: int) -> bytes:
    out = (C.c_uint8 * 18)()
    lib().lorenz_ref_subpassword(pw, len(pw), b, out)
    return bytes(out)


def keymaterial(pw_norm: bytes, variant: int = 0) -> KeyMaterial:
    km = KeyMaterial()
    st = lib().lorenz_ref_keymaterial(pw_norm, len(pw_norm), C.byref(km))
    if st:
        raise OracleError(st)
    lib().lorenz_ref_apply_variant(C.byref(km), variant)
    return km


def _buf(x) -> np.ndarray:
    a = np.ascontiguousarray(np.frombuffer(bytes(x), dtype=np.uint8) if isinstance(x, (bytes, bytearray)) else x,
                             dtype=np.uint8)
    return a


def encrypt_stream(km: KeyMaterial, p: bytes, prm: Params, trace=False):
    pa = _buf(p)
    c = np.zeros(len(pa) + 16, dtype=np.uint8)
    tr = np.zeros((len(pa) + 16, 3), dtype=np.float64) if trace else None
    st = lib().lorenz_ref_encrypt_stream(C.byref(km), C.byref(prm), pa.ctypes.data, len(pa), c.ctypes.data,
                                         tr.ctypes.data if trace else None)
    if st:
        raise OracleError(st)
    return (c.tobytes(), tr) if trace else c.tobytes()


def decrypt_stream(km: KeyMaterial, c: bytes, prm: Params, trace=False):
    ca = _buf(c)
    p = np.zeros(max(len(ca) - 16, 0), dtype=np.uint8)
    ok = C.c_int(0)
    tr = np.zeros((len(ca), 3), dtype=np.float64) if trace else None
    st = lib().lorenz_ref_decrypt_stream(C.byref(km), C.byref(prm), ca.ctypes.data, len(ca), p.ctypes.data,
                                         C.byref(ok), tr.ctypes.data if trace else None)
    if st:
        raise OracleError(st)
    out = (p.tobytes(), bool(ok.value))
    return out + (tr,) if trace else out


# ---------------------------------------------------------------- messages
def num_blocks(prm: Params, n: int) -> int:
    return lib().lorenz_ref_num_blocks(C.byref(prm), n)


def ct_len(prm: Params, n: int) -> int:
    return lib().lorenz_ref_ct_len(C.byref(prm), n)


def pt_len(prm: Params, clen: int) -> int:
    out = C.c_uint64()
    st = lib().lorenz_ref_pt_len(C.byref(prm), clen, C.byref(out))
    if st:
        raise OracleError(st)
    return out.value


def encrypt(pw: bytes, pt, prm: Params, b0=0, b1=None, threads=0):
    """Encrypt global blocks [b0,b1) of message pt. Returns (ct_full, tag_xor);
    bytes of ct outside the range are left zero."""
    pa = _buf(pt)
    n = len(pa)
    nb = num_blocks(prm, n)
    b1 = nb if b1 is None else b1
    ct = np.zeros(ct_len(prm, n), dtype=np.uint8)
    tag = (C.c_uint8 * 16)()
    st = lib().lorenz_ref_encrypt(pw, len(pw), C.byref(prm), n, b0, b1, pa.ctypes.data, ct.ctypes.data, tag,
                                  threads)
    if st:
        raise OracleError(st)
    return ct, bytes(tag)


def digit_hist(ic: np.ndarray, skip: int, samples: int, stride: int, dt_code=0, integrator=RK4) -> np.ndarray:
    """Fig.1 digit histograms of trajectories from ic (lanes x 3 doubles): uint64[3, 4, 128]."""
    ic = np.ascontiguousarray(ic, dtype=np.float64).reshape(-1, 3)
    hist = np.zeros((3, 4, 128), dtype=np.uint64)
    lib().lorenz_ref_digit_hist(ic.ctypes.data, ic.shape[0], skip, samples, stride, dt_code, integrator,
                                hist.ctypes.data)
    return hist


def _image(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.uint8)
    if a.ndim != 2:
        raise ValueError("expected an H x W uint8 matrix")
    return a


def autocorr(x) -> np.ndarray:
    """Fig.3: normalised circular 2-D autocorrelation r[u, v] of an H x W byte matrix (Q25)."""
    a = _image(x)
    r = np.zeros(a.shape, dtype=np.float64)
    lib().lorenz_ref_autocorr(a.ctypes.data, a.shape[0], a.shape[1], r.ctypes.data)
    return r


def autocorr_at(x, u: int, v: int) -> float:
    a = _image(x)
    return lib().lorenz_ref_autocorr_at(a.ctypes.data, a.shape[0], a.shape[1], u, v)


def power_spectrum(x) -> np.ndarray:
    """Fig.4 (g)-(i): |2-D DFT|^2 / N^2, DC-centred (Q26)."""
    a = _image(x)
    p = np.zeros(a.shape, dtype=np.float64)
    lib().lorenz_ref_power_spectrum(a.ctypes.data, a.shape[0], a.shape[1], p.ctypes.data)
    return p


def power_at(x, k: int, l: int) -> float:
    """One frequency (k, l), unshifted indices, of power_spectrum."""
    a = _image(x)
    return lib().lorenz_ref_power_at(a.ctypes.data, a.shape[0], a.shape[1], k, l)


def spectral_flatness(p) -> float:
    p = np.ascontiguousarray(p, dtype=np.float64)
    return lib().lorenz_ref_spectral_flatness(p.ctypes.data, p.shape[0], p.shape[1])


def encrypt_block(pw: bytes, n: int, b: int, blk_pt, prm: Params) -> np.ndarray:
    """Ciphertext (body + tag) of global block b of an n-byte message, from its bytes."""
    pa = _buf(blk_pt)
    ct = np.zeros(len(pa) + 16, dtype=np.uint8)
    st = lib().lorenz_ref_encrypt_block(pw, len(pw), C.byref(prm), n, b, pa.ctypes.data if len(pa) else None,
                                        ct.ctypes.data)
    if st:
        raise OracleError(st)
    return ct


def decrypt(pw: bytes, ct, prm: Params, b0=0, b1=None, threads=0, per_block=False):
    """Decrypt global blocks [b0,b1). Returns (status, pt_full, first_bad[, block_ok])."""
    ca = _buf(ct)
    n = pt_len(prm, len(ca))
    nb = num_blocks(prm, n)
    b1 = nb if b1 is None else b1
    pt = np.zeros(n, dtype=np.uint8)
    fb = C.c_int64(0)
    ok = np.zeros(max(b1 - b0, 1), dtype=np.uint8)
    st = lib().lorenz_ref_decrypt(pw, len(pw), C.byref(prm), n, b0, b1, ca.ctypes.data, pt.ctypes.data,
                                  C.byref(fb), ok.ctypes.data if per_block else None, threads)
    if st not in (OK, E_INTEGRITY):
        raise OracleError(st)
    if per_block:
        return st, pt, fb.value, ok[: b1 - b0]
    return st, pt, fb.value
