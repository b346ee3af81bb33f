"""Thin Python binding of include/lorenz.h (liblorenz.so): same names, marshalling only.

Every step of the cipher runs in the CUDA kernels of ``csrc/``; this module only
turns Python objects (bytes, torch tensors, streams) into the C ABI's pointers and
sizes. There is no CPU fallback: if liblorenz.so is missing, importing
:func:`lib` raises.

Device buffers are torch uint8 CUDA tensors (or raw device addresses as ints);
streams default to torch's current stream.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LORENZ_LIB") or os.path.join(HERE, "csrc", "liblorenz.so")  # override: tuning runs

OK, E_INTEGRITY, E_ARG, E_PASSWORD, E_LENGTH, E_DIVERGENCE, E_CUDA = range(7)
STRONG, FAST = 0, 1
RK4, EULER, RK4_FMA = 0, 1, 2
TAG_BYTES = 16
KEY_BYTES = 384

EXPORTS = ["lorenz_abi_version", "lorenz_last_error", "lorenz_status_string", "lorenz_keysetup",
           "lorenz_key_params", "lorenz_num_blocks", "lorenz_ct_len", "lorenz_pt_len",
           "lorenz_encrypt", "lorenz_decrypt", "lorenz_verify", "lorenz_result_init_async",
           "lorenz_encrypt_async", "lorenz_decrypt_async", "lorenz_verify_async",
           "lorenz_encrypt_batch", "lorenz_encrypt_host", "lorenz_decrypt_host",
           "lorenz_compare_spans", "lorenz_histograms", "lorenz_envelope_write", "lorenz_envelope_read",
           "lorenz_encrypt_file", "lorenz_decrypt_file", "lorenz_digit_histograms",
           "lorenz_autocorrelation", "lorenz_power_spectrum", "lorenz_encrypt_ragged", "lorenz_decrypt_ragged",
           "lorenz_launch_plan", "lorenz_set_tuning"]
E_IO, E_FORMAT = 7, 8
ENVELOPE_BYTES = 24


class lorenz_span(C.Structure):
    _fields_ = [("a_off", C.c_uint64), ("b_off", C.c_uint64), ("len", C.c_uint64)]


class lorenz_params(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("n_it", C.c_uint32), ("dt_code", C.c_uint32),
                ("block_size", C.c_uint32), ("integrator", C.c_uint32), ("variant", C.c_uint32)]


V_LITERAL, V_CYCLIC, V_DISTINCT_K = 1, 2, 4  # NEXT-4 Step-3 reading variants


class lorenz_key(C.Structure):
    _fields_ = [("opaque", C.c_uint8 * KEY_BYTES)]


class lorenz_result(C.Structure):
    _fields_ = [("tag_xor", C.c_uint8 * 16), ("first_bad", C.c_uint64), ("status", C.c_uint32),
                ("reserved", C.c_uint32)]


class LorenzError(RuntimeError):
    def __init__(self, status: int, where: str = ""):
        msg = lib().lorenz_status_string(status).decode()
        if status == E_CUDA:
            msg += ": " + lib().lorenz_last_error().decode()
        super().__init__(f"{where}: {msg} (status {status})")
        self.status = status


_lib = None


def lib():
    """Load liblorenz.so (fails loudly when the CUDA library was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        vp, u64, u32, sz = C.c_void_p, C.c_uint64, C.c_uint32, C.c_size_t
        kp = C.POINTER(lorenz_key)
        L.lorenz_abi_version.restype = C.c_int
        L.lorenz_last_error.restype = C.c_char_p
        L.lorenz_status_string.restype = C.c_char_p
        L.lorenz_status_string.argtypes = [C.c_int]
        L.lorenz_keysetup.argtypes = [C.c_char_p, sz, C.POINTER(lorenz_params), kp]
        L.lorenz_key_params.argtypes = [kp, C.POINTER(lorenz_params)]
        L.lorenz_num_blocks.argtypes = [kp, u64]
        L.lorenz_num_blocks.restype = u64
        L.lorenz_ct_len.argtypes = [kp, u64]
        L.lorenz_ct_len.restype = u64
        L.lorenz_pt_len.argtypes = [kp, u64, C.POINTER(u64)]
        L.lorenz_launch_plan.argtypes = [kp, u64, u64, u64, C.POINTER(lorenz_plan)]
        L.lorenz_set_tuning.argtypes = [C.POINTER(lorenz_tuning)]
        L.lorenz_encrypt.argtypes = [kp, u64, u64, u64, vp, vp, vp, vp]
        L.lorenz_decrypt.argtypes = [kp, u64, u64, u64, vp, vp, C.POINTER(C.c_int64), vp, vp]
        L.lorenz_verify.argtypes = [kp, u64, u64, u64, vp, C.POINTER(C.c_int64), vp, vp]
        L.lorenz_result_init_async.argtypes = [vp, vp]
        L.lorenz_encrypt_async.argtypes = [kp, u64, u64, u64, vp, vp, vp, vp]
        L.lorenz_decrypt_async.argtypes = [kp, u64, u64, u64, vp, vp, vp, vp, vp]
        L.lorenz_verify_async.argtypes = [kp, u64, u64, u64, vp, vp, vp]
        L.lorenz_encrypt_batch.argtypes = [kp, u32, u64, vp, vp, vp, vp]
        L.lorenz_encrypt_ragged.argtypes = [kp, u32, vp, vp, vp, vp, vp, vp, vp]
        L.lorenz_decrypt_ragged.argtypes = [kp, u32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.lorenz_compare_spans.argtypes = [vp, vp, C.POINTER(lorenz_span), u32, vp, vp]
        L.lorenz_histograms.argtypes = [vp, C.POINTER(lorenz_span), u32, vp, vp]
        L.lorenz_digit_histograms.argtypes = [vp, u64, u32, u32, u32, u32, u32, vp, vp]
        L.lorenz_autocorrelation.argtypes = [vp, u32, u32, vp, vp]
        L.lorenz_power_spectrum.argtypes = [vp, u32, u32, vp, vp, vp]
        L.lorenz_envelope_write.argtypes = [kp, u64, vp]
        L.lorenz_envelope_read.argtypes = [C.c_char_p, sz, C.POINTER(lorenz_params), C.POINTER(u64),
                                           C.POINTER(u64)]
        L.lorenz_encrypt_file.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, sz, C.POINTER(lorenz_params),
                                          u64, vp]
        L.lorenz_decrypt_file.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, sz, u64, C.POINTER(C.c_int64)]
        L.lorenz_encrypt_host.argtypes = [kp, u64, u64, u64, vp, vp, vp, u32]
        L.lorenz_decrypt_host.argtypes = [kp, u64, u64, u64, vp, vp, C.POINTER(C.c_int64), u32]
        for name in EXPORTS:
            if name not in ("lorenz_abi_version", "lorenz_last_error", "lorenz_status_string",
                            "lorenz_num_blocks", "lorenz_ct_len"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != OK:
        raise LorenzError(st, where)


def _ptr(x) -> int | None:
    """Device address of a torch tensor (must be contiguous) or a raw int; None -> NULL."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if not x.is_contiguous():
        raise ValueError("buffer must be contiguous")
    return x.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


@dataclass
class Key:
    """A lorenz_key (384-byte POD) plus its effective params."""
    raw: lorenz_key

    @property
    def params(self) -> lorenz_params:
        p = lorenz_params()
        _check(lib().lorenz_key_params(C.byref(self.raw), C.byref(p)), "lorenz_key_params")
        return p

    def num_blocks(self, n: int) -> int:
        return lorenz_num_blocks(self, n)

    def ct_len(self, n: int) -> int:
        return lorenz_ct_len(self, n)

    @property
    def block_size(self) -> int:
        return self.params.block_size


def lorenz_keysetup(pw: bytes, mode: int = FAST, n_it: int = 0, dt_code: int = 0, block_size: int = 0,
                    integrator: int = RK4, variant: int = 0) -> Key:
    k = lorenz_key()
    p = lorenz_params(mode, n_it, dt_code, block_size, integrator, variant)
    _check(lib().lorenz_keysetup(bytes(pw), len(pw), C.byref(p), C.byref(k)), "lorenz_keysetup")
    return Key(k)


class lorenz_plan(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("cta", C.c_uint32), ("grid", C.c_uint64), ("lanes", C.c_uint64),
                ("slots", C.c_uint64), ("chunks_per_slot", C.c_uint64), ("chunks_skew", C.c_uint64)]


def lorenz_launch_plan(key: Key, n: int, b0: int, b1: int) -> dict:
    """The chain kernel's launch plan for blocks [b0, b1) (host only): kind 'wave' or 'balanced',
    CTA size, grid, lanes, and for the balanced kernel its warp slots and chunks per slot."""
    p = lorenz_plan()
    _check(lib().lorenz_launch_plan(C.byref(key.raw), n, b0, b1, C.byref(p)), "lorenz_launch_plan")
    return {"kind": ("wave", "balanced")[p.kind], "cta": p.cta, "grid": p.grid, "lanes": p.lanes,
            "slots": p.slots, "chunks_per_slot": p.chunks_per_slot, "chunks_skew": p.chunks_skew}


class lorenz_tuning(C.Structure):
    _fields_ = [("schedule", C.c_uint32), ("seg_slots", C.c_uint32), ("seg_skew", C.c_int32), ("cta", C.c_uint32)]


SCHED_AUTO, SCHED_WAVE, SCHED_BALANCED = 0, 1, 2


def lorenz_set_tuning(schedule: int = SCHED_AUTO, seg_slots: int = 0, seg_skew: int = -1, cta: int = 0,
                      reset: bool = False):
    """Process-wide launch-plan overrides for tests and tuning (lorenz.h); reset=True restores
    the defaults."""
    t = None if reset else C.byref(lorenz_tuning(schedule, seg_slots, seg_skew, cta))
    _check(lib().lorenz_set_tuning(t), "lorenz_set_tuning")


class tuning:
    """Context manager over lorenz_set_tuning: `with L.tuning(schedule=L.SCHED_BALANCED, seg_slots=3): ...`
    restores the defaults on exit."""

    def __init__(self, **kw):
        self.kw = kw

    def __enter__(self):
        lorenz_set_tuning(**self.kw)
        return self

    def __exit__(self, *exc):
        lorenz_set_tuning(reset=True)


def lorenz_num_blocks(key: Key, n: int) -> int:
    return lib().lorenz_num_blocks(C.byref(key.raw), n)


def lorenz_ct_len(key: Key, n: int) -> int:
    return lib().lorenz_ct_len(C.byref(key.raw), n)


def lorenz_pt_len(key: Key, ct_len: int) -> int:
    out = C.c_uint64()
    _check(lib().lorenz_pt_len(C.byref(key.raw), ct_len, C.byref(out)), "lorenz_pt_len")
    return out.value


def lorenz_encrypt(key: Key, n: int, b0: int, b1: int, pt, ct, stream=None) -> bytes:
    """Encrypt global blocks [b0,b1); pt/ct are the slice starts. Returns the tag XOR."""
    tag = (C.c_uint8 * 16)()
    _check(lib().lorenz_encrypt(C.byref(key.raw), n, b0, b1, _ptr(pt), _ptr(ct), tag, _stream(stream)),
           "lorenz_encrypt")
    return bytes(tag)


def lorenz_decrypt(key: Key, n: int, b0: int, b1: int, ct, pt, block_ok=None, stream=None,
                   raise_on_integrity: bool = False):
    """Returns (status, first_bad_block): status OK or E_INTEGRITY (others raise)."""
    fb = C.c_int64(-1)
    st = lib().lorenz_decrypt(C.byref(key.raw), n, b0, b1, _ptr(ct), _ptr(pt), C.byref(fb), _ptr(block_ok),
                              _stream(stream))
    if st != OK and (st != E_INTEGRITY or raise_on_integrity):
        raise LorenzError(st, "lorenz_decrypt")
    return st, fb.value


def lorenz_verify(key: Key, n: int, b0: int, b1: int, ct, stream=None):
    """Returns (status, first_bad_block, tag_xor)."""
    fb = C.c_int64(-1)
    tag = (C.c_uint8 * 16)()
    st = lib().lorenz_verify(C.byref(key.raw), n, b0, b1, _ptr(ct), C.byref(fb), tag, _stream(stream))
    if st not in (OK, E_INTEGRITY):
        raise LorenzError(st, "lorenz_verify")
    return st, fb.value, bytes(tag)


def lorenz_result_init_async(res, stream=None):
    _check(lib().lorenz_result_init_async(_ptr(res), _stream(stream)), "lorenz_result_init_async")


def lorenz_encrypt_async(key: Key, n: int, b0: int, b1: int, pt, ct, res, stream=None):
    _check(lib().lorenz_encrypt_async(C.byref(key.raw), n, b0, b1, _ptr(pt), _ptr(ct), _ptr(res),
                                      _stream(stream)), "lorenz_encrypt_async")


def lorenz_decrypt_async(key: Key, n: int, b0: int, b1: int, ct, pt, res, block_ok=None, stream=None):
    _check(lib().lorenz_decrypt_async(C.byref(key.raw), n, b0, b1, _ptr(ct), _ptr(pt), _ptr(block_ok),
                                      _ptr(res), _stream(stream)), "lorenz_decrypt_async")


def lorenz_verify_async(key: Key, n: int, b0: int, b1: int, ct, res, stream=None):
    _check(lib().lorenz_verify_async(C.byref(key.raw), n, b0, b1, _ptr(ct), _ptr(res), _stream(stream)),
           "lorenz_verify_async")


def lorenz_encrypt_batch(keys: list[Key], n: int, pts, cts, tags, stream=None):
    arr = (lorenz_key * len(keys))(*[k.raw for k in keys])
    _check(lib().lorenz_encrypt_batch(arr, len(keys), n, _ptr(pts), _ptr(cts), _ptr(tags), _stream(stream)),
           "lorenz_encrypt_batch")


def _u64(xs):
    import numpy as np
    return np.ascontiguousarray(np.asarray(xs, dtype=np.uint64))


def lorenz_encrypt_ragged(keys: list[Key], n, pt_off, ct_off, pts, cts, tags, stream=None):
    """Ragged batch: message s (n[s] bytes, keys[s]) at pts + pt_off[s] -> cts + ct_off[s]; tags
    device uint8[16 * len(keys)]. n / offsets: host sequences (offsets multiples of 16)."""
    arr = (lorenz_key * len(keys))(*[k.raw for k in keys])
    nn, po, co = _u64(n), _u64(pt_off), _u64(ct_off)
    _check(lib().lorenz_encrypt_ragged(arr, len(keys), nn.ctypes.data, po.ctypes.data, co.ctypes.data, _ptr(pts),
                                       _ptr(cts), _ptr(tags), _stream(stream)), "lorenz_encrypt_ragged")


def lorenz_decrypt_ragged(keys: list[Key], n, ct_off, pt_off, cts, pts, tags, stream=None):
    """Returns (status, first_bad: list of per-message lowest failing block or -1)."""
    import numpy as np
    arr = (lorenz_key * len(keys))(*[k.raw for k in keys])
    nn, co, po = _u64(n), _u64(ct_off), _u64(pt_off)
    fb = np.full(len(keys), -1, dtype=np.int64)
    st = lib().lorenz_decrypt_ragged(arr, len(keys), nn.ctypes.data, co.ctypes.data, po.ctypes.data, _ptr(cts),
                                     _ptr(pts), _ptr(tags), fb.ctypes.data, _stream(stream))
    if st not in (OK, E_INTEGRITY):
        raise LorenzError(st, "lorenz_decrypt_ragged")
    return st, fb.tolist()


def _spans(spans) -> tuple:
    """spans: (count, 3) uint64 numpy array (same layout as lorenz_span) or a list of triples."""
    import numpy as np
    arr = np.ascontiguousarray(np.asarray(spans, dtype=np.uint64).reshape(-1, 3))
    return arr.ctypes.data_as(C.POINTER(lorenz_span)), arr.shape[0], arr


def lorenz_compare_spans(a, b, spans, out, stream=None):
    """spans: list of (a_off, b_off, len); out: device uint64[3*len(spans)] (bits, bytes, equal-LSB)."""
    arr, cnt, _keep = _spans(spans)
    _check(lib().lorenz_compare_spans(_ptr(a), _ptr(b), arr, cnt, _ptr(out), _stream(stream)),
           "lorenz_compare_spans")


def lorenz_histograms(a, spans, hist, stream=None):
    """spans: list of (a_off, _, len); hist: device uint64[256*len(spans)]."""
    arr, cnt, _keep = _spans(spans)
    _check(lib().lorenz_histograms(_ptr(a), arr, cnt, _ptr(hist), _stream(stream)), "lorenz_histograms")


def lorenz_digit_histograms(ic, lanes: int, skip: int, samples: int, stride: int, hist, dt_code: int = 0,
                            integrator: int = RK4, stream=None):
    """Fig.1 digit histograms (NEXT-4): ic device float64 (lanes x 3), hist device int64[3*4*128]."""
    _check(lib().lorenz_digit_histograms(_ptr(ic), lanes, skip, samples, stride, dt_code, integrator, _ptr(hist),
                                         _stream(stream)), "lorenz_digit_histograms")


def lorenz_autocorrelation(x, r, stream=None):
    """Fig.3 (NEXT-4): x device uint8 (H, W), r device float64 (H, W) <- normalised circular 2-D
    autocorrelation, lag (0, 0) at r[0, 0]. H, W powers of two in [2, 4096]."""
    h, w = x.shape
    _check(lib().lorenz_autocorrelation(_ptr(x), h, w, _ptr(r), _stream(stream)), "lorenz_autocorrelation")


def lorenz_power_spectrum(x, power, flatness=None, stream=None):
    """Fig.4 (NEXT-4): power device float64 (H, W) <- |DFT2(x)|^2 / (HW)^2, DC-centred;
    flatness (device float64[1], optional) <- geometric / arithmetic mean of the non-DC bins."""
    h, w = x.shape
    _check(lib().lorenz_power_spectrum(_ptr(x), h, w, _ptr(power), _ptr(flatness), _stream(stream)),
           "lorenz_power_spectrum")


def lorenz_envelope_write(key: Key, n: int) -> bytes:
    hdr = (C.c_uint8 * ENVELOPE_BYTES)()
    _check(lib().lorenz_envelope_write(C.byref(key.raw), n, hdr), "lorenz_envelope_write")
    return bytes(hdr)


def lorenz_envelope_read(hdr: bytes):
    """Returns (params, payload_len, ct_len)."""
    p, n, ctl = lorenz_params(), C.c_uint64(), C.c_uint64()
    _check(lib().lorenz_envelope_read(bytes(hdr), len(hdr), C.byref(p), C.byref(n), C.byref(ctl)),
           "lorenz_envelope_read")
    return p, n.value, ctl.value


def lorenz_encrypt_file(in_path: str, out_path: str, pw: bytes, mode: int = FAST, n_it: int = 0,
                        dt_code: int = 0, block_size: int = 0, integrator: int = RK4, chunk_bytes: int = 0,
                        variant: int = 0) -> bytes:
    p = lorenz_params(mode, n_it, dt_code, block_size, integrator, variant)
    tag = (C.c_uint8 * 16)()
    _check(lib().lorenz_encrypt_file(os.fsencode(in_path), os.fsencode(out_path), bytes(pw), len(pw), C.byref(p),
                                     chunk_bytes, tag), "lorenz_encrypt_file")
    return bytes(tag)


def lorenz_decrypt_file(in_path: str, out_path: str, pw: bytes, chunk_bytes: int = 0):
    """Returns (status, first_bad_block); E_INTEGRITY leaves no output file. Other errors raise."""
    fb = C.c_int64(-1)
    st = lib().lorenz_decrypt_file(os.fsencode(in_path), os.fsencode(out_path), bytes(pw), len(pw), chunk_bytes,
                                   C.byref(fb))
    if st not in (OK, E_INTEGRITY):
        raise LorenzError(st, "lorenz_decrypt_file")
    return st, fb.value


def _host_ptr(buf) -> int | None:
    if buf is None or isinstance(buf, int):
        return buf
    if hasattr(buf, "data_ptr"):
        if buf.is_cuda:
            raise ValueError("host buffer expected")
        return buf.data_ptr()
    import numpy as np
    if not isinstance(buf, np.ndarray) or not buf.flags.c_contiguous:
        raise TypeError("pass a contiguous numpy array, a CPU torch tensor, or an address")
    return buf.ctypes.data if buf.size else None


def lorenz_encrypt_host(key: Key, n: int, b0: int, b1: int, pt_host, ct_host, n_chunks: int = 0) -> bytes:
    """End to end from host slices (pinned for overlap). Returns the tag XOR of [b0,b1)."""
    tag = (C.c_uint8 * 16)()
    _check(lib().lorenz_encrypt_host(C.byref(key.raw), n, b0, b1, _host_ptr(pt_host), _host_ptr(ct_host), tag,
                                     n_chunks), "lorenz_encrypt_host")
    return bytes(tag)


def lorenz_decrypt_host(key: Key, n: int, b0: int, b1: int, ct_host, pt_host, n_chunks: int = 0):
    """Returns (status, first_bad_block); the host plaintext slice is zeroed on failure."""
    fb = C.c_int64(-1)
    st = lib().lorenz_decrypt_host(C.byref(key.raw), n, b0, b1, _host_ptr(ct_host), _host_ptr(pt_host),
                                   C.byref(fb), n_chunks)
    if st not in (OK, E_INTEGRITY):
        raise LorenzError(st, "lorenz_decrypt_host")
    return st, fb.value


# ---------------------------------------------------------------- conveniences over whole messages
def encrypt(key: Key, pt, stream=None):
    """Encrypt a whole message held in a CUDA uint8 tensor. Returns (ct tensor, tag bytes)."""
    import torch
    n = pt.numel()
    ct = torch.empty(lorenz_ct_len(key, n), dtype=torch.uint8, device=pt.device)
    tag = lorenz_encrypt(key, n, 0, lorenz_num_blocks(key, n), pt if n else None, ct, stream)
    return ct, tag


def decrypt(key: Key, ct, stream=None):
    """Decrypt a whole ciphertext (CUDA uint8 tensor). Returns (pt tensor, status, first_bad)."""
    import torch
    n = lorenz_pt_len(key, ct.numel())
    pt = torch.empty(max(n, 1), dtype=torch.uint8, device=ct.device)
    st, fb = lorenz_decrypt(key, n, 0, lorenz_num_blocks(key, n), ct, pt if n else None, stream=stream)
    return pt[:n], st, fb
