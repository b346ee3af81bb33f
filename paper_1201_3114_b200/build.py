"""Build liblorenz.so in-tree with nvcc for sm_100a (no torch JIT, no CPU fallback).

Flags: -fmad=false keeps nvcc from contracting any a*b+c into an FMA (the kernels
also use __dadd_rn/__dmul_rn, which are never contracted); -prec-div=true keeps
every '/' correctly rounded; -lineinfo maps ncu's source page to the .cuh lines.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(CSRC, "liblorenz.so")
SOURCES = ["lorenz.cu", "lorenz_io.cu", "lorenz_seg.cu", "lorenz_spectra.cu"]
HEADERS = ["lorenz_device.cuh", "sha256.cuh", "stats.cuh", "analysis.cuh", "spectra.cuh", "seg_launch.h",
           os.path.join("..", "..", "include", "lorenz.h")]
# translation units, compiled in parallel: lorenz_seg.cu once per OP (its kernel instantiations
# are the bulk of the compile time)
UNITS = [("lorenz.cu", []), ("lorenz_io.cu", []), ("lorenz_spectra.cu", [])] + [("lorenz_seg.cu", [f"-DLZ_SEG_OP={op}"]) for op in range(3)]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-Xptxas", "-v",
              "-Xcompiler", "-fPIC,-O2,-ffp-contract=off"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


STAMP = LIB + ".srchash"  # hash of the sources the library was built from (travels with it)


def source_hash() -> str:
    """SHA-256 over the library's sources, headers and flags. Content-based, so a copy of the
    tree (a GPU box's snapshot, where file times are the copy's) does not look stale."""
    import hashlib
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for f in sorted(SOURCES + HEADERS + ["lorenz_cli.cpp"]):
        h.update(f.encode())
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def stale() -> bool:
    if not (os.path.exists(LIB) and os.path.exists(STAMP) and os.path.exists(CLI)):
        return True
    with open(STAMP) as fh:
        return fh.read().strip() != source_hash()


def compile_lib(out: str, defines=()) -> str:
    """nvcc every translation unit to an object (in parallel), then link the shared library.
    Returns the compilers' stderr (ptxas -v register / spill report)."""
    import tempfile
    out = os.path.abspath(out)
    with tempfile.TemporaryDirectory(prefix="lorenz_build_") as tmp:
        procs = []
        for i, (src, extra) in enumerate(UNITS):
            obj = os.path.join(tmp, f"{i}_{src}.o")
            cmd = [nvcc()] + NVCC_FLAGS + list(defines) + extra + ["-c", "-o", obj, os.path.join(CSRC, src)]
            procs.append((obj, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                                     text=True, cwd=CSRC)))
        log = []
        for obj, cmd, p in procs:
            o, e = p.communicate()
            if p.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(cmd) + "\n" + o + e)
            log.append(e)
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o", out]
        r = subprocess.run(link + [o for o, _, _ in procs], capture_output=True, text=True, cwd=CSRC)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    return "".join(log)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    log = compile_lib(LIB)
    if verbose:
        print(log)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write(log)
    build_cli()
    with open(STAMP, "w") as f:
        f.write(source_hash() + "\n")
    return LIB


CLI = os.path.join(HERE, "bin", "lorenz")


def build_cli() -> str:
    """The `lorenz` command (csrc/lorenz_cli.cpp) linked against liblorenz.so (rpath $ORIGIN/../csrc)."""
    os.makedirs(os.path.dirname(CLI), exist_ok=True)
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", os.path.join(CSRC, "lorenz_cli.cpp"), "-L" + CSRC, "-llorenz",
           "-Wl,-rpath,$ORIGIN/../csrc", "-o", CLI]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("g++ (cli) failed:\n" + r.stdout + r.stderr)
    return CLI


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser(description="build liblorenz.so (or a tuning variant of it)")
    ap.add_argument("-D", dest="defines", action="append", default=[],
                    help="extra macro for a tuning variant, e.g. -D LZ_SEG_TRACE (needs --out)")
    ap.add_argument("--out", help="write the variant library here instead of csrc/liblorenz.so")
    a = ap.parse_args()
    if a.out:
        compile_lib(a.out, ["-D" + d for d in a.defines])
        print(a.out)
    else:
        assert not a.defines, "variants (-D) go to --out, never over the product library"
        print(build(force=True, verbose=True))
