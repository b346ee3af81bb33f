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
SOURCES = ["lorenz.cu", "lorenz_io.cu"]
HEADERS = ["lorenz_device.cuh", "sha256.cuh", "stats.cuh", "analysis.cuh", "spectra.cuh",
           os.path.join("..", "..", "include", "lorenz.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-Xptxas", "-v",
              "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-shared"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(CSRC, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=CSRC)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write(r.stderr)
    build_cli()
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
    print(build(force=True, verbose=True))
