"""SASS invariants of the built liblorenz.so (CPU only: cuobjdump, no GPU).

The cipher's bytes depend on every FP64 rounding (§3.1: xi = 52, IEEE double; the
north star's bit-exactness), so the integration loops must execute exactly the operations of
DESIGN.md §2 in RN with no contraction into FMA:

  RK4 (canonical):   43 DADD + 32 DMUL + 0 DFMA per step, + 3 loop instructions;
  Euler (NEXT-1):    28 DADD + 32 DMUL per 4-step unrolled iteration, 7 + 8 for the remainder;
  RK4-FMA (NEXT-3):  7 DADD + 8 DMUL + 30 DFMA per step (the FMA sites of DESIGN.md §2b).

and nothing else inside a loop but its counter / branch and the handling of its constants
(uniform-register moves / reloads).

Checked for every innermost FP64 loop of every chain-kernel instantiation (wave kernel: its
loop copies; balanced kernel: the first-piece, whole-unit and last-piece copies), plus no local
memory. A negative control compiles the same RK4 step written with plain operators: with
nvcc's default -fmad=true the checker must see DFMA (contraction changes the ciphertext),
with -fmad=false it must see the canonical mix.
"""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import sass_stats  # noqa: E402

from paper_1201_3114_b200 import build as B  # noqa: E402

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists(
    "/usr/local/cuda/bin/cuobjdump"), reason="cuobjdump not installed")

RK4, EULER, RK4_FMA = 0, 1, 2
# FP64 mix of each integration loop shape. Besides it a loop may only carry its counter, compare and
# branch and the handling of its constants — UMOV (beta into a uniform register, RK4 / Euler take
# sigma, rho, beta as compile-time operands) and LDCU (the balanced kernel's FMA loop reloads its six
# constants into uniform registers every step, off the FP64 pipe) — at most 6 of them.
EXPECTED = {
    RK4: [{"DADD": 43, "DMUL": 32, "DFMA": 0}],
    EULER: [{"DADD": 28, "DMUL": 32, "DFMA": 0}, {"DADD": 7, "DMUL": 8, "DFMA": 0}],
    RK4_FMA: [{"DADD": 7, "DMUL": 8, "DFMA": 30}],
}
ALLOWED_OTHER = {"IADD3", "VIADD", "UIADD3", "IMAD", "MOV", "ISETP", "UISETP", "BRA", "UMOV", "LDCU"}


def fp64(lp):
    return {k: lp[k] for k in ("DADD", "DMUL", "DFMA")}


@pytest.fixture(scope="module")
def loops():
    so = B.build()  # no-op when the library is current
    os.environ["PATH"] = os.environ.get("PATH", "") + ":/usr/local/cuda/bin"
    return sass_stats.chain_kernel_loops(so)


def test_every_chain_kernel_is_instantiated(loops):
    kinds = {(k[0], k[2]) for k in loops}
    for kern in ("lorenz_chain_kernel", "lorenz_chain_seg_kernel"):
        for integ in (RK4, EULER, RK4_FMA):
            assert (kern, integ) in kinds
    assert len(loops) >= 48


def test_integration_loops_exact_op_mix(loops):
    for (kern, op, integ, cta), (found, local) in loops.items():
        want = EXPECTED[integ]
        assert found, (kern, op, integ, cta, "no integration loop found")
        for lp in found:
            assert fp64(lp) in want, (kern, op, integ, cta, lp)
            assert lp["other"] <= 6 and set(lp["other_ops"]) <= ALLOWED_OTHER, (kern, op, integ, cta, lp)
        # every expected loop shape is present, in every inlined copy of the character loop
        copies = 3 if kern == "lorenz_chain_seg_kernel" else 1
        for w in want:
            assert sum(fp64(lp) == w for lp in found) >= copies, (kern, op, integ, cta, w, found)
        assert local == 0, (kern, op, integ, cta, "local memory")


RK4_PLAIN = r"""
struct S { double x, y, z; };
__global__ void rk4_plain(S* s, const double* c, int n) {
  double x = s[threadIdx.x].x, y = s[threadIdx.x].y, z = s[threadIdx.x].z;
  const double sg = c[0], r = c[1], b = c[2], h = c[3], h2 = c[4], h6 = c[5];
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    double k1x = sg * (y - x), k1y = (r * x - y) - x * z, k1z = x * y - b * z;
    double ax = x + h2 * k1x, ay = y + h2 * k1y, az = z + h2 * k1z;
    double k2x = sg * (ay - ax), k2y = (r * ax - ay) - ax * az, k2z = ax * ay - b * az;
    double bx = x + h2 * k2x, by = y + h2 * k2y, bz = z + h2 * k2z;
    double k3x = sg * (by - bx), k3y = (r * bx - by) - bx * bz, k3z = bx * by - b * bz;
    double cx = x + h * k3x, cy = y + h * k3y, cz = z + h * k3z;
    double k4x = sg * (cy - cx), k4y = (r * cx - cy) - cx * cz, k4z = cx * cy - b * cz;
    x = x + h6 * ((((k1x + k2x) + k2x) + k3x) + k3x + k4x);
    y = y + h6 * ((((k1y + k2y) + k2y) + k3y) + k3y + k4y);
    z = z + h6 * ((((k1z + k2z) + k2z) + k3z) + k3z + k4z);
  }
  s[threadIdx.x].x = x; s[threadIdx.x].y = y; s[threadIdx.x].z = z;
}
"""


@pytest.mark.parametrize("fmad,contracted", [("true", True), ("false", False)])
def test_negative_control_contraction(tmp_path, fmad, contracted):
    src = tmp_path / "rk4_plain.cu"
    src.write_text(RK4_PLAIN)
    cubin = tmp_path / "rk4_plain.cubin"
    subprocess.run([B.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", f"-fmad={fmad}", "-cubin",
                    "-o", str(cubin), str(src)], check=True)
    sass = subprocess.run(["cuobjdump", "-sass", str(cubin)], capture_output=True, text=True, check=True).stdout
    (name, body), = list(sass_stats.kernels(sass))
    found = sass_stats.innermost_fp64_loops(sass_stats.parse(body))
    assert found
    if contracted:
        assert all(lp["DFMA"] > 0 for lp in found), found
        assert all(fp64(lp) not in EXPECTED[RK4] for lp in found)
    else:
        assert all(fp64(lp) in EXPECTED[RK4] and lp["other"] == 3 for lp in found), found  # counter, compare, branch
