"""Pins for the oracle's Lorenz dynamics (§3.1 Eq.1; RK4 per the north star).

Pinned to: exact-rational RK4 (Python fractions, correctly rounded once),
the Lorenz fixed points (0,0,0) and (±sqrt(beta(rho-1)), ±sqrt(beta(rho-1)), rho-1),
a 30-digit Taylor-series solution (mpmath.odefun) for the order-4 convergence,
SPEC's hand-evaluated Euler step, and the attractor's known boundedness/sensitivity.
"""
import json
import math
import os
import random
import struct
from fractions import Fraction

import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
PAPER = json.load(open(os.path.join(GOLD, "paper_constants.json")))

SIG = Fraction(PAPER["sigma"]["value"])
RHO = Fraction(PAPER["rho"]["value"])
BETA = Fraction(PAPER["beta"]["num"], PAPER["beta"]["den"])


def f_exact(s):
    x, y, z = s
    return (SIG * (y - x), RHO * x - y - x * z, x * y - BETA * z)


def rk4_exact(s, h):
    """Classical RK4 (Kutta 1901) in exact rational arithmetic."""
    k1 = f_exact(s)
    k2 = f_exact([s[i] + h / 2 * k1[i] for i in range(3)])
    k3 = f_exact([s[i] + h / 2 * k2[i] for i in range(3)])
    k4 = f_exact([s[i] + h * k3[i] for i in range(3)])
    return [s[i] + h / 6 * (k1[i] + 2 * k2[i] + 2 * k3[i] + k4[i]) for i in range(3)]


def test_dt_table_inside_paper_range(ref):
    for code in range(4):
        assert 0 < ref.dt(code) <= PAPER["dt_max"]["value"]
    assert ref.dt(0) == 0.01


def test_rhs_exact_on_integers(ref):
    """On small integers every RHS operation is exact except beta*z."""
    for s in [(1.0, 2.0, 3.0), (-4.0, 7.0, 30.0), (0.5, -0.25, 12.0)]:
        f = ref.rhs(s)
        fe = f_exact([Fraction(v) for v in s])
        assert f[0] == float(fe[0]) and f[1] == float(fe[1])
        assert abs(f[2] - float(fe[2])) <= 2 * math.ulp(abs(float(fe[2])) + 1)


def test_rk4_one_step_equals_exact_rational_map(ref):
    """from (1,1,1), h = 0.01, the canonical-order RK4 step equals the
    correctly rounded exact-rational RK4 map (beta = 8/3 exactly, h = double 0.01)."""
    h = 0.01
    got = ref.rk4_step((1.0, 1.0, 1.0), h)
    want = [float(v) for v in rk4_exact([Fraction(1)] * 3, Fraction(h))]
    assert list(got) == want


def test_rk4_step_near_exact_random_states(ref):
    rng = random.Random(8)
    for _ in range(200):
        s = (rng.uniform(-20, 20), rng.uniform(-25, 25), rng.uniform(0, 50))
        got = ref.rk4_step(s, 0.01)
        want = rk4_exact([Fraction(v) for v in s], Fraction(0.01))
        for g, w in zip(got, want):
            assert abs(Fraction(g) - w) < Fraction(1, 10 ** 12)


def test_origin_is_fixed_exactly(ref):
    assert ref.iterate((0.0, 0.0, 0.0), 3000) == (0.0, 0.0, 0.0)
    assert ref.iterate((0.0, 0.0, 0.0), 3000, integrator=ref.EULER) == (0.0, 0.0, 0.0)


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_c_plus_minus_stationary(ref, sign):
    """C± = (±sqrt(beta(rho-1)), ±sqrt(beta(rho-1)), rho-1) are equilibria of Eq.1's
    ODE; RK4 keeps them (bit-exactly in the canonical order)."""
    q = math.sqrt(float(BETA * (RHO - 1)))
    c = (sign * q, sign * q, float(RHO - 1))
    f = ref.rhs(c)
    assert max(abs(v) for v in f) < 1e-12
    out = ref.iterate(c, 3000)
    assert max(abs(out[i] - c[i]) for i in range(3)) <= 1e-12
    assert out == c  # canonical order: bit-exact


def test_rk4_order_four_against_taylor_series(ref):
    """Global error at T=0.1 from (1,1,1) vs a 30-digit Taylor solution; halving h
    must divide the error by ~2^4 = 16 (9.5e-6, 6.0e-7, ratio 15.8)."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 30
    sol = mpmath.odefun(lambda t, v: [10 * (v[1] - v[0]), 28 * v[0] - v[1] - v[0] * v[2],
                                      v[0] * v[1] - mpmath.mpf(8) / 3 * v[2]], 0, [1, 1, 1])
    exact = [float(v) for v in sol(mpmath.mpf("0.1"))]
    e1 = max(abs(a - b) for a, b in zip(ref.iterate((1.0, 1.0, 1.0), 10, dt_code=0), exact))
    e2 = max(abs(a - b) for a, b in zip(ref.iterate((1.0, 1.0, 1.0), 20, dt_code=1), exact))
    assert e1 < 2e-5
    assert 12.0 <= e1 / e2 <= 20.0


def test_euler_spec_examples(ref):
    for ex in SPEC["euler_step"]:
        got = ref.euler_step(tuple(ex["s"]), ex["h"])
        for g, w in zip(got, ex["out"]):
            assert math.isclose(g, w, rel_tol=ex.get("rel_tol", 0.0), abs_tol=0.0) or g == w, ex["cite"]


def test_literal_eq1_collapses_to_origin():
    """Reading Q2: Eq.1 as printed is contracting, so the paper's
    'chaotic sequences' claim needs the standard RHS."""
    x, y, z = 1.0, 1.0, 1.0
    dt, s, r, b = 0.01, 10.0, 28.0, 8.0 / 3.0
    for _ in range(200):
        x, y, z = ((1 - s) * x + s * y) * dt, (r * x - 2 * y - x * z) * dt, (x * y + (1 - b) * z) * dt
    assert max(abs(x), abs(y), abs(z)) < 1e-100


def test_trajectories_stay_bounded(ref):
    """From the corners of the lambda box widened by a' <= 1 the
    RK4 trajectory stays in the guard box of reading Q18."""
    lo, hi = PAPER["lambda_ranges"]["lo"], PAPER["lambda_ranges"]["hi"]
    for cx in (lo[0], hi[0] + 1):
        for cy in (lo[1], hi[1] + 1):
            for cz in (lo[2], hi[2] + 1):
                s = (cx, cy, cz)
                for _ in range(30):
                    s = ref.iterate(s, 100)
                    assert abs(s[0]) <= 100 and abs(s[1]) <= 100 and -50 <= s[2] <= 150


def test_sensitive_dependence(ref):
    """Chaos: a 1e-10 perturbation of x grows past distance 1 within 10,000 RK4
    steps at h = 0.01 (SPEC's 2000-step bound is recalibrated)."""
    rng = random.Random(31)
    lo, hi = PAPER["lambda_ranges"]["lo"], PAPER["lambda_ranges"]["hi"]
    for _ in range(100):
        s = tuple(rng.uniform(lo[i], hi[i]) for i in range(3))
        t = (s[0] + 1e-10, s[1], s[2])
        crossed = False
        for _ in range(100):
            s, t = ref.iterate(s, 100), ref.iterate(t, 100)
            if math.dist(s, t) > 1.0:
                crossed = True
                break
        assert crossed


def test_golden_trajectory_file(ref):
    """Regression fixture written by tools/make_golden.py (oracle only); its
    first state is pinned independently by the exact-rational test above."""
    path = os.path.join(GOLD, "rk4_trajectory_h001.txt")
    rows = [ln.split() for ln in open(path) if ln.strip() and not ln.startswith("#")]
    s = (1.0, 1.0, 1.0)
    for i, row in enumerate(rows):
        s = ref.rk4_step(s, 0.01)
        assert [struct.pack(">d", v).hex() for v in s] == row, i
