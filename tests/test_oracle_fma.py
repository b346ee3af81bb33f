"""Pins for the oracle's FMA-formulated RK4 (NEXT-3).

The FMA form is a different cipher definition (fewer roundings); it is pinned like the
canonical form: to the exact-rational RK4 map, the fixed points, order-4 convergence
against a Taylor solution, and bit-exact agreement with an independent Python reading
whose fma is computed exactly with fractions.
"""
import math
import random
from fractions import Fraction

import pytest

import pyref
from test_oracle_dynamics import BETA, RHO, rk4_exact


def test_one_step_within_an_ulp_or_two_of_exact(ref):
    got = ref.rk4fma_step((1.0, 1.0, 1.0), 0.01)
    want = rk4_exact([Fraction(1)] * 3, Fraction(0.01))
    for g, w in zip(got, want):
        assert abs(Fraction(g) - w) <= 2 * Fraction(math.ulp(float(w)))


def test_random_states_near_exact_and_differs_from_unfused(ref):
    rng = random.Random(81)
    differ = 0
    for _ in range(300):
        s = (rng.uniform(-20, 20), rng.uniform(-25, 25), rng.uniform(0, 50))
        got = ref.rk4fma_step(s, 0.01)
        want = rk4_exact([Fraction(v) for v in s], Fraction(0.01))
        for g, w in zip(got, want):
            assert abs(Fraction(g) - w) < Fraction(1, 10 ** 12)
        differ += got != ref.rk4_step(s, 0.01)
    assert differ > 30  # a genuinely different rounding sequence (~30% of single steps differ)


def test_fixed_points(ref):
    assert ref.iterate((0.0, 0.0, 0.0), 3000, integrator=ref.RK4_FMA) == (0.0, 0.0, 0.0)
    q = math.sqrt(float(BETA * (RHO - 1)))
    for sg in (1.0, -1.0):
        c = (sg * q, sg * q, 27.0)
        out = ref.iterate(c, 3000, integrator=ref.RK4_FMA)
        assert max(abs(out[i] - c[i]) for i in range(3)) <= 1e-12


def test_order_four(ref):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 30
    sol = mpmath.odefun(lambda t, v: [10 * (v[1] - v[0]), 28 * v[0] - v[1] - v[0] * v[2],
                                      v[0] * v[1] - mpmath.mpf(8) / 3 * v[2]], 0, [1, 1, 1])
    exact = [float(v) for v in sol(mpmath.mpf("0.1"))]
    e1 = max(abs(a - b) for a, b in zip(ref.iterate((1.0, 1.0, 1.0), 10, 0, ref.RK4_FMA), exact))
    e2 = max(abs(a - b) for a, b in zip(ref.iterate((1.0, 1.0, 1.0), 20, 1, ref.RK4_FMA), exact))
    assert e1 < 2e-5 and 12.0 <= e1 / e2 <= 20.0


def test_steps_match_python_exact_fma(ref):
    rng = random.Random(82)
    for _ in range(200):
        s = [rng.uniform(-20, 20), rng.uniform(-25, 25), rng.uniform(0, 50)]
        assert list(ref.rk4fma_step(tuple(s), 0.01)) == pyref.rk4fma(s, 0.01)


def test_cipher_matches_python_reading(ref):
    rng = random.Random(83)
    for _ in range(3):
        pw = rng.randbytes(12)
        pt = rng.randbytes(rng.randrange(0, 40))
        prm = ref.params(mode=ref.STRONG, n_it=5, integrator=ref.RK4_FMA)
        ct, _ = ref.encrypt(pw, pt, prm)
        assert ct.tobytes() == pyref.run_stream(pyref.key_material(pw), pt, 5, integrator="rk4fma")
        st, back, _ = ref.decrypt(pw, ct, prm)
        assert st == ref.OK and back.tobytes() == pt
        ct0, _ = ref.encrypt(pw, pt, ref.params(mode=ref.STRONG, n_it=5))
        assert ct0.tobytes()[:len(pt) + 16] != ct.tobytes() or len(pt) == 0
