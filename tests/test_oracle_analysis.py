"""Pins of the oracle's NEXT-4 analysis suite (§4, Figs. 3 and 4; readings Q25-Q27).

Each pin is fixed by something other than the oracle's own formula: closed forms of
structured images, the Wiener-Khinchin theorem / numpy's FFT (a library route with a
different algorithm and summation order), Parseval, symmetry, and the exponential law of
white-noise periodograms (flatness -> exp(-gamma)).
"""
import math

import numpy as np
import pytest

import oracle
from paper_1201_3114_b200 import inputs

EPS = np.finfo(np.float64).eps


def noise(h, w, seed=5):
    return inputs.message(h * w, seed=seed).reshape(h, w)


# ---------------------------------------------------------------- autocorrelation (Fig.3)
def test_autocorr_checkerboard_closed_form():
    """x = 255 * ((i + j) mod 2): d = +-127.5, r(u,v) = (-1)^(u+v) exactly."""
    h, w = 8, 16
    i, j = np.indices((h, w))
    r = oracle.autocorr(255 * ((i + j) % 2))
    assert np.array_equal(r, (-1.0) ** (i + j))


def test_autocorr_stripes_closed_form():
    """Horizontal stripes x = 255 * (i mod 2): r(u,v) = (-1)^u, independent of v."""
    h, w = 6, 10
    i, _ = np.indices((h, w))
    r = oracle.autocorr(255 * (i % 2))
    assert np.array_equal(r, (-1.0) ** i)


def test_autocorr_impulse_closed_form():
    """One bright pixel on black: r(0,0) = 1 and r = -1/(N-1) at every other lag (algebra in
    DESIGN.md §2e: c = -a^2/N, var = a^2 (N-1)/N)."""
    h, w = 8, 8
    x = np.zeros((h, w), dtype=np.uint8)
    x[3, 5] = 255
    r = oracle.autocorr(x)
    want = np.full((h, w), -1.0 / (h * w - 1))
    want[0, 0] = 1.0
    np.testing.assert_allclose(r, want, rtol=0, atol=64 * EPS)


def test_autocorr_constant_convention():
    """Zero variance: zero lag 1, every other lag 0 (S:436 convention, Q25)."""
    r = oracle.autocorr(np.full((4, 8), 77, dtype=np.uint8))
    want = np.zeros((4, 8))
    want[0, 0] = 1.0
    assert np.array_equal(r, want)


def test_autocorr_wiener_khinchin():
    """Random bytes: equals Re(ifft2(|fft2(x - mean)|^2)) normalised (numpy FFT route); symmetric
    under (u,v) -> (-u,-v); zero lag 1; the _at entry agrees with the matrix bit for bit."""
    x = noise(16, 32)
    r = oracle.autocorr(x)
    d = x - x.mean()
    c = np.fft.ifft2(np.abs(np.fft.fft2(d)) ** 2).real
    np.testing.assert_allclose(r, c / c[0, 0], rtol=0, atol=1e-13)
    assert r[0, 0] == 1.0
    rs = np.roll(np.flip(r, (0, 1)), (1, 1), (0, 1))  # r(-u,-v)
    np.testing.assert_allclose(r, rs, rtol=0, atol=1e-15)
    for u, v in [(0, 0), (1, 0), (0, 1), (5, 17), (15, 31)]:
        assert oracle.autocorr_at(x, u, v) == r[u, v]
    assert np.abs(r).max() <= 1.0


def test_autocorr_white_noise_is_flat():
    """white-noise bytes -> off-origin |r| small (std 1/sqrt(N) = 1/64 at 64x64)."""
    r = oracle.autocorr(noise(64, 64, seed=9))
    off = np.abs(r.ravel()[1:])
    assert off.max() < 6 / 64 and abs(off.mean() - math.sqrt(2 / math.pi) / 64) < 0.002


# ---------------------------------------------------------------- power spectrum (Fig.4)
def shifted_numpy(x):
    n = x.size
    return np.fft.fftshift(np.abs(np.fft.fft2(x.astype(np.float64))) ** 2) / n**2


def test_power_spectrum_vs_numpy_fft_and_parseval():
    x = noise(16, 8)
    p = oracle.power_spectrum(x)
    q = shifted_numpy(x)
    n = x.size
    tol = 4 * math.sqrt(2) * x.mean() ** 2 * (n + 64) * EPS  # DESIGN.md §2e error bound
    assert np.abs(p - q).max() <= tol
    assert math.isclose(p.sum(), (x.astype(np.float64) ** 2).mean(), rel_tol=1e-12)
    assert p[8, 4] == pytest.approx(x.mean() ** 2, rel=1e-13)  # DC at the centre
    for k, l in [(0, 0), (3, 5), (15, 7), (8, 4)]:
        assert oracle.power_at(x, k, l) == pytest.approx(p[(k + 8) % 16, (l + 4) % 8], rel=1e-12, abs=1e-12)


def test_power_spectrum_constant_image():
    """a constant image has all its power at DC (c^2; numerically ~0 elsewhere)."""
    p = oracle.power_spectrum(np.full((8, 16), 200, dtype=np.uint8))
    assert p[4, 8] == pytest.approx(200.0**2, rel=1e-14)
    p[4, 8] = 0
    assert np.abs(p).max() < 1e-20 * 200**2 * 1e6


def test_power_spectrum_column_alternation():
    """x[m][n] = 255 (n odd): DC and the horizontal Nyquist bin (0, W/2) each hold 127.5^2
    (the DFT pair of a period-2 square wave, S:447 'two symmetric peaks' folded at Nyquist)."""
    h, w = 8, 16
    x = np.zeros((h, w), dtype=np.uint8)
    x[:, 1::2] = 255
    p = oracle.power_spectrum(x)
    want = np.zeros((h, w))
    want[h // 2, w // 2] = 127.5**2  # DC
    want[h // 2, 0] = 127.5**2  # (k, l) = (0, W/2)
    np.testing.assert_allclose(p, want, rtol=1e-13, atol=1e-9)


def test_power_spectrum_checkerboard():
    h, w = 8, 8
    i, j = np.indices((h, w))
    p = oracle.power_spectrum(255 * ((i + j) % 2))
    want = np.zeros((h, w))
    want[4, 4] = want[0, 0] = 127.5**2  # DC and (H/2, W/2)
    np.testing.assert_allclose(p, want, rtol=1e-13, atol=1e-9)


def test_power_spectrum_separable_cosine():
    """A real sinusoid along n with frequency f = 3: bins (0, +-3) carry (A/2)^2 each.
    Bytes are rounded, so compare against numpy on the same bytes and check the peak."""
    h, w = 4, 32
    n = np.arange(w)
    row = np.round(127.5 + 100 * np.cos(2 * np.pi * 3 * n / w)).astype(np.uint8)
    x = np.tile(row, (h, 1))
    p = oracle.power_spectrum(x)
    assert np.unravel_index(np.argsort(p.ravel())[-3:], p.shape)[1].tolist().count(16) == 1
    a1 = abs(np.dot(row.astype(np.float64), np.exp(-2j * np.pi * 3 * n / w))) / w  # the row's 1-D DFT at f
    assert p[2, 16 + 3] == pytest.approx(a1**2, rel=1e-12) and p[2, 16 - 3] == pytest.approx(a1**2, rel=1e-12)
    assert a1 == pytest.approx(50.0, rel=1e-2)  # amplitude 100 -> 100/2 per side band, before byte rounding
    assert p[:2].max() < 1e-18 * p.max() * 1e6 and p[3:].max() < 1e-18 * p.max() * 1e6  # no vertical frequency


def test_flatness_white_noise_is_exp_minus_gamma():
    """A white-noise periodogram is exponentially distributed per bin, whose geometric / arithmetic
    mean ratio is exp(-gamma) = 0.5615 (Q26: S:446's '> 0.8' does not hold for this definition)."""
    p = oracle.power_spectrum(noise(64, 64, seed=21))
    f = oracle.spectral_flatness(p)
    assert abs(f - math.exp(-0.5772156649015329)) < 0.02
    lp = np.log(np.delete(p.ravel(), 32 * 64 + 32))
    assert f == pytest.approx(math.exp(lp.mean()) / np.exp(lp).mean(), rel=1e-12)


def test_flatness_degenerate():
    assert oracle.spectral_flatness(np.zeros((4, 4))) == 0.0
    p = np.ones((4, 4))
    assert oracle.spectral_flatness(p) == pytest.approx(1.0, rel=1e-15)
    p[0, 1] = 0
    assert oracle.spectral_flatness(p) == 0.0
