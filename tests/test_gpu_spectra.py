"""GPU parity of the NEXT-4 §4 analysis kernels (Fig.3 autocorrelation, Fig.4 power spectra)
against the oracle's plain-sum definitions, within the FP64 error bounds of DESIGN.md §2e.

Full matrices at sizes the O(N^2) oracle finishes in seconds; at 4096 x 4096 (16 MiB of
ciphertext) sampled lags / frequencies recomputed one by one by the oracle plus
size-independent properties (Parseval, r(0,0) = 1, symmetry, exp(-gamma) flatness).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
EPS = np.finfo(np.float64).eps
GAMMA = 0.5772156649015329


def tol_power(x: np.ndarray) -> float:
    """|dP| bound: both sides' |dF| <= (N + 16 log2 N) eps sum|x| per component."""
    n = x.size
    return 4 * math.sqrt(2) * float(x.mean()) ** 2 * (n + 16 * math.log2(n)) * EPS


def tol_autocorr(n: int) -> float:
    return 4 * (n + 64 * math.sqrt(n) * math.log2(n)) * EPS


def gpu_autocorr(x: np.ndarray) -> np.ndarray:
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    r = torch.empty(x.shape, dtype=torch.float64, device=DEV)
    L.lorenz_autocorrelation(xd, r)
    return r.cpu().numpy()


def gpu_spectrum(x: np.ndarray):
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    p = torch.empty(x.shape, dtype=torch.float64, device=DEV)
    f = torch.empty(1, dtype=torch.float64, device=DEV)
    L.lorenz_power_spectrum(xd, p, f)
    return p.cpu().numpy(), float(f.item())


def cipher_image(h, w, seed=3):
    """The first h*w ciphertext bytes of an encrypted synthetic message (Fig.3(b) / Fig.4(b))."""
    n = h * w
    key = L.lorenz_keysetup(inputs.password(seed=seed), mode=L.FAST, n_it=20)
    pt = torch.from_numpy(inputs.message(n, seed=seed)).to(DEV)
    ct = torch.empty(key.ct_len(n), dtype=torch.uint8, device=DEV)
    L.lorenz_encrypt(key, n, 0, key.num_blocks(n), pt, ct)
    return ct[:n].cpu().numpy().reshape(h, w)


def plain_image(h, w):
    """Synthetic 'plain image' with global and local structure: gradient + disc + stripes."""
    i, j = np.indices((h, w))
    g = 60 + 100 * i / h + 40 * j / w
    g += 50 * (((i - h / 2) ** 2 + (j - w / 3) ** 2) < (min(h, w) / 4) ** 2)
    g += 20 * ((j // 4) % 2)
    return np.clip(g, 0, 255).astype(np.uint8)


def structured(kind, h, w):
    i, j = np.indices((h, w))
    if kind == "checker":
        return (255 * ((i + j) % 2)).astype(np.uint8)
    if kind == "constant":
        return np.full((h, w), 91, dtype=np.uint8)
    if kind == "near_constant":  # large mean, tiny variance: the autocorrelation's centring must be exact
        x = np.full((h, w), 200, dtype=np.uint8)
        x[h // 3, (2 * w) // 3] = 201
        return x
    if kind == "impulse":
        x = np.zeros((h, w), dtype=np.uint8)
        x[h - 1, w // 3] = 255
        return x
    if kind == "plain":
        return plain_image(h, w)
    return inputs.message(h * w, seed=17).reshape(h, w)


# W = 64, 256, 128, 1024, 2048: the C2R row pass's first radix is 2, 8, 4, 2, 4 -> its register-paired
# pre-processing with 8, 2, 4, 8, 4 groups per thread (spectra.cuh c2r_registers)
SHAPES = [(2, 2), (2, 8), (8, 2), (4, 16), (16, 32), (64, 64), (128, 32), (32, 256), (16, 128), (8, 1024),
          (4, 2048)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["noise", "plain", "checker", "impulse", "constant"])
def test_power_spectrum_parity(shape, kind):
    x = structured(kind, *shape)
    p, f = gpu_spectrum(x)
    want = oracle.power_spectrum(x)
    assert np.abs(p - want).max() <= tol_power(x)
    # flatness is well conditioned only when every non-DC bin is far above the rounding bound:
    # then |d log P| <= tol / min P per bin and |df| / f <= 2 tol / min P (zero bins of structured
    # images come out as exact zeros on one side and ~1e-26 residues on the other)
    nondc = np.delete(want.ravel(), (shape[0] // 2) * shape[1] + shape[1] // 2)
    if nondc.size and nondc.min() > 1e3 * tol_power(x):
        assert f == pytest.approx(oracle.spectral_flatness(want), rel=2 * tol_power(x) / nondc.min())
    if kind == "constant":
        assert f == 0.0 or f < 1e-6  # rounding residue only


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("kind", ["noise", "plain", "checker", "impulse", "constant", "near_constant"])
def test_autocorrelation_parity(shape, kind):
    x = structured(kind, *shape)
    r = gpu_autocorr(x)
    want = oracle.autocorr(x)
    assert np.abs(r - want).max() <= tol_autocorr(x.size)
    assert r[0, 0] == 1.0 or abs(r[0, 0] - 1.0) <= 2 * EPS
    if kind == "constant":
        assert np.array_equal(r, want)  # the exact S:436 convention


def test_cipher_image_fig3_fig4_statistics():
    """Fig.3(b) / Fig.4(h): ciphertext has a flat autocorrelation and a white spectrum."""
    x = cipher_image(128, 128)
    r = gpu_autocorr(x)
    np.testing.assert_allclose(r, oracle.autocorr(x), rtol=0, atol=tol_autocorr(x.size))
    assert np.abs(r.ravel()[1:]).max() < 0.05  # S:437 at this size
    p, f = gpu_spectrum(x)
    assert abs(f - math.exp(-GAMMA)) < 0.02
    xp = plain_image(128, 128)
    _, fp = gpu_spectrum(xp)
    assert fp < 0.2  # the plain image's spectrum is far from flat
    rp = gpu_autocorr(xp)
    assert rp[1, 0] > 0.5


def test_full_size_sampled_and_properties():
    """4096 x 4096 ciphertext (16 MiB): sampled lags / frequencies against the oracle, Parseval,
    symmetry, flatness -> exp(-gamma)."""
    h = w = 4096
    x = cipher_image(h, w, seed=8)
    r = gpu_autocorr(x)
    rng = np.random.default_rng(4)
    lags = [(0, 0), (1, 0), (0, 1), (h - 1, w - 1), (h // 2, w // 2)] + [tuple(rng.integers(0, h, 2)) for _ in range(3)]
    for u, v in lags:
        assert abs(r[u, v] - oracle.autocorr_at(x, int(u), int(v))) <= tol_autocorr(x.size), (u, v)
    rs = np.roll(np.flip(r, (0, 1)), (1, 1), (0, 1))
    assert np.abs(r - rs).max() <= tol_autocorr(x.size)
    assert np.abs(r.ravel()[1:]).max() < 6 / 4096 * 1.5
    p, f = gpu_spectrum(x)
    assert math.isclose(p.sum(), float((x.astype(np.float64) ** 2).mean()), rel_tol=1e-11)
    assert p[h // 2, w // 2] == pytest.approx(float(x.mean(dtype=np.float64)) ** 2, rel=1e-12)
    for k, l in [(1, 0), (0, 1), (777, 3001), (h // 2, w // 2), (h - 1, 5)]:
        got = p[(k + h // 2) % h, (l + w // 2) % w]
        assert abs(got - oracle.power_at(x, k, l)) <= tol_power(x), (k, l)
    assert abs(f - math.exp(-GAMMA)) < 0.003


@pytest.mark.parametrize("h,w", [(3, 4), (4, 3), (1, 8), (8192, 2), (0, 4)])
def test_bad_shapes_rejected(h, w):
    x = torch.zeros(max(h * w, 1), dtype=torch.uint8, device=DEV)
    out = torch.zeros(max(h * w, 1), dtype=torch.float64, device=DEV)
    st = L.lib().lorenz_power_spectrum(x.data_ptr(), h, w, out.data_ptr(), None, None)
    assert st == L.E_ARG
    st = L.lib().lorenz_autocorrelation(x.data_ptr(), h, w, out.data_ptr(), None)
    assert st == L.E_ARG


@pytest.mark.parametrize("h,w", [(2048, 16), (2048, 32)])
def test_tall_matrices_full(h, w):
    """Tall matrices (2048-point column transforms over 8-16 packed columns, the packed DC /
    Nyquist column included): full matrices against the oracle's plain sums."""
    x = cipher_image(h, w, seed=h + w)
    p, f = gpu_spectrum(x)
    want = oracle.power_spectrum(x)
    assert np.abs(p - want).max() <= tol_power(x)
    assert abs(f - oracle.spectral_flatness(want)) <= 1e-9
    r = gpu_autocorr(x)
    assert np.abs(r - oracle.autocorr(x)).max() <= tol_autocorr(x.size)


@pytest.mark.parametrize("h,w", [(4096, 16), (4096, 64), (2048, 128)])
def test_tall_matrices_sampled(h, w):
    """4096- and 2048-point column transforms: frequencies in every residue class k mod 4 and at
    both ends, the packed column's DC / Nyquist outputs (l = 0, W/2) and their neighbours, against
    the oracle one frequency / lag at a time; Parseval and r(0,0) = 1 over the whole matrix."""
    x = cipher_image(h, w, seed=h ^ w)
    p, _ = gpu_spectrum(x)
    r = gpu_autocorr(x)
    rng = np.random.default_rng(h + w)
    ks = [0, 1, 2, 3, 4, 5, h // 2 - 1, h // 2, h // 2 + 1, h - 4, h - 3, h - 2, h - 1] + list(rng.integers(0, h, 8))
    ls = [0, 1, w // 2 - 1, w // 2, w // 2 + 1, w - 1] + list(rng.integers(0, w, 2))
    for k in ks:
        for l in ls:
            got = p[(k + h // 2) % h, (l + w // 2) % w]
            assert abs(got - oracle.power_at(x, int(k), int(l))) <= tol_power(x), (k, l)
    for k in ks[::2]:
        for l in ls[::2]:
            assert abs(r[k, l] - oracle.autocorr_at(x, int(k), int(l))) <= tol_autocorr(x.size), (k, l)
    assert math.isclose(p.sum(), float((x.astype(np.float64) ** 2).mean()), rel_tol=1e-11)
    assert r[0, 0] == pytest.approx(1.0, abs=1e-13)


@pytest.mark.parametrize("h,w", [(4096, 64), (2048, 128)])
def test_tma_column_pass_is_the_one_that_runs(h, w):
    """The autocorrelation's column pass at H = 2048 / 4096 is the TMA kernel (fft_col_tma_kernel), not
    the fft_pass_kernel fallback the library keeps for when no tensor map can be built: the kernel
    names CUPTI records for one call, and the result against the oracle at sampled lags."""
    x = cipher_image(h, w, seed=h + 3 * w)
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    r = torch.empty((h, w), dtype=torch.float64, device=DEV)
    L.lorenz_autocorrelation(xd, r)  # warm (tensor-map encoder fetched, kernels loaded)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        L.lorenz_autocorrelation(xd, r)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    assert any("fft_col_tma_kernel" in n for n in names), names
    assert not any("fft_pass_kernel<2, 6" in n for n in names), names  # (IN_COMPLEX, OUT_POWER_FFT fallback)
    rc = r.cpu().numpy()
    for u, v in [(0, 0), (1, 0), (0, 1), (h - 1, w - 1), (h // 2, 3), (17, w // 2)]:
        assert abs(rc[u, v] - oracle.autocorr_at(x, u, v)) <= tol_autocorr(x.size), (u, v)


def test_near_constant_full_size_closed_form():
    """4096 x 4096 of 200 with one pixel of 201 (mean 200 + 1/N, variance ~1/N): the whole r matrix against
    its closed form r = -1/(N-1) off the origin (any single-pixel deviation from a constant gives it). The
    large mean makes this the case where the centring has to be exact before the transforms."""
    h = w = 4096
    n = h * w
    x = structured("near_constant", h, w)
    r = gpu_autocorr(x)
    off = np.ones((h, w), dtype=bool)
    off[0, 0] = False
    assert r[0, 0] == 1.0
    assert np.abs(r[off] + 1.0 / (n - 1)).max() <= tol_autocorr(n)


@pytest.mark.parametrize("h,w", [(4096, 4096), (2048, 2048), (4096, 64), (2048, 128), (1024, 4096)])
def test_full_size_every_bin_against_numpy_fft(h, w):
    """Ciphertext images up to 4096 x 4096: EVERY frequency and lag (not a sample) against numpy's FFT in
    float64 — a different algorithm (pocketfft), the route the oracle's own pins use
    (test_oracle_analysis.py) — within the same FP64 bounds; the four-step spectrum, the TMA column pass
    (H = 2048, 4096) and the paired C2R rows at full size."""
    x = cipher_image(h, w, seed=21 + h + w)
    n = x.size
    p, _ = gpu_spectrum(x)
    xf = x.astype(np.float64)
    want_p = np.fft.fftshift(np.abs(np.fft.fft2(xf)) ** 2) / float(n) ** 2
    assert np.abs(p - want_p).max() <= tol_power(x)
    del want_p
    r = gpu_autocorr(x)
    d = xf - xf.mean()
    c = np.fft.ifft2(np.abs(np.fft.fft2(d)) ** 2).real
    want_r = c / c[0, 0]
    assert np.abs(r - want_r).max() <= tol_autocorr(n)
