"""Pins for the oracle's Fig.1 digit histograms (NEXT-4 analysis; §3.1).

Counting invariants, an independent Python recount over oracle-integrated trajectories,
the attractor's known extent for the integer part, and the paper's claim that
the 3rd-4th and 5th-6th decimal digits are "practically uniform".
"""
import numpy as np

from paper_1201_3114_b200 import inputs


def test_counts_and_python_recount(ref):
    ic = inputs.initial_states(3)
    skip, samples, stride = 50, 40, 7
    h = ref.digit_hist(ic, skip, samples, stride)
    assert (h.sum(axis=2) == 3 * samples).all()
    want = np.zeros((3, 4, 128), dtype=np.uint64)
    for lane in range(3):
        s = ref.iterate(tuple(ic[lane]), skip)
        for _ in range(samples):
            s = ref.iterate(s, stride)
            for c, v in enumerate(s):
                want[c, 0, min(127, max(0, int(v) + 64))] += 1  # int() truncates toward zero
                for k, sc in ((1, 100.0), (2, 1e4), (3, 1e6)):
                    want[c, k, int(abs(v) * sc) % 100] += 1
    assert np.array_equal(h, want)


def test_integer_part_extent_and_low_digit_uniformity(ref):
    ic = inputs.initial_states(32)
    h = ref.digit_hist(ic, 1000, 400, 10).astype(np.int64)
    lims = [(-21, 21), (-28, 28), (0, 50)]  # attractor extent, trunc toward zero
    for c in range(3):
        nz = np.nonzero(h[c, 0])[0] - 64
        assert lims[c][0] <= nz.min() and nz.max() <= lims[c][1]
        assert (h[c, 1:, 100:] == 0).all()
        for k in (2, 3):  # "practically uniform": chi-square, 99 dof
            e = h[c, k, :100].sum() / 100
            assert (((h[c, k, :100] - e) ** 2) / e).sum() < 170


def _closed_form_bins(v: float):
    """Integer-part bin and the digit pairs 1-2, 3-4, 5-6 after the decimal point of |v|, read off
    v's exact decimal expansion (Python's decimal: no binary arithmetic of the oracle's)."""
    from decimal import ROUND_DOWN, Decimal
    d = Decimal(v)  # exact value of the double
    ip = int(d.to_integral_value(rounding=ROUND_DOWN))
    frac = str(abs(d) - abs(d).to_integral_value(rounding=ROUND_DOWN))  # "0.ddddd..." or "0"
    digits = (frac[2:] if "." in frac else "") + "0" * 6
    return ip + 64, [int(digits[0:2]), int(digits[2:4]), int(digits[4:6])]


def test_closed_form_samples_without_integration(ref):
    """skip = stride = 0: every sample is the initial state itself, so the histogram is fixed by the
    decimal digits of the chosen values (Fig.1's "integer part" and "decimal digits" 1-2, 3-4,
    5-6). Values are exact binary fractions with finite decimal expansions, so the
    scaled products are exact and the bins follow from the printed digits alone."""
    vals = [(12.34375, -7.8125, 0.5), (63.999755859375, -0.0078125, 27.0), (-19.96875, 0.0, 48.015625)]
    samples = 3
    h = ref.digit_hist(np.array(vals), 0, samples, 0)
    want = np.zeros((3, 4, 128), dtype=np.uint64)
    for lane in vals:
        for c, v in enumerate(lane):
            b0, pairs = _closed_form_bins(v)
            want[c, 0, b0] += samples
            for k, p in enumerate(pairs):
                want[c, k + 1, p] += samples
    assert _closed_form_bins(63.999755859375) == (127, [99, 97, 55])  # spelled out: 63.99|97|55|859375
    assert _closed_form_bins(-7.8125) == (57, [81, 25, 0])
    assert np.array_equal(h, want)


def test_fixed_points_give_single_bins(ref):
    """Trajectories started at the fixed points (0,0,0) and C+- = (+-sqrt(72), +-sqrt(72), 27) stay
    there bit for bit (pinned in test_oracle_dynamics), so every sample of a lane falls
    in the bins of those coordinates, read from sqrt(72) = 8.485281374238570...: integer part
    +-8, digit pairs 48, 52, 81; z = 27: integer part 27, digits 00."""
    import math
    s = math.sqrt(72.0)
    ic = np.array([(0.0, 0.0, 0.0), (s, s, 27.0), (-s, -s, 27.0)])
    samples = 25
    h = ref.digit_hist(ic, 40, samples, 9)
    want = np.zeros((3, 4, 128), dtype=np.uint64)
    for c, bins in enumerate([(64, 72, 56), (64, 72, 56), (64, 91, 91)]):
        for b in bins:
            want[c, 0, b] += samples
    for c in range(3):
        pairs = [(0, 0, 0), (48, 52, 81), (48, 52, 81)] if c < 2 else [(0, 0, 0)] * 3
        for lane_pairs in pairs:
            for k, p in enumerate(lane_pairs):
                want[c, k + 1, p] += samples
    assert np.array_equal(h, want)
