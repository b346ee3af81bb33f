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
