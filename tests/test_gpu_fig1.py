"""NEXT-4 analysis on the GPU: Fig.1 digit histograms, exact against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from paper_1201_3114_b200 import inputs
from paper_1201_3114_b200 import lorenz as L

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


@pytest.mark.parametrize("integrator,dt_code", [(L.RK4, 0), (L.EULER, 1), (L.RK4_FMA, 2)])
def test_digit_histograms_match_oracle(integrator, dt_code):
    lanes, skip, samples, stride = 300, 200, 60, 5
    ic = inputs.initial_states(lanes)
    hist = torch.empty(3 * 4 * 128, dtype=torch.int64, device=DEV)
    L.lorenz_digit_histograms(torch.from_numpy(ic).to(DEV), lanes, skip, samples, stride, hist, dt_code=dt_code,
                              integrator=integrator)
    want = oracle.digit_hist(ic, skip, samples, stride, dt_code, integrator)
    assert np.array_equal(hist.cpu().numpy().reshape(3, 4, 128), want.astype(np.int64))


def test_digit_histograms_edge_lanes():
    hist = torch.empty(3 * 4 * 128, dtype=torch.int64, device=DEV)
    L.lorenz_digit_histograms(None, 0, 10, 10, 1, hist)
    assert not hist.any()
    ic = inputs.initial_states(129)  # one lane past a CTA
    L.lorenz_digit_histograms(torch.from_numpy(ic).to(DEV), 129, 3, 4, 2, hist)
    assert np.array_equal(hist.cpu().numpy().reshape(3, 4, 128),
                          oracle.digit_hist(ic, 3, 4, 2).astype(np.int64))


def test_digit_histograms_closed_form_and_fixed_points():
    """The closed-form cases of tests/test_oracle_fig1.py on the GPU kernel: samples equal to the
    initial states (skip = stride = 0) and trajectories held at the fixed points 0 and C+-."""
    import math
    s = math.sqrt(72.0)
    cases = [(np.array([(12.34375, -7.8125, 0.5), (63.999755859375, -0.0078125, 27.0),
                        (-19.96875, 0.0, 48.015625)]), 0, 3, 0),
             (np.array([(0.0, 0.0, 0.0), (s, s, 27.0), (-s, -s, 27.0)]), 40, 25, 9)]
    hist = torch.empty(3 * 4 * 128, dtype=torch.int64, device=DEV)
    for ic, skip, samples, stride in cases:
        L.lorenz_digit_histograms(torch.from_numpy(ic).to(DEV), len(ic), skip, samples, stride, hist)
        got = hist.cpu().numpy().reshape(3, 4, 128)
        assert np.array_equal(got, oracle.digit_hist(ic, skip, samples, stride).astype(np.int64))
        assert (got.sum(axis=2) == len(ic) * samples).all()
