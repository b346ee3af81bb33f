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
