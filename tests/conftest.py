import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built liblorenz.so")
    config.addinivalue_line("markers", "slow: longer-running CPU test")


@pytest.fixture(scope="session")
def ref():
    import oracle
    oracle.lib()
    return oracle


@pytest.fixture
def tune():
    """Launch-plan overrides through the C ABI (lorenz_set_tuning): tune(schedule="wave"|"seg"|None,
    seg_slots=S|None, seg_skew=k|None, cta=C|None); None restores that field's default. Every
    override is cleared when the test ends."""
    from paper_1201_3114_b200 import lorenz as L
    state = {}
    codes = {None: L.SCHED_AUTO, "wave": L.SCHED_WAVE, "seg": L.SCHED_BALANCED}
    defaults = {"schedule": None, "seg_slots": 0, "seg_skew": -1, "cta": 0}

    def set_(**kw):
        state.update(kw)
        args = {k: (defaults[k] if state.get(k) is None and k != "schedule" else state.get(k)) for k in defaults}
        args["schedule"] = codes[args["schedule"]]
        L.lorenz_set_tuning(**args)
    yield set_
    L.lorenz_set_tuning(reset=True)
