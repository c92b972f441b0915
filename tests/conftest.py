import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))  # test-only checker


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")
    config.addinivalue_line("markers", "slow: full-size BASELINE configuration cases")


GOLDEN_CASES = ["gen64", "gen64_x255", "gen64_p0", "gen64_p2", "gen96_tol", "accept_c3",
                "plateau64", "identical48", "c1", "c1_x255"]


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


@pytest.fixture(params=GOLDEN_CASES)
def golden_case(request):
    return request.param, golden(request.param)
