import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path")


@pytest.fixture(scope="session")
def small_golden():
    with open(os.path.join(GOLDEN, "small.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def config_golden():
    path = os.path.join(GOLDEN, "configs.json")
    if not os.path.exists(path):
        pytest.skip("configs.json golden digests not generated")
    with open(path) as f:
        return json.load(f)


@pytest.fixture(params=[2, 1], ids=["coef64x5", "coef32x3"])
def coef_words(request):
    """Run a GPU test in both convolution modes: 64-bit coefficients over five
    primes (the default up to 121,295,104 bits) and 32-bit over three (beyond)."""
    from paper_1910_04429_b200 import _native

    _native.force_coef_words(request.param)
    try:
        yield request.param
    finally:
        _native.force_coef_words(0)
