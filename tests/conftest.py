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
