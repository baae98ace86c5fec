import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


from goldens import load_npz  # noqa: E402  (tests/golden/goldens.py)


@pytest.fixture(scope="session")
def constants():
    with open(os.path.join(GOLDEN, "constants.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_cdc():
    return load_npz("cdc")


@pytest.fixture(scope="session")
def golden_rotary():
    return load_npz("rotary")


@pytest.fixture(scope="session")
def golden_registry():
    return load_npz("registry")


@pytest.fixture(scope="session")
def golden_traces():
    return load_npz("traces")


@pytest.fixture(scope="session")
def golden_radix():
    return load_npz("radix")
