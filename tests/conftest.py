"""pytest configuration: the `gpu` marker and shared fixtures/helpers."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def pinned():
    with open(os.path.join(GOLDEN, "pinned.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ref_runs():
    with open(os.path.join(GOLDEN, "ref_runs.json")) as f:
        return json.load(f)


from gfq_testutil import arr  # noqa: E402,F401
