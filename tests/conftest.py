"""Shared pytest setup: the `gpu` marker and repo-root imports."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def golden_cases():
    import numpy as np

    return np.load(os.path.join(GOLDEN, "filter_cases.npz"))


@pytest.fixture(scope="session")
def box_params():
    import json

    with open(os.path.join(GOLDEN, "box_params.json")) as fh:
        return json.load(fh)
