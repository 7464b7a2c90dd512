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


def pytest_collection_modifyitems(config, items):
    # a kernel that never finishes must end the run, not stall it: GPU tests get a
    # thread-method timeout (dumps the stacks and exits) unless they set their own
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(240, method="thread"))


@pytest.fixture(scope="session")
def golden_cases():
    import numpy as np

    return np.load(os.path.join(GOLDEN, "filter_cases.npz"))


@pytest.fixture(scope="session")
def box_params():
    import json

    with open(os.path.join(GOLDEN, "box_params.json")) as fh:
        return json.load(fh)
