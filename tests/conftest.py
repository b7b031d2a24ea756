"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden_path(*parts):
    return os.path.join(GOLDEN, *parts)


def load_manifest():
    with open(golden_path("manifest.json")) as fh:
        return json.load(fh)["cases"]


def load_case(name):
    arr = np.load(golden_path(f"{name}.npz"))
    with open(golden_path(f"{name}.reports.json")) as fh:
        reports = json.load(fh)
    return arr, reports


@pytest.fixture(scope="session")
def manifest():
    return load_manifest()
