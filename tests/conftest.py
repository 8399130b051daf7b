"""Shared test setup: gpu marker, repo on sys.path, golden fixtures."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
# the reference's own test files, vendored unmodified; they import `hetsched`
# and run only through tests/test_gpu_reference_suite.py (a shim package)
collect_ignore = ["reference_suite"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def small_cases():
    return _load("small_graphs.json")


@pytest.fixture(scope="session")
def medium_cases():
    return _load("medium_graphs.json")


@pytest.fixture(scope="session")
def compare_golden():
    return _load("compare_cfg5_64.json")
