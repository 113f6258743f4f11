import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE = "/root/reference/proj"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "multigpu: needs two or more CUDA devices (skips otherwise)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def instance_fixtures():
    with open(os.path.join(GOLDEN, "instances_v1.json")) as f:
        return json.load(f)


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype == np.float64:
        return np.array_equal(a.view(np.int64), b.view(np.int64))
    return np.array_equal(a, b)


def factors_equal(fa, fb):
    for n in ("ahat", "u", "m", "v"):
        for x, y in zip(fa[n], fb[n]):
            if not bits_equal(x, y):
                return False
    return True
