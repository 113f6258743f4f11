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


@pytest.fixture(autouse=True)
def _checked_build_guards(request):
    """Under the bounds-checked build (KR_CUDA_LIB_VARIANT=checked), every GPU
    test ends with the guard zones of all device allocations intact."""
    yield
    if os.environ.get("KR_CUDA_LIB_VARIANT") != "checked" or request.node.get_closest_marker("gpu") is None:
        return
    import gc

    from paper_2112_03804_b200 import _native as N
    gc.collect()  # engines / solvers freed now have their guards checked too
    bad = N.cuda().kr_checked_verify()
    assert bad == 0, f"{bad} device allocation(s) had a guard zone overwritten"
