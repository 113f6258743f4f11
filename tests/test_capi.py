"""The C-ABI libraries load and export every symbol their headers declare
(CPU: no compute calls; creating an engine without a GPU must fail loudly,
never fall back to the CPU)."""
import os
import re

import pytest

from conftest import ROOT
from paper_2112_03804_b200 import _native as N
from paper_2112_03804_b200 import host as H


def header_functions(name):
    text = open(os.path.join(ROOT, "include", name)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kr[h]?_[a-z_0-9]+)\s*\(", text)))


def test_engine_header_symbols_exported():
    L = N.cuda()
    declared = header_functions("kr_engine.h")
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(N.CUDA_SYMBOLS) == declared


def test_host_header_symbols_exported():
    L = H.host()
    declared = header_functions("kr_host.h")
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(H.HOST_SYMBOLS) == declared


def test_cuda_library_is_sm100a():
    data = open(N.cuda_lib_path(), "rb").read()
    assert b"sm_100a" in data


@pytest.mark.skipif(N.device_count() > 0, reason="a CUDA device is present")
def test_no_device_no_fallback():
    f = H.builtin("golden").sparsify("b")
    from paper_2112_03804_b200 import CudaEngine
    with pytest.raises(N.NoDeviceError):
        CudaEngine(f)
