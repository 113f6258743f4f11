"""Device-side factor construction: Technique B with
postprocessing built by kernels from the KronPayoff pieces must equal the host
builder's factors BIT FOR BIT (structure and values; the host builder is
itself bit-exact against the oracle, tests/test_host_builder.py), and engines
built on either give the same products bitwise."""
import numpy as np
import pytest

from conftest import factors_equal
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H

pytestmark = pytest.mark.gpu

CASES = [("golden", {}), ("twenty_card", {}), ("bluffing", {}), ("all_tie", {}),
         ("random_small", dict(seed=3)), ("random_small", dict(seed=6)), ("bench", dict(seed=2, hands=100)),
         ("river_full", dict(seed=2, board="Kc9d7c4d2c", deck=26, tree=3)),
         ("river_full", dict(seed=1, board="Ks7d4c2h9s", tree=3)),
         ("river_full", dict(seed=1, board="AhKhQh7c7d", tree=1))]


@pytest.mark.parametrize("name,kw", CASES)
def test_device_factors_bit_exact(name, kw):
    p = H.builtin(name, **kw)
    host = p.sparsify("b", True)
    dev = p.sparsify_device()
    assert (dev.rows, dev.cols, dev.k) == (host.rows, host.cols, host.k)
    assert dev.nnz == host.nnz
    assert factors_equal(dev.factors(), host.factors())


def test_device_factors_engine_products_bitwise():
    p = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    e_host, e_dev = CudaEngine(p.sparsify("b", True)), CudaEngine(p.sparsify_device())
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
    assert np.array_equal(e_host.Ax(x).view(np.int64), e_dev.Ax(x).view(np.int64))
    assert np.array_equal(e_host.ATx(y).view(np.int64), e_dev.ATx(y).view(np.int64))
