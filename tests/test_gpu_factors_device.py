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


@pytest.mark.parametrize("name,kw", CASES)
def test_device_built_engine_bitwise(name, kw):
    """The engine laid out on the device (kr_engine_create_device_b) against
    the engine built from the host builder's factors: identical products
    bit for bit and the same flop count."""
    p = H.builtin(name, **kw)
    e_host, e_dev = CudaEngine(p.sparsify("b", True)), CudaEngine.device_built(p)
    assert (e_dev.rows, e_dev.cols, e_dev.k) == (e_host.rows, e_host.cols, e_host.k)
    assert e_dev.nnz == e_host.nnz
    rng = np.random.default_rng(11)
    for _ in range(2):
        x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
        assert np.array_equal(e_host.Ax(x).view(np.int64), e_dev.Ax(x).view(np.int64))
        assert np.array_equal(e_host.ATx(y).view(np.int64), e_dev.ATx(y).view(np.int64))
    assert e_host.last_flops() == e_dev.last_flops()


def test_device_built_engine_multiboard_and_solver():
    boards = H.turn_instances("Ks7d4c2h", nboards=5, tree=3)
    mixed = [i for i, _ in boards] + [H.builtin("river_full", seed=5, board="Kc9d7c4d2c", deck=26, tree=3)]
    e_host = CudaEngine([b.sparsify("b", True) for b in mixed])
    e_dev = CudaEngine.device_built(mixed)
    rng = np.random.default_rng(12)
    x, y = rng.standard_normal(e_host.cols), rng.standard_normal(e_host.rows)
    assert np.array_equal(e_host.Ax(x).view(np.int64), e_dev.Ax(x).view(np.int64))
    assert np.array_equal(e_host.ATx(y).view(np.int64), e_dev.ATx(y).view(np.int64))
    # a DCFR solve driven by the device-built engine is bitwise the host-built one
    from paper_2112_03804_b200.solver import CudaSolver, DcfrParams
    i0 = boards[0][0]
    ins = [i for i, _ in boards]
    runs = []
    for eng in (CudaEngine([f for _, f in boards]), CudaEngine.device_built(ins)):
        s = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [b.m1 for b in ins], [b.m2 for b in ins], i0.pot)
        runs.append(s.run(DcfrParams(max_iters=20, checkpoint_every=5)))
    assert np.array_equal(runs[0].trace_expl.view(np.int64), runs[1].trace_expl.view(np.int64))
