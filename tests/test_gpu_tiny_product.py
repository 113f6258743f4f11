"""The fused small-engine product (kr_engine.cu k_tiny_product): the three
stages of a factored product in one cluster launch.  Every row, slice and
chain runs the separate kernels' device code, so the products must be
BITWISE the three-launch path's (KR_TINY=0) and the oracle's, for every
cluster size (the rows, slices and chains are strided over the cluster's
warps, so the cluster size changes only who computes what)."""
import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H

pytestmark = pytest.mark.gpu


def products(p, sp, monkeypatch, tiny, cluster=None, trials=2):
    monkeypatch.setenv("KR_TINY", tiny)
    if cluster is None:
        monkeypatch.delenv("KR_TINY_CLUSTER", raising=False)
    else:
        monkeypatch.setenv("KR_TINY_CLUSTER", str(cluster))
    eng = CudaEngine(sp)
    rng = np.random.default_rng(5)
    out = []
    for _ in range(trials):
        x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
        n0 = eng.launches()
        ax = eng.Ax(x)
        n1 = eng.launches()
        aty = eng.ATx(y)
        n2 = eng.launches()
        out.append((ax, aty, n1 - n0, n2 - n1))
    return out


@pytest.mark.parametrize("name,kw,tech", [
    ("twenty_card", {}, "b"),
    ("golden", {}, "b"),
    ("bluffing", {}, "b"),
    ("random_small", dict(seed=3), "b"),
    ("bench", dict(seed=2, hands=100), "b"),
    ("twenty_card", {}, "a"),   # Technique A: general M keeps the level kernels
])
@pytest.mark.parametrize("cluster", [None, 1, 2, 7, 16])
def test_tiny_product_bitwise(name, kw, tech, cluster, monkeypatch):
    p, o = H.builtin(name, **kw), po.Instance.builtin(name, **kw)
    sp = p.sparsify(tech, True)
    fused = products(p, sp, monkeypatch, "1000000000", cluster)
    plain = products(p, sp, monkeypatch, "0")
    osp = o.sparsify(tech, True)
    rng = np.random.default_rng(5)
    for (ax, aty, la, lt), (bx, bty, _, _) in zip(fused, plain):
        x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
        assert bits_equal(ax, bx) and bits_equal(aty, bty)
        assert bits_equal(ax, osp.matvec(x)) and bits_equal(aty, osp.matvec_t(y))
        if tech == "b":
            assert la == 1 and lt == 1, (la, lt)   # one launch per product


@pytest.mark.parametrize("cluster", [4, 16])
def test_tiny_product_config4_bitwise(cluster, monkeypatch):
    """The 26-card river (config 4, ~0.5 M stored entries: above the default
    limit) forced through the fused product, against the three launches."""
    p = H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
    sp = p.sparsify("b", True)
    fused = products(p, sp, monkeypatch, "1000000000", cluster, trials=1)
    plain = products(p, sp, monkeypatch, "0", trials=1)
    for (ax, aty, la, lt), (bx, bty, lb, lbt) in zip(fused, plain):
        assert bits_equal(ax, bx) and bits_equal(aty, bty)
        assert (la, lt) == (1, 1) and lb >= 3 and lbt >= 3


@pytest.mark.parametrize("name,kw", [("golden", {}), ("random_small", dict(seed=3)),
                                     ("bench", dict(seed=2, hands=100))])
def test_default_fuses_stream_products_only(name, kw, monkeypatch):
    """Defaults: a small engine's product launched on a stream is fused (one
    launch); graph-captured products (the host API's replayed calls) keep the
    three launches; same bits."""
    import torch
    monkeypatch.delenv("KR_TINY", raising=False)
    monkeypatch.delenv("KR_TINY_CLUSTER", raising=False)
    p = H.builtin(name, **kw)
    eng = CudaEngine(p.sparsify("b", True))
    rng = np.random.default_rng(9)
    x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
    for _ in range(3):   # first call direct, then captured and replayed
        ax, aty = eng.Ax(x), eng.ATx(y)
    dev = torch.device("cuda", 0)
    xd, yd = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    a = torch.empty(p.rows, dtype=torch.float64, device=dev)
    b = torch.empty(p.cols, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    n0 = eng.launches()
    eng.ax_device(xd.data_ptr(), a.data_ptr())
    eng.atx_device(yd.data_ptr(), b.data_ptr())
    assert eng.launches() - n0 == 2
    torch.cuda.synchronize(dev)
    st = torch.cuda.ExternalStream(eng.stream)
    st.synchronize()
    assert bits_equal(a.cpu().numpy(), ax) and bits_equal(b.cpu().numpy(), aty)
