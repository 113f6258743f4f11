"""GPU parity of the Kronecker-factored engine (kr_engine_create_kfactored).

The engine keeps Technique B post as its hand-space factors and the tree's F
and S and expands every Kronecker product on the fly (kr_kfengine.cu).  Its
contract is the factored engine's: BITWISE equality with the oracle's
matvec / matvecTranspose (engine.hpp:58-133) on the Technique B post factors,
and therefore bitwise DCFR gap trajectories (solver.hpp:343-404).  The
north star's 1e-12 normwise bound is asserted as the weaker statement."""
import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal
from paper_2112_03804_b200 import CudaEngine, InvalidInputError
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import CudaSolver, DcfrParams

pytestmark = pytest.mark.gpu

TOL = 1e-12


def normwise(got, exp):
    return np.abs(got - exp).max() / (1 + np.abs(exp).max())


def corpus():
    out = [(n, {}) for n in ("golden", "twenty_card", "bluffing", "all_tie")]
    out += [("random_small", dict(seed=s)) for s in range(8)]
    out += [("bench", dict(seed=2, hands=100)), ("bench", dict(seed=5, hands=300, shared=40))]
    out += [("river_full", dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3))]
    return out


def check(eng, sps, rng, trials=2, scale=1.0):
    cx = np.cumsum([0] + [s.cols for s in sps])
    cy = np.cumsum([0] + [s.rows for s in sps])
    for _ in range(trials):
        x, y = scale * rng.standard_normal(eng.cols), scale * rng.standard_normal(eng.rows)
        ax, aty = eng.Ax(x), eng.ATx(y)
        ex = np.concatenate([sp.matvec(x[cx[b]:cx[b + 1]]) for b, sp in enumerate(sps)])
        ey = np.concatenate([sp.matvec_t(y[cy[b]:cy[b + 1]]) for b, sp in enumerate(sps)])
        assert normwise(ax, ex) <= TOL and normwise(aty, ey) <= TOL
        assert bits_equal(ax, ex), "Ax differs from the oracle"
        assert bits_equal(aty, ey), "ATx differs from the oracle"


class _Sp:
    def __init__(self, sp, rows, cols):
        self.sp, self.rows, self.cols = sp, rows, cols

    def matvec(self, x):
        return self.sp.matvec(x)

    def matvec_t(self, y):
        return self.sp.matvec_t(y)


def oracle_b(name, kw):
    o = po.Instance.builtin(name, **kw)
    return _Sp(o.sparsify("b", True), o.rows, o.cols)


@pytest.mark.parametrize("name,kw", corpus())
def test_products_bitwise(name, kw):
    p = H.builtin(name, **kw)
    eng = CudaEngine.kfactored(p)
    check(eng, [oracle_b(name, kw)], np.random.default_rng(11), trials=3)
    f = p.sparsify("b", True)
    assert eng.nnz == f.nnz and eng.k == f.k
    eng.Ax(np.ones(eng.cols))
    assert eng.last_flops() == f.nnz["v"] + f.nnz["u"] + f.nnz["ahat"] + f.nnz["m"] - f.k


@pytest.mark.parametrize("board,v", [("Ks7d4c2h9s", 3390846), ("AhKhQh7c7d", 2049828)], ids=["dry", "wet"])
def test_config2_products_bitwise(board, v):
    kw = dict(seed=1, board=board, tree=3)
    eng = CudaEngine.kfactored(H.builtin("river_full", **kw))
    assert eng.nnz == {"ahat": 2754388, "u": 61617, "m": 62697, "v": v}
    check(eng, [oracle_b("river_full", kw)], np.random.default_rng(3))


def test_tiny_and_huge_inputs_take_the_literal_path_bitwise():
    """Inputs whose products would be subnormal (or near overflow) void the
    Y-factoring rewrite; the kernels detect that per CTA and evaluate the
    literal expressions, so the bits still match the oracle."""
    kw = dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
    eng = CudaEngine.kfactored(H.builtin("river_full", **kw))
    sp = oracle_b("river_full", kw)
    rng = np.random.default_rng(5)
    for scale in (1e-310, 1e-300, 1e280):
        check(eng, [sp], rng, trials=1, scale=scale)
    x = rng.standard_normal(eng.cols)
    x[::7] *= 1e-312   # a mix: most CTAs fast, some literal
    assert bits_equal(eng.Ax(x), sp.matvec(x))


@pytest.mark.parametrize("groups", ["1", "3", "8"])
def test_multiboard_and_host_pipeline_bitwise(groups, monkeypatch):
    monkeypatch.setenv("KR_GROUPS", groups)
    specs = [dict(seed=10 + k, board=b, deck=26, tree=3)
             for k, b in enumerate(["Kc9d7c4d2c", "Ac8d6c3d2d", "QcJd9c5d3c", "Tc7d5c4d2c"])]
    eng = CudaEngine.kfactored([H.builtin("river_full", **s) for s in specs])
    check(eng, [oracle_b("river_full", s) for s in specs], np.random.default_rng(4))


def test_matches_device_built_and_pair_call():
    import torch
    insts = [i for i, _ in H.turn_instances(nboards=3, factors=False)]
    kf, db = CudaEngine.kfactored(insts), CudaEngine.device_built(insts)
    assert kf.nnz == db.nnz and kf.k == db.k
    x = torch.randn(kf.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(kf.rows, dtype=torch.float64, device="cuda")
    a1, t1 = torch.empty_like(y), torch.empty_like(x)
    a2, t2 = torch.empty_like(y), torch.empty_like(x)
    torch.cuda.synchronize()
    db.ax_device(x.data_ptr(), a1.data_ptr())
    db.atx_device(y.data_ptr(), t1.data_ptr())
    torch.cuda.ExternalStream(db.stream).synchronize()
    for _ in range(3):
        kf.pair_device(x.data_ptr(), a2.data_ptr(), y.data_ptr(), t2.data_ptr())
    torch.cuda.ExternalStream(kf.stream).synchronize()
    assert torch.equal(a1, a2) and torch.equal(t1, t2)


@pytest.mark.parametrize("name,kw,iters,every", [
    ("twenty_card", {}, 1000, 1),
    ("river_full", dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3), 100, 1),
    ("river_full", dict(seed=1, board="Ks7d4c2h9s", tree=3), 100, 10),
])
def test_dcfr_gap_trajectory_bitwise(name, kw, iters, every):
    """dcfrSolve driven by the Kronecker-factored engine: the whole gap
    trajectory, averages and flop count bitwise equal to the oracle's."""
    p = H.builtin(name, **kw)
    o = po.Instance.builtin(name, **kw)
    eng = CudaEngine.kfactored(p)
    s = CudaSolver(eng, p.treeplex(0), p.treeplex(1), [p.m1], [p.m2], p.pot)
    r = s.run(DcfrParams(max_iters=iters, checkpoint_every=every))
    ro = po.dcfr(o, o.sparsify("b", True), max_iters=iters, checkpoint_every=every)
    assert bits_equal(r.trace_expl, ro["trace_expl"])
    assert bits_equal(r.trace_br1, ro["trace_br1"]) and bits_equal(r.trace_br2, ro["trace_br2"])
    assert bits_equal(r.avg1, ro["avg1"]) and bits_equal(r.avg2, ro["avg2"])
    assert r.gradient_flops == ro["gradient_flops"]


def test_readme_golden_solve():
    """The README's 600-iteration twenty_card solve (README.md:81-82)."""
    p = H.builtin("twenty_card")
    eng = CudaEngine.kfactored(p)
    r = CudaSolver(eng, p.treeplex(0), p.treeplex(1), [p.m1], [p.m2], p.pot).run(DcfrParams(max_iters=600))
    assert r.exploitability == 0.0001893321325118753
    assert r.gradient_flops == 67228200


def test_rejects_bad_boards():
    p = H.builtin("twenty_card")
    v = p.kron_view()
    v.m1 = 3000
    with pytest.raises(InvalidInputError):
        _create_kf([v])


def _create_kf(views):
    import ctypes as C

    from paper_2112_03804_b200 import _native as N
    arr = (N.kr_kron_board * len(views))(*views)
    h = C.c_void_p()
    N.check(N.cuda().kr_engine_create_kfactored(arr, len(views), 0, 0, C.byref(h)))
