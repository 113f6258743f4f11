"""GPU parity of the implicit Kronecker engine (kr_engine_create_kron).

The implicit engine sums in a different order from both the reference's
referenceMatvec (kron.hpp:211-254) and the factored engine, so the bar is the
north star's floating-point tolerance, written here: normwise
max|got − exp| ≤ 1e-12 · (1 + max|exp|) — against the oracle's
referenceMatvec(T) on the small corpus and against the (bitwise-pinned)
factored engine on the full-size configs.  DCFR driven by the implicit
engine must reproduce the factored solve's exploitability to 1e-7 relative.
"""
import ctypes as C

import numpy as np
import pytest

import pyoracle as po
from paper_2112_03804_b200 import CudaEngine, InvalidInputError
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for

pytestmark = pytest.mark.gpu

TOL = 1e-12


def normwise(got, exp):
    return np.abs(got - exp).max() / (1 + np.abs(exp).max())


CASES = [("golden", {}), ("twenty_card", {}), ("bluffing", {}), ("all_tie", {}),
         ("random_small", dict(seed=3)), ("random_small", dict(seed=5)), ("bench", dict(seed=2, hands=100)),
         ("river_full", dict(seed=2, board="Kc9d7c4d2c", deck=26, tree=3))]


@pytest.mark.parametrize("name,kw", CASES)
def test_kron_matches_reference_matvec(name, kw):
    p = H.builtin(name, **kw)
    o = po.Instance.builtin(name, **kw)
    eng = CudaEngine.kron(p)
    assert (eng.rows, eng.cols) == (p.rows, p.cols)
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(3):
        x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
        e1 = normwise(eng.Ax(x), o.reference_matvec(x))
        e2 = normwise(eng.ATx(y), o.reference_matvec_t(y))
        worst = max(worst, e1, e2)
    assert worst <= TOL, worst


@pytest.mark.parametrize("seq,per_product", [("0", 1), ("1", 3)])
def test_kron_launches_and_flops(seq, per_product, monkeypatch):
    # KR_KRON_SEQ=0: one fused kernel per product; =1: transpose, fused
    # kernel, transpose
    monkeypatch.setenv("KR_KRON_SEQ", seq)
    p = H.builtin("twenty_card")
    eng = CudaEngine.kron(p)
    l0 = eng.launches()
    eng.Ax(np.ones(p.cols))
    eng.ATx(np.ones(p.rows))
    assert eng.launches() - l0 == 2 * per_product
    assert eng.last_flops() > 0 and eng.flops() >= eng.last_flops()


@pytest.mark.parametrize("tree", [1, 3])
def test_kron_config2_matches_factored(tree):
    p = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=tree)
    fac = CudaEngine(p.sparsify("b", True))
    imp = CudaEngine.kron(p)
    rng = np.random.default_rng(9)
    x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
    assert normwise(imp.Ax(x), fac.Ax(x)) <= TOL
    assert normwise(imp.ATx(y), fac.ATx(y)) <= TOL


def test_kron_multiboard_matches_factored():
    boards = H.turn_instances("Ks7d4c2h", nboards=6, tree=3)
    fac = CudaEngine([f for _, f in boards])
    imp = CudaEngine.kron([i for i, _ in boards])
    assert (imp.rows, imp.cols) == (fac.rows, fac.cols)
    rng = np.random.default_rng(2)
    for _ in range(2):
        x, y = rng.standard_normal(fac.cols), rng.standard_normal(fac.rows)
        assert normwise(imp.Ax(x), fac.Ax(x)) <= TOL
        assert normwise(imp.ATx(y), fac.ATx(y)) <= TOL


def test_kron_rejects_mixed_trees():
    a = H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=1)
    b = H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
    assert (a.n1, a.n2) != (b.n1, b.n2)
    with pytest.raises(InvalidInputError):
        CudaEngine.kron([a, b])


def test_kron_rejects_unsorted_keys():
    p = H.builtin("twenty_card")
    v = p.kron_view()
    keys = np.ctypeslib.as_array(C.cast(v.key1, C.POINTER(C.c_uint32)), (v.m1,))[::-1].copy()
    v.key1 = keys.ctypes.data
    from paper_2112_03804_b200 import _native as N
    h = C.c_void_p()
    rc = N.cuda().kr_engine_create_kron(C.byref(v), 1, 0, 0, C.byref(h))
    assert rc == 1 and not h.value


def test_kron_solver_matches_factored_golden():
    """600 DCFR iterations of twenty_card (the README's golden solve,
    exploitability 0.000189332132512) driven by the implicit engine."""
    p = H.builtin("twenty_card")
    prm = DcfrParams(max_iters=600, checkpoint_every=50)
    r_imp = solver_for([p], implicit=True).run(prm)
    r_fac = solver_for([(p, p.sparsify("b", True))]).run(prm)
    assert r_imp.iterations == r_fac.iterations == 600
    assert abs(r_imp.exploitability - r_fac.exploitability) <= 1e-7 * r_fac.exploitability
    assert abs(r_imp.exploitability - 0.000189332132512) <= 1e-7 * 0.000189332132512
    np.testing.assert_allclose(r_imp.trace_expl, r_fac.trace_expl, rtol=1e-7)


def test_kron_solver_turn_boards():
    """On four full-range turn boards DCFR amplifies the engines' different
    rounding (≈3e-14 in the averages after one iteration) about tenfold per
    ten iterations (tools/kron_diverge.py, measured on the B200): the
    trajectories agree tightly at the first checkpoint and both keep
    converging, but they are not the same trajectory at iteration 100 —
    exactly as two summation orders of referenceMatvec would not be."""
    boards = H.turn_instances("Ks7d4c2h", nboards=4, tree=3)
    prm = DcfrParams(max_iters=100, checkpoint_every=50)
    r_imp = solver_for(boards, implicit=True).run(prm)
    r_fac = solver_for(boards).run(prm)
    assert r_imp.trace_iter.tolist() == r_fac.trace_iter.tolist() == [50, 100]
    np.testing.assert_allclose(r_imp.trace_expl[0], r_fac.trace_expl[0], rtol=1e-5)
    np.testing.assert_allclose(r_imp.board_br1[0], r_fac.board_br1[0], rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(r_imp.trace_expl[1], r_fac.trace_expl[1], rtol=5e-2)
    assert r_imp.trace_expl[1] < 0.5 * r_imp.trace_expl[0]


def test_kron_mixed_hand_counts_match_factored():
    """Boards with different hand counts in one engine (1081-hand and 210-hand
    rivers sharing the 3-bet tree): every per-board offset of K7 is exercised."""
    boards = [H.builtin("river_full", seed=4, board="Ks7d4c2h9s", tree=3),
              H.builtin("river_full", seed=5, board="Kc9d7c4d2c", deck=26, tree=3),
              H.builtin("river_full", seed=6, board="AhKhQh7c7d", tree=3)]
    assert len({(b.n1, b.n2) for b in boards}) == 1 and len({b.m1 for b in boards}) == 2
    fac = CudaEngine([b.sparsify("b", True) for b in boards])
    imp = CudaEngine.kron(boards)
    rng = np.random.default_rng(8)
    x, y = rng.standard_normal(fac.cols), rng.standard_normal(fac.rows)
    assert normwise(imp.Ax(x), fac.Ax(x)) <= TOL
    assert normwise(imp.ATx(y), fac.ATx(y)) <= TOL


@pytest.mark.parametrize("groups", ["1", "3"])
def test_kron_host_pipeline_groups(groups, monkeypatch):
    """Host-buffer calls pipelined over board groups (KR_GROUPS) give the
    same bits as the device-pointer path."""
    import torch
    monkeypatch.setenv("KR_GROUPS", groups)
    boards = [i for i, _ in H.turn_instances("Ks7d4c2h", nboards=5, tree=3, factors=False)]
    eng = CudaEngine.kron(boards)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(eng.cols)
    hx = eng.Ax(x)
    dx = torch.tensor(x, device="cuda")
    dy = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    eng.ax_device(dx.data_ptr(), dy.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(hx, dy.cpu().numpy())
