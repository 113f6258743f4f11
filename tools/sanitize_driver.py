"""Exercise every libkrcuda kernel family once on small inputs, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Run as: compute-sanitizer --tool <tool> python tools/sanitize_driver.py [part]
Parts: engine (factored SELL SpMV, long rows, x' transpose, TMA chain ring,
level-scheduled solve, host pipeline, pair call), kron (K7), devb (device-built
factors and engine), solver (team step, best responses, graphs), turn (turn
solver), kf (Kronecker-factored engine, when built).  Each part checks its
results against the CPU oracle so a sanitizer run is also a parity run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import pyoracle as po  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402


def beq(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


BOARDS = ["Kc9d7c4d2c", "Ac8d6c3d2d", "QcJd9c5d3c"]


def deck26():
    ps = [H.builtin("river_full", seed=10 + k, board=b, deck=26, tree=3) for k, b in enumerate(BOARDS)]
    os_ = [po.Instance.builtin("river_full", seed=10 + k, board=b, deck=26, tree=3) for k, b in enumerate(BOARDS)]
    return ps, os_


def expect(os_, x, y):
    sps = [o.sparsify("b", True) for o in os_]
    cx = np.cumsum([0] + [o.cols for o in os_])
    cy = np.cumsum([0] + [o.rows for o in os_])
    ex = np.concatenate([sp.matvec(x[cx[b]:cx[b + 1]]) for b, sp in enumerate(sps)])
    ey = np.concatenate([sp.matvec_t(y[cy[b]:cy[b + 1]]) for b, sp in enumerate(sps)])
    return ex, ey


def part_engine():
    import torch
    f = H.builtin("twenty_card").sparsify("b", True)
    o = po.Instance.builtin("twenty_card").sparsify("b", True)
    eng = CudaEngine(f)
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(f.cols), rng.standard_normal(f.rows)
    assert beq(eng.Ax(x), o.matvec(x)) and beq(eng.ATx(y), o.matvec_t(y))
    # long rows, x' copy, three board groups, pair call
    os.environ.update(KR_LONG_ROW="32", KR_XSEQ="1", KR_GROUPS="3")
    ps, os_ = deck26()
    eng = CudaEngine([p.sparsify("b", True) for p in ps])
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ex, ey = expect(os_, x, y)
    assert beq(eng.Ax(x), ex) and beq(eng.ATx(y), ey)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    oa, ob = torch.empty_like(dy), torch.empty_like(dx)
    torch.cuda.synchronize()
    eng.pair_device(dx.data_ptr(), oa.data_ptr(), dy.data_ptr(), ob.data_ptr())
    torch.cuda.ExternalStream(eng.stream).synchronize()
    assert beq(oa.cpu().numpy(), ex) and beq(ob.cpu().numpy(), ey)
    for k in ("KR_LONG_ROW", "KR_XSEQ", "KR_GROUPS"):
        del os.environ[k]
    # register-pipeline chain and the level-scheduled general M
    os.environ["KR_CHAIN"] = "reg"
    eng = CudaEngine(H.builtin("twenty_card").sparsify("b", True))
    x = rng.standard_normal(eng.cols)
    assert beq(eng.Ax(x), po.Instance.builtin("twenty_card").sparsify("b", True).matvec(x))
    del os.environ["KR_CHAIN"]
    fa = H.builtin("random_small", seed=2).sparsify("b", False)
    arr = fa.factors()
    k = fa.k
    cols = []
    for j in range(k):
        rows = [j] + sorted(i for i in range(j + 1, k) if rng.uniform() < 0.05)
        cols.append((rows, [1.0] + list(rng.uniform(-1, 1, len(rows) - 1))))
    arr["m"] = (np.cumsum([0] + [len(r) for r, _ in cols]).astype(np.int64),
                np.concatenate([r for r, _ in cols]).astype(np.int32), np.concatenate([v for _, v in cols]))
    eng = CudaEngine(dict(arr, rows=fa.rows, cols=fa.cols, k=k))
    osp = po.Sparsification.from_arrays(fa.rows, fa.cols, k, arr)
    x, y = rng.standard_normal(fa.cols), rng.standard_normal(fa.rows)
    assert beq(eng.Ax(x), osp.matvec(x)) and beq(eng.ATx(y), osp.matvec_t(y))
    print("engine ok")


def part_kron():
    ps, os_ = deck26()
    eng = CudaEngine.kron(ps)
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ex, ey = expect(os_, x, y)
    ax, aty = eng.Ax(x), eng.ATx(y)
    assert np.abs(ax - ex).max() <= 1e-12 * (1 + np.abs(ex).max())
    assert np.abs(aty - ey).max() <= 1e-12 * (1 + np.abs(ey).max())
    print("kron ok")


def part_devb():
    ps, os_ = deck26()
    eng = CudaEngine.device_built(ps)
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ex, ey = expect(os_, x, y)
    assert beq(eng.Ax(x), ex) and beq(eng.ATx(y), ey)
    fd = ps[0].sparsify_device()
    assert fd.size() == os_[0].sparsify("b", True).size_total()
    print("devb ok")


def part_solver():
    inst = H.builtin("twenty_card")
    f = inst.sparsify("b", True)
    o = po.Instance.builtin("twenty_card")
    so = o.sparsify("b", True)
    r = solver_for([(inst, f)]).run(DcfrParams(max_iters=12, checkpoint_every=4))
    ro = po.dcfr(o, so, max_iters=12, checkpoint_every=4)
    assert beq(r.trace_expl, ro["trace_expl"])
    os.environ["KR_NO_GRAPH"] = "1"
    r = solver_for([(inst, f)]).run(DcfrParams(max_iters=6, checkpoint_every=3))
    del os.environ["KR_NO_GRAPH"]
    ps, _ = deck26()
    r = solver_for(ps, implicit=True).run(DcfrParams(max_iters=6, checkpoint_every=3))
    assert np.isfinite(r.exploitability)
    print("solver ok")


def part_turn():
    from paper_2112_03804_b200.turn import TurnGame, TurnSolver
    g = TurnGame()
    r = TurnSolver(g).run(max_iters=3, checkpoint_every=1)
    assert r["iterations"] == 3
    print("turn ok")


def part_kf():
    if not hasattr(CudaEngine, "kfactored"):
        print("kf: not built")
        return
    ps, os_ = deck26()
    eng = CudaEngine.kfactored(ps)
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ex, ey = expect(os_, x, y)
    assert beq(eng.Ax(x), ex) and beq(eng.ATx(y), ey)
    print("kf ok")


PARTS = dict(engine=part_engine, kron=part_kron, devb=part_devb, solver=part_solver, turn=part_turn, kf=part_kf)

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(PARTS)):
        PARTS[name]()
