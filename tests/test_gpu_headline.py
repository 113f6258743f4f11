"""The headline configuration, pinned: config 3 exactly as bench.py builds it.

Turn Ks7d4c2h x 48 river boards, 1,081 hands per side, 3-bet tree, Technique
B post (2.98e8 stored nonzeros), on the engines the bench times:
  * the factored engine over kr_engine_create_boards with its default layout
    (the sequence-major x' copy is on from 1M columns, so this is the path the
    bench's `value` runs, not a knob);
  * the Kronecker-factored engine (kr_engine_create_kfactored);
  * the factored engine built on the device (kr_engine_create_device_b).
Each product is compared BITWISE, board by board, with the oracle's
matvec / matvecTranspose (engine.hpp:58-133) on the oracle's own factors; the
DCFR solve (solver.hpp:343-404, default parameters, 100 iterations,
checkpointEvery = 50) is compared bitwise per board with the oracle's dcfr on
each board (a board is an independent river under the chance root)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import CudaSolver, DcfrParams

pytestmark = pytest.mark.gpu

TURN, NB = "Ks7d4c2h", 48
THREADS = max(1, min(16, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def config3():
    boards = H.turn_instances(TURN, NB)                     # product host builder
    specs = H.turn_boards(TURN, NB)

    def oracle(b):
        card, seed = specs[b]
        o = po.Instance.builtin("river_full", seed=seed, board=TURN + card, tree=3)
        return o, o.sparsify("b", True)

    with ThreadPoolExecutor(THREADS) as ex:
        orc = list(ex.map(oracle, range(NB)))
    return boards, orc


def slices(sizes):
    c = np.cumsum([0] + list(sizes))
    return [slice(int(c[b]), int(c[b + 1])) for b in range(len(sizes))]


def oracle_products(orc, x, y):
    cs, rs = slices([o.cols for o, _ in orc]), slices([o.rows for o, _ in orc])

    def one(b):
        sp = orc[b][1]
        return sp.matvec(x[cs[b]]), sp.matvec_t(y[rs[b]])

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(one, range(len(orc))))
    return np.concatenate([a for a, _ in res]), np.concatenate([t for _, t in res])


@pytest.mark.parametrize("kind", ["factored", "kfactored", "device_built"])
def test_config3_products_bitwise(config3, kind):
    boards, orc = config3
    insts = [i for i, _ in boards]
    if kind == "factored":
        eng = CudaEngine([f for _, f in boards])
        assert eng.nnz["ahat"] + eng.nnz["u"] + eng.nnz["m"] + eng.nnz["v"] == 297897654
    elif kind == "kfactored":
        eng = CudaEngine.kfactored(insts)
    else:
        eng = CudaEngine.device_built(insts)
    assert eng.cols > 1_000_000  # the default x' layout of the factored engine
    rng = np.random.default_rng(2024)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    ex, ey = oracle_products(orc, x, y)
    ax, aty = eng.Ax(x), eng.ATx(y)
    assert bits_equal(ax, ex), f"{kind}: A x differs from the oracle"
    assert bits_equal(aty, ey), f"{kind}: A^T y differs from the oracle"
    # the device-pointer pair (what bench.py's timed region calls)
    import torch
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    oa, ob = torch.empty_like(dy), torch.empty_like(dx)
    torch.cuda.synchronize()
    eng.pair_device(dx.data_ptr(), oa.data_ptr(), dy.data_ptr(), ob.data_ptr())
    torch.cuda.ExternalStream(eng.stream).synchronize()
    assert bits_equal(oa.cpu().numpy(), ex) and bits_equal(ob.cpu().numpy(), ey)


@pytest.mark.parametrize("kind", ["factored", "kfactored"])
def test_config3_dcfr_trace_bitwise_per_board(config3, kind):
    boards, orc = config3
    i0 = boards[0][0]
    eng = CudaEngine([f for _, f in boards]) if kind == "factored" else CudaEngine.kfactored([i for i, _ in boards])
    s = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i, _ in boards], [i.m2 for i, _ in boards], i0.pot)
    # the player step runs compiled for the treeplex here (kr_jit.cu); the
    # per-board comparison below is against the oracle's own walk
    assert s.step_kind(0)[0] == 2 and s.step_kind(1)[0] == 2, (s.step_kind(0), s.step_kind(1))
    r = s.run(DcfrParams(max_iters=100, checkpoint_every=50))
    assert r.iterations == 100 and len(r.trace_iter) == 2

    def one(b):
        o, sp = orc[b]
        return po.dcfr(o, sp, max_iters=100, checkpoint_every=50)

    with ThreadPoolExecutor(THREADS) as ex:
        ro = list(ex.map(one, range(NB)))
    for b in range(NB):
        assert bits_equal(r.board_br1[:, b], ro[b]["trace_br1"]), (kind, b)
        assert bits_equal(r.board_br2[:, b], ro[b]["trace_br2"]), (kind, b)
    expl = np.sum([o["trace_expl"] for o in ro], axis=0) / NB
    np.testing.assert_allclose(r.trace_expl, expl, rtol=1e-14, atol=0)
