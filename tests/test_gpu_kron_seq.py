"""The sequence-major K7 product (KR_KRON_SEQ=1: k_board_transpose →
k_kron_fused<SEQ> → k_board_transpose) changes only addressing, not the
order of any sum, so it must return the same bits as the hand-major kernel —
on single boards, on boards with different hand counts, over the board-group
host pipeline, in the concurrent pair call and through a K7-driven DCFR solve.
"""
import numpy as np
import pytest

from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for

pytestmark = pytest.mark.gpu


def _products(boards, monkeypatch, seq, seed=4):
    monkeypatch.setenv("KR_KRON_SEQ", seq)
    eng = CudaEngine.kron(boards)
    rng = np.random.default_rng(seed)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    return eng.Ax(x), eng.ATx(y)


BOARDS = {
    "twenty_card": lambda: [H.builtin("twenty_card")],
    "golden": lambda: [H.builtin("golden")],
    "config4": lambda: [H.builtin("river_full", seed=2, board="Kc9d7c4d2c", deck=26, tree=3)],
    "config2": lambda: [H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)],
    "mixed": lambda: [H.builtin("river_full", seed=4, board="Ks7d4c2h9s", tree=3),
                      H.builtin("river_full", seed=5, board="Kc9d7c4d2c", deck=26, tree=3),
                      H.builtin("river_full", seed=6, board="AhKhQh7c7d", tree=3)],
    "turn5_91seq": lambda: [i for i, _ in H.turn_instances("Ks7d4c2h", nboards=5, tree=91, factors=False)],
}


@pytest.mark.parametrize("name", list(BOARDS))
def test_seq_major_bitwise(name, monkeypatch):
    boards = BOARDS[name]()
    a0, t0 = _products(boards, monkeypatch, "0")
    a1, t1 = _products(boards, monkeypatch, "1")
    assert np.array_equal(a0, a1)
    assert np.array_equal(t0, t1)


@pytest.mark.parametrize("groups", ["1", "3", "8"])
def test_seq_major_pipeline_and_pair(groups, monkeypatch):
    import torch
    monkeypatch.setenv("KR_GROUPS", groups)
    boards = [i for i, _ in H.turn_instances("Ks7d4c2h", nboards=6, tree=3, factors=False)]
    monkeypatch.setenv("KR_KRON_SEQ", "0")
    ref = CudaEngine.kron(boards)
    monkeypatch.setenv("KR_KRON_SEQ", "1")
    eng = CudaEngine.kron(boards)
    rng = np.random.default_rng(7)
    x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
    monkeypatch.setenv("KR_KRON_SEQ", "0")
    ax0, atx0 = ref.Ax(x), ref.ATx(y)
    monkeypatch.setenv("KR_KRON_SEQ", "1")
    assert np.array_equal(eng.Ax(x), ax0)       # host buffers, board groups
    assert np.array_equal(eng.ATx(y), atx0)
    dx, dy = torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda")
    dax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    datx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    eng.pair_device(dx.data_ptr(), dax.data_ptr(), dy.data_ptr(), datx.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(dax.cpu().numpy(), ax0)
    assert np.array_equal(datx.cpu().numpy(), atx0)


def test_seq_major_solver_trajectory(monkeypatch):
    boards = H.turn_instances("Ks7d4c2h", nboards=3, tree=3)
    prm = DcfrParams(max_iters=60, checkpoint_every=20)
    monkeypatch.setenv("KR_KRON_SEQ", "0")
    r0 = solver_for(boards, implicit=True).run(prm)
    monkeypatch.setenv("KR_KRON_SEQ", "1")
    r1 = solver_for(boards, implicit=True).run(prm)
    assert r0.trace_iter.tolist() == r1.trace_iter.tolist()
    assert r0.trace_expl.tolist() == r1.trace_expl.tolist()
