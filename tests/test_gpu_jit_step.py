"""The DCFR player step compiled for the instance's treeplex (kr_jit.cu).

The compiled step performs the reference's per-node operations in the
reference's order, like the generic team kernel, so every result must be
BITWISE the team kernel's and the oracle's:
* the oracle's gap trajectories (checkpointEvery = 1) on the corpus trees
  with the compiled step forced (KR_STEP=jit: small instances end in partial
  32-hand tiles, `bench` with 60 hands has a full TMA tile and a partial one);
* a 12-board turn (12,972 hands per player: the compiled step is the default
  there) against KR_STEP=team for DCFR, CFR+ and PRM+, through the graph-
  replayed run and the incremental iterate path."""
import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, dcfr_solve, jit_step_source, solver_for

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kw,tech,iters", [
    ("twenty_card", {}, "b", 300),
    ("golden", {}, "b", 300),
    ("bluffing", {}, "b", 300),
    ("all_tie", {}, "b", 100),
    ("random_small", dict(seed=1), "b", 200),
    ("random_small", dict(seed=5), "a", 150),
    ("random_small", dict(seed=9), "b", 150),
    ("bench", dict(seed=7, hands=60), "b", 200),
    ("bench", dict(seed=11, hands=97), "b", 120),
])
@pytest.mark.parametrize("groups", ["1", "4"], ids=["one-thread", "four-groups"])
def test_forced_jit_gap_trajectory_bitwise(name, kw, tech, iters, groups, monkeypatch):
    """Every corpus tree through the compiled step, one thread per hand
    (KR_STEP=jit) and split over four warp groups (the single-board default),
    against the oracle's gap trajectory."""
    if groups == "1":
        monkeypatch.setenv("KR_STEP", "jit")
    else:
        monkeypatch.setenv("KR_JIT_GROUPS", "4")
    p, o = H.builtin(name, **kw), po.Instance.builtin(name, **kw)
    s = solver_for([(p, p.sparsify(tech, True))])
    if groups == "1":
        assert s.step_kind(0)[0] == 2 and s.step_kind(1)[0] == 2, s.step_kind(0)
    r = s.run(DcfrParams(max_iters=iters, checkpoint_every=1))
    ro = po.dcfr(o, o.sparsify(tech, True), max_iters=iters, checkpoint_every=1)
    assert bits_equal(r.trace_br1, ro["trace_br1"]) and bits_equal(r.trace_br2, ro["trace_br2"])
    assert bits_equal(r.avg1, ro["avg1"]) and bits_equal(r.avg2, ro["avg2"])


@pytest.fixture(scope="module")
def turn12():
    return H.turn_instances(nboards=12, factors=False)


def run_turn(boards, params, step, monkeypatch, incremental=False):
    if step == "default":
        monkeypatch.delenv("KR_STEP", raising=False)
    else:
        monkeypatch.setenv("KR_STEP", step)
    s = solver_for(boards, implicit=True)
    kinds = (s.step_kind(0)[0], s.step_kind(1)[0])
    if incremental:
        s.begin(params)
        s.iterate(params.max_iters)
        return kinds, s.averages()
    return kinds, s.run(params)


@pytest.mark.parametrize("split", ["0", "1"], ids=["one-thread", "two-groups"])
@pytest.mark.parametrize("preset", ["dcfr", "cfr_plus", "prm_plus"])
def test_turn12_jit_equals_team(turn12, preset, split, monkeypatch):
    monkeypatch.setenv("KR_JIT_SPLIT", split)
    prm = DcfrParams(max_iters=40, checkpoint_every=10) if preset == "dcfr" else \
        getattr(DcfrParams, preset)(max_iters=40, checkpoint_every=10)
    kinds, rj = run_turn(turn12, prm, "default", monkeypatch)
    assert kinds == (2, 2)
    kt, rt = run_turn(turn12, prm, "team", monkeypatch)
    assert kt == (1, 1)
    assert bits_equal(rj.trace_br1, rt.trace_br1) and bits_equal(rj.trace_br2, rt.trace_br2)
    assert bits_equal(rj.avg1, rt.avg1) and bits_equal(rj.avg2, rt.avg2)


def test_turn12_incremental_jit_equals_team(turn12, monkeypatch):
    prm = DcfrParams(max_iters=25)
    kj, aj = run_turn(turn12, prm, "default", monkeypatch, incremental=True)
    kt, at = run_turn(turn12, prm, "team", monkeypatch, incremental=True)
    assert kj == (2, 2) and kt == (1, 1)
    assert bits_equal(aj[0], at[0]) and bits_equal(aj[1], at[1])


def test_step_kind_reports_why(monkeypatch):
    p = H.builtin("twenty_card")
    monkeypatch.setenv("KR_STEP", "team")
    s = solver_for([(p, p.sparsify("b", True))])
    k, why = s.step_kind(0)
    assert k == 1 and why   # the team kernel, with the reason
    monkeypatch.delenv("KR_STEP")
    monkeypatch.setenv("KR_JIT_GROUPS", "0")
    s = solver_for([(p, p.sparsify("b", True))])
    k, why = s.step_kind(0)
    assert k == 1 and "two CTAs per SM" in why   # 105 hands, warp groups off: the team kernel
    monkeypatch.delenv("KR_JIT_GROUPS")
    s = solver_for([(p, p.sparsify("b", True))])
    assert s.step_kind(0)[0] == 2                # the tree split over warp groups
    assert "kr_step" in jit_step_source(p.treeplex(0))


@pytest.mark.parametrize("kind", ["implicit", "kfactored"])
def test_board_half_pipelining_bitwise(turn12, kind, monkeypatch):
    """The captured iteration with its board halves pipelined (each step
    beside the other half's product, kr_solver.cu overlapped_iteration)
    against the serial order (KR_OVERLAP=0): same bits."""
    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200.solver import CudaSolver

    def solve(overlap):
        monkeypatch.setenv("KR_OVERLAP", overlap)
        monkeypatch.setenv("KR_K7SEQ", "0")   # the pipelined form runs on hand-major solves
        monkeypatch.setenv("KR_KFSEQ", "0")
        insts = [i for i, _ in turn12] if isinstance(turn12[0], tuple) else list(turn12)
        eng = CudaEngine.kron(insts) if kind == "implicit" else CudaEngine.kfactored(insts)
        i0 = insts[0]
        s = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts], i0.pot)
        return s.run(DcfrParams(max_iters=30, checkpoint_every=10))  # KR_OVERLAP=1 opts in

    a, b = solve("1"), solve("0")
    assert bits_equal(a.trace_br1, b.trace_br1) and bits_equal(a.trace_br2, b.trace_br2)
    assert bits_equal(a.avg1, b.avg1) and bits_equal(a.avg2, b.avg2)
    assert a.gradient_flops == b.gradient_flops


@pytest.mark.parametrize("preset", ["dcfr", "cfr_plus", "prm_plus"])
def test_k7_sequence_major_solve_bitwise(turn12, preset, monkeypatch):
    """Implicit-engine solves keep x and the gradients sequence-major per
    board (no transposes around the coalesced K7 kernel, the compiled step
    reads and writes that layout): the same bits as the hand-major solve
    (KR_K7SEQ=0), through the graph-replayed run and iterate(1) steps."""
    prm = DcfrParams(max_iters=30, checkpoint_every=10) if preset == "dcfr" else \
        getattr(DcfrParams, preset)(max_iters=30, checkpoint_every=10)

    def solve(seq, incremental):
        monkeypatch.setenv("KR_K7SEQ", seq)
        s = solver_for(turn12, implicit=True)
        if incremental:
            s.begin(prm)
            for _ in range(12):
                s.iterate(1)
            s.iterate(5)
            return s.checkpoint(), s.averages()
        r = s.run(prm)
        return (r.trace_br1, r.trace_br2), (r.avg1, r.avg2)

    for incremental in (False, True):
        (b1, b2), (a1, a2) = solve("1", incremental)
        (c1, c2), (d1, d2) = solve("0", incremental)
        assert bits_equal(b1, c1) and bits_equal(b2, c2), incremental
        assert bits_equal(a1, d1) and bits_equal(a2, d2), incremental


@pytest.mark.parametrize("preset", ["dcfr", "prm_plus"])
def test_kf_staged_solve_bitwise(turn12, preset, monkeypatch):
    """Kronecker-factored solves keep x in the engine's staging layout (the
    compiled step writes it, kf_product_staged skips the per-product
    transpose): the same bits as the hand-major solve (KR_KFSEQ=0)."""
    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200.solver import CudaSolver
    prm = DcfrParams(max_iters=25, checkpoint_every=5) if preset == "dcfr" else \
        DcfrParams.prm_plus(max_iters=25, checkpoint_every=5)

    def solve(flag, incremental):
        monkeypatch.setenv("KR_KFSEQ", flag)
        insts = [i for i, _ in turn12]
        eng = CudaEngine.kfactored(insts)
        i0 = insts[0]
        s = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts], i0.pot)
        if incremental:
            s.begin(prm)
            for _ in range(7):
                s.iterate(1)
            s.iterate(4)
            return s.checkpoint(), s.averages()
        r = s.run(prm)
        return (r.trace_br1, r.trace_br2), (r.avg1, r.avg2)

    for incremental in (False, True):
        (b1, b2), (a1, a2) = solve("1", incremental)
        (c1, c2), (d1, d2) = solve("0", incremental)
        assert bits_equal(b1, c1) and bits_equal(b2, c2), incremental
        assert bits_equal(a1, d1) and bits_equal(a2, d2), incremental


def test_spilling_tree_keeps_the_team_kernel(monkeypatch):
    """A tree whose regrets overflow the compiled step's register budget (the
    91-sequence tree: ~2 KB of spills per thread) keeps the generic team
    kernel, which is faster there; the reason says so."""
    monkeypatch.setenv("KR_STEP", "jit")   # one thread per hand, any size
    p = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=91)
    s = solver_for([(p, p.sparsify("b", True))])
    k, why = s.step_kind(0)
    assert k == 1 and "spills" in why, (k, why)


@pytest.mark.parametrize("kind", ["kfactored"])
@pytest.mark.parametrize("board,deck", [("Kc9d7c4d2c", 26), ("Ks7d4c2h9s", 52)], ids=["config4", "config2"])
def test_single_board_sequence_major_solve_bitwise(kind, board, deck, monkeypatch):
    """Single boards (the warp-group step) in the Kronecker-factored staging
    layout against the hand-major solve: same bits.  (The implicit engine
    keeps hand-major vectors on single boards; its sequence-major warp-group
    form was measured no faster and is covered by the generator's layout
    switch.)"""
    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200.solver import CudaSolver
    p = H.builtin("river_full", seed=1, board=board, deck=deck, tree=3)

    def solve(flag):
        monkeypatch.setenv("KR_K7SEQ" if kind == "implicit" else "KR_KFSEQ", flag)
        eng = CudaEngine.kron([p]) if kind == "implicit" else CudaEngine.kfactored([p])
        s = CudaSolver(eng, p.treeplex(0), p.treeplex(1), [p.m1], [p.m2], p.pot)
        return s.run(DcfrParams(max_iters=40, checkpoint_every=10))

    a, b = solve("1"), solve("0")
    assert bits_equal(a.trace_br1, b.trace_br1) and bits_equal(a.trace_br2, b.trace_br2)
    assert bits_equal(a.avg1, b.avg1) and bits_equal(a.avg2, b.avg2)
