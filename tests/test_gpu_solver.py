"""GPU DCFR solver (kr_solver C ABI) against the CPU oracle's dcfrSolve.

With bitwise-equal gradients and per-hand walks replaying the reference's
arithmetic order, the per-iteration saddle-point gap trajectory (br1 + br2,
checkpointEvery = 1) is asserted BITWISE equal to the oracle's, which
implies the north star's 1e-12 relative tolerance.  The golden 600-iteration
twenty-card solve (README.md:81-82) is reproduced on the device."""
import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal
from paper_2112_03804_b200 import InvalidInputError
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, dcfr_solve, solver_for

pytestmark = pytest.mark.gpu


def both(name, **kw):
    return H.builtin(name, **kw), po.Instance.builtin(name, **kw)


def test_golden_twenty_card_600(golden):
    g = golden["twenty_card_solve_600"]
    p, o = both("twenty_card")
    fp = p.sparsify("b", True)
    r = dcfr_solve(p, fp, DcfrParams(max_iters=600))
    ro = po.dcfr(o, o.sparsify("b", True), max_iters=600)
    assert "%.12g" % r.exploitability == g["exploitability_12g"]
    assert r.gradient_flops == g["gradient_flops"]
    assert r.iterations == 600
    assert bits_equal(r.exploitability, ro["exploitability"])
    assert bits_equal(r.avg1, ro["avg1"]) and bits_equal(r.avg2, ro["avg2"])
    assert bits_equal(r.trace_br1, ro["trace_br1"]) and bits_equal(r.trace_br2, ro["trace_br2"])


def gap_trajectory_case(name, kw, tech, iters):
    p, o = both(name, **kw)
    r = dcfr_solve(p, p.sparsify(tech, True), DcfrParams(max_iters=iters, checkpoint_every=1))
    ro = po.dcfr(o, o.sparsify(tech, True), max_iters=iters, checkpoint_every=1)
    gap, gap_o = r.trace_br1 + r.trace_br2, ro["trace_br1"] + ro["trace_br2"]
    assert len(gap) == iters
    rel = np.abs(gap - gap_o).max() / (1 + np.abs(gap_o).max())
    assert rel <= 1e-12
    assert bits_equal(r.trace_br1, ro["trace_br1"]) and bits_equal(r.trace_br2, ro["trace_br2"])
    assert bits_equal(r.trace_expl, ro["trace_expl"])
    assert bits_equal(r.avg1, ro["avg1"]) and bits_equal(r.avg2, ro["avg2"])
    assert r.gradient_flops == ro["gradient_flops"]


@pytest.mark.parametrize("name,kw,tech,iters", [
    ("twenty_card", {}, "b", 1000),
    ("twenty_card", {}, "a", 300),
    ("golden", {}, "b", 1000),
    ("bluffing", {}, "b", 1000),
    ("all_tie", {}, "b", 400),
    ("random_small", dict(seed=1), "b", 500),
    ("random_small", dict(seed=4), "a", 500),
    ("bench", dict(seed=7, hands=60), "b", 300),
])
def test_gap_trajectory_bitwise(name, kw, tech, iters):
    gap_trajectory_case(name, kw, tech, iters)


def test_config4_trajectory_bitwise():
    gap_trajectory_case("river_full", dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3), "b", 100)


def test_config2_trajectory_bitwise():
    p, o = both("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    r = dcfr_solve(p, p.sparsify("b", True), DcfrParams(max_iters=40, checkpoint_every=4))
    ro = po.dcfr(o, o.sparsify("b", True), max_iters=40, checkpoint_every=4)
    assert bits_equal(r.trace_br1, ro["trace_br1"]) and bits_equal(r.trace_br2, ro["trace_br2"])
    assert bits_equal(r.avg1, ro["avg1"])


def test_multiboard_turn_matches_independent_boards():
    """Config 3 semantics: the board dimension is block diagonal, each board's
    trajectory equals its own reference run, expl = mean over boards."""
    boards = H.turn_instances(nboards=3)
    solver = solver_for(boards)
    r = solver.run(DcfrParams(max_iters=30, checkpoint_every=10))
    expl = np.zeros(len(r.trace_iter))
    for b, (inst, f) in enumerate(boards):
        card, seed = H.turn_boards(nboards=3)[b]
        o = po.Instance.builtin("river_full", seed=seed, board="Ks7d4c2h" + card, tree=3)
        ro = po.dcfr(o, o.sparsify("b", True), max_iters=30, checkpoint_every=10)
        assert bits_equal(r.board_br1[:, b], ro["trace_br1"]) and bits_equal(r.board_br2[:, b], ro["trace_br2"])
        expl += ro["trace_expl"]
    assert np.allclose(r.trace_expl, expl / len(boards), rtol=1e-14, atol=0)


def test_known_answers_bluffing(golden):
    g = golden["bluffing_dcfr_5000"]
    p = H.builtin("bluffing")
    f = p.sparsify("b", True)
    s = solver_for([(p, f)])
    r = s.run(DcfrParams(max_iters=5000))
    assert r.exploitability < g["exploitability_below"]
    assert abs(-s.best_response(1, r.avg1) - g["value"]) < g["value_tol"]
    assert abs(r.avg1[1] - g["air_bet"]) < g["air_bet_tol"]
    assert abs(r.avg1[p.n1 + 1] - g["nuts_bet"]) < g["nuts_bet_tol"]
    assert abs(r.avg2[2] - g["call"]) < g["call_tol"]
    r0 = s.run(DcfrParams(max_iters=100000, target_exploitability=0.01))
    assert r0.iterations < 100000 and r0.exploitability <= 0.01


def test_best_response_validation_and_value():
    p, o = both("random_small", seed=3)
    s = solver_for([(p, p.sparsify("b", True))])
    u2 = o.uniform(1)
    assert bits_equal(s.best_response(0, u2), po.best_response(o, o.sparsify("b", True), 0, u2))
    bad = u2.copy()
    bad[0] = -0.25
    with pytest.raises(InvalidInputError):
        s.best_response(0, bad)
    leaky = u2.copy()
    leaky[1] += 0.5
    with pytest.raises(InvalidInputError):
        s.best_response(0, leaky)
    with pytest.raises(InvalidInputError):
        s.best_response(0, np.zeros(5))


def test_solver_rejects_bad_parameters():
    p = H.builtin("bluffing")
    s = solver_for([(p, p.sparsify("b", True))])
    with pytest.raises(InvalidInputError):
        s.run(DcfrParams(max_iters=0))
    with pytest.raises(InvalidInputError):
        s.run(DcfrParams(max_iters=10, checkpoint_every=0))


@pytest.mark.parametrize("preset", ["cfr_plus", "prm_plus"])
@pytest.mark.parametrize("name,kw,iters", [("twenty_card", {}, 400), ("golden", {}, 300), ("bluffing", {}, 300),
                                           ("random_small", dict(seed=2), 200)])
def test_rule_presets_bitwise(preset, name, kw, iters):
    """CFR+ and PRM+ (beyond the reference: its only solver is DCFR) against
    the oracle's restatement of the same rules, gap trajectory per iteration."""
    p, o = both(name, **kw)
    prm = getattr(DcfrParams, preset)(max_iters=iters, checkpoint_every=1)
    r = dcfr_solve(p, p.sparsify("b", True), prm)
    ro = po.dcfr(o, o.sparsify("b", True), alpha=prm.alpha, beta=prm.beta, gamma=prm.gamma, max_iters=iters,
                 checkpoint_every=1, rule=prm.rule)
    assert bits_equal(r.trace_br1, ro["trace_br1"]) and bits_equal(r.trace_br2, ro["trace_br2"])
    assert bits_equal(r.avg1, ro["avg1"]) and bits_equal(r.avg2, ro["avg2"])
    assert r.trace_expl[-1] <= r.trace_expl[0]


def test_cfr_plus_config1_1000_iterations():
    """BASELINE.json config 1's "1000 CFR+ iterations" on the parity game
    (twenty_card plays the Leduc role): completes and converges."""
    p = H.builtin("twenty_card")
    r = dcfr_solve(p, p.sparsify("b", True), DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=100))
    assert r.iterations == 1000
    assert r.exploitability < 1e-3
    assert r.trace_expl[-1] < 0.2 * r.trace_expl[0]


@pytest.mark.parametrize("knob", [("KR_STEP", "thread"), ("KR_TEAM", "2"), ("KR_TEAM", "8"), ("KR_NO_GRAPH", "1"),
                                  ("KR_CHAIN", "reg"), ("KR_NO_LEAN", "1"), ("KR_PF", "2"), ("KR_LPT_ALL", "1"),
                                  ("KR_BR_SERIAL", "1"), ("KR_SELL_COMP", "1"), ("KR_ORDER", "sm"),
                                  ("KR_TEAM_THREADS", "256"), ("KR_PDL", "0"), ("KR_PDL_MAXGRID", "100000"), ("KR_PDL_MAXPREV", "100000"),
                                  ("KR_XSEQ", "1")])
def test_knobs_keep_the_bits(knob, monkeypatch):
    """Every execution variant reproduces the oracle's gap
    trajectory bitwise."""
    monkeypatch.setenv(*knob)
    gap_trajectory_case("golden", {}, "b", 200)


def test_selfcheck_mode_passes_and_catches_a_tampered_factor():
    """SelfCheckEngine (solver.hpp:67-99) on the device: the factored engine's
    products replayed through the implicit engine (the block formula) pass at
    the reference's tolerance; a U entry multiplied by 3 (the reference's own
    fault injection, test_solver.cpp:217-232) fails the first check with
    ContractError, through the host calls and through a solver run."""
    from paper_2112_03804_b200 import ContractError, CudaEngine
    p = H.builtin("twenty_card")
    f = p.sparsify("b", True)
    eng, ref = CudaEngine(f), CudaEngine.kron(p)
    eng.set_selfcheck(ref, every=1, tol=1e-8)
    x = np.random.default_rng(0).standard_normal(f.cols)
    eng.Ax(x)
    eng.ATx(np.ones(f.rows))
    r = solver_for([(p, f)]).run(DcfrParams(max_iters=5))  # its own engine: unchecked
    s = solver_for([(p, f)])
    s.engine.set_selfcheck(ref, every=7, tol=1e-8)
    r2 = s.run(DcfrParams(max_iters=40, checkpoint_every=10))
    assert bits_equal(r2.trace_expl, solver_for([(p, f)]).run(DcfrParams(max_iters=40, checkpoint_every=10)).trace_expl)
    checks, worst = s.engine.selfcheck_status()
    assert checks == (2 * 40 + 2 * 4 + 6) // 7 and worst < 1e-3
    # fault injection: one U entry x 3
    arr = f.factors()
    uo, ui, uv = arr["u"]
    uv = uv.copy()
    uv[len(uv) // 2] *= 3.0
    bad = CudaEngine(dict(arr, rows=f.rows, cols=f.cols, k=f.k, u=(uo, ui, uv)))
    bad.set_selfcheck(ref, every=500, tol=1e-8)
    with pytest.raises(ContractError):
        bad.Ax(x)   # call 0 is checked (calls_++ % every_ == 0)
    assert r.iterations == 5
