"""Pins the CPU oracle (oracle/kr_oracle.hpp) to the reference's published
golden numbers and known answers, before it is trusted as the checker for the
product (CPU-only; the reference itself cannot be compiled here: Eigen3,
Catch2 and CLI11 are absent — DESIGN.md §2)."""
import json
import os

import numpy as np
import pytest

import pyoracle as po
from conftest import GOLDEN, REFERENCE


def test_twenty_card_factor_counts(golden):
    g = golden["twenty_card_b_post"]
    inst = po.Instance.builtin("twenty_card")
    assert inst.dense_nnz() == g["dense_nnz"]
    s = inst.sparsify("b", post=True)
    assert s.nnz == {"ahat": g["ahat"], "u": g["u"], "m": g["m"], "v": g["v"]}
    assert s.k == g["k"] and s.size_total() == g["size"]


def test_twenty_card_600_iteration_solve(golden):
    """README.md:81-82: exploitability 0.000189332132512, gradient_flops 67228200."""
    g = golden["twenty_card_solve_600"]
    inst = po.Instance.builtin("twenty_card")
    s = inst.sparsify("b", post=True)
    r = po.dcfr(inst, s, max_iters=600)
    assert r["iterations"] == g["iterations"]
    assert "%.12g" % r["exploitability"] == g["exploitability_12g"]
    assert r["gradient_flops"] == g["gradient_flops"]


def test_reference_tree(golden):
    g = golden["reference_tree"]
    inst = po.Instance.builtin("golden")
    assert (inst.nodes, inst.dec0, inst.dec1, inst.n1, inst.n2) == (g["nodes"], *g["decisions"], *g["sequences"])
    assert (inst.terminals, inst.folds, inst.showdowns) == (g["terminals"], g["folds"], g["showdowns"])
    ints, qs, paths = inst.terminals_table()
    got = sorted((float(a), float(b)) for a, b in qs)
    assert np.allclose(got, g["contributions_sorted"], atol=0.05)
    assert paths[0] == g["terminal0_path"] and paths[19] == g["terminal19_path"]
    assert list(ints[19, 2:]) == g["terminal19_seqs"]
    _, _, fv = inst.FS(0)
    _, _, sv = inst.FS(1)
    assert np.allclose(sorted(fv), g["F_sorted"]) and np.allclose(sorted(sv), g["S_sorted"])


def test_peel_budget_and_ones(golden):
    g = golden["peel_ones_6x8"]
    assert po.peel(np.ones((6, 8)), 0)[:2] == (0, g["what_nnz_budget0"])
    rank, what, u, v = po.peel(np.ones((6, 8)))
    assert (rank, what, u + v) == (g["rank"], 0, g["u_plus_v_nnz"])
    with pytest.raises(po.OracleError) as e:
        po.peel(np.full((3, 3), 0.5))
    assert e.value.code == "INVALID_INPUT"


def test_peel_reconstructs_staircase():
    n = 10
    W = np.array([[1.0 if i > j else (-1.0 if i < j else 0.0) for j in range(n)] for i in range(n)])
    rank, what, u, v = po.peel(W)
    assert rank > 0 and what + u + v < np.count_nonzero(W)


def test_technique_b_structure():
    """test_sparsify.cpp:279-288: k = m1 n1 + n1 and the -1 sub-diagonal."""
    inst = po.Instance.builtin("random_small", seed=3, hands=4)
    s = inst.sparsify("b", post=False)
    assert s.k == inst.m1 * inst.n1 + inst.n1
    o, i, v = s.export("m")
    for col in range((inst.m1 - 1) * inst.n1):
        assert list(i[o[col]:o[col + 1]]) == [col, col + inst.n1]
        assert list(v[o[col]:o[col + 1]]) == [1.0, -1.0]


def _terminal_walk_dense(inst):
    """Independent dense payoff (tests/oracles.hpp:120-154 restated in numpy):
    walks every terminal for every compatible hand pair."""
    ints, qs, _ = inst.terminals_table()
    h1, h2 = inst.hands(0), inst.hands(1)
    mu1, mu2, _, _ = inst.vectors()
    W, H = inst.W()
    beta = sum(mu1[i] * mu2[j] for i in range(inst.m1) for j in range(inst.m2) if H[i, j] == 0)
    A = np.zeros((inst.rows, inst.cols))
    for i in range(inst.m1):
        for j in range(inst.m2):
            if H[i, j] != 0:
                continue
            p = mu1[i] * mu2[j] / beta
            for (fold, folder, s1, s2), (q1, q2) in zip(ints, qs):
                pay = (q2 if folder == 1 else -q1) if fold else W[i, j] * q1
                A[i * inst.n1 + s1 - 1, j * inst.n2 + s2 - 1] += p * pay
    return A


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_dense_and_matvecs_against_terminal_walk(seed):
    inst = po.Instance.builtin("random_small", seed=seed)
    A = inst.dense()
    B = _terminal_walk_dense(inst)
    assert np.abs(A - B).max() < 1e-12 * np.abs(B).max()
    rng = np.random.default_rng(seed)
    scale = 1 + np.abs(A).max()
    for tech in ("a", "b"):
        for post in (False, True):
            s = inst.sparsify(tech, post)
            for _ in range(3):
                x, y = rng.standard_normal(inst.cols), rng.standard_normal(inst.rows)
                assert np.abs(s.matvec(x) - A @ x).max() < 1e-9 * scale
                assert np.abs(s.matvec_t(y) - A.T @ y).max() < 1e-9 * scale
                ax = A @ x
                assert np.abs(inst.reference_matvec(x) - ax).max() < 1e-12 * (1 + np.abs(ax).max())


def test_flop_counter_rule():
    """test_engine.cpp:133-157: identity M skips the solve in the count."""
    inst = po.Instance.builtin("random_small", seed=5)
    a = inst.sparsify("a", post=False)
    a.matvec(np.ones(inst.cols))
    assert a.last_flops == a.nnz["v"] + a.nnz["u"] + a.nnz["ahat"]
    b = inst.sparsify("b", post=False)
    b.matvec_t(np.ones(inst.rows))
    assert b.last_flops == b.nnz["v"] + b.nnz["u"] + b.nnz["ahat"] + b.nnz["m"] - b.k


def test_bluffing_solution(golden):
    g = golden["bluffing_dcfr_5000"]
    inst = po.Instance.builtin("bluffing")
    s = inst.sparsify("b", True)
    r = po.dcfr(inst, s, max_iters=5000)
    assert r["exploitability"] < g["exploitability_below"]
    value = -po.best_response(inst, s, 1, r["avg1"])
    assert abs(value - g["value"]) < g["value_tol"]
    assert abs(r["avg1"][1] - g["air_bet"]) < g["air_bet_tol"]
    assert abs(r["avg1"][inst.n1 + 1] - g["nuts_bet"]) < g["nuts_bet_tol"]
    assert abs(r["avg2"][2] - g["call"]) < g["call_tol"]


def test_all_tie_exactly_zero(golden):
    inst = po.Instance.builtin("all_tie")
    s = inst.sparsify("b", True)
    assert po.dcfr(inst, s, max_iters=400)["exploitability"] == golden["all_tie_dcfr_400"]["exploitability"]


def test_factored_vs_dense_traces():
    """test_solver.cpp:234-253 / acceptance C6: traces agree within 1e-8."""
    inst = po.Instance.builtin("random_small", seed=12021)
    s = inst.sparsify("b", True)
    rf = po.dcfr(inst, s, max_iters=150, checkpoint_every=25)
    rd = po.dcfr(inst, None, engine="dense", max_iters=150, checkpoint_every=25)
    assert np.abs(rf["trace_expl"] - rd["trace_expl"]).max() < 1e-8


def test_config_sizes_match_the_sizing_model(golden):
    g = golden["config_sizes"]
    for key, board, deck in (("config2_Ks7d4c2h9s_b_post", "Ks7d4c2h9s", 52),
                             ("config4_Kc9d7c4d2c_b_post", "Kc9d7c4d2c", 26)):
        inst = po.Instance.builtin("river_full", seed=1, board=board, deck=deck, tree=3)
        s = inst.sparsify("b", True)
        assert s.nnz == {k: g[key][k] for k in ("ahat", "u", "m", "v")} and s.k == g[key]["k"]
        assert inst.dense_nnz() == g[key]["dense_nnz"]


@pytest.mark.skipif(not os.path.isdir(REFERENCE), reason="reference tree not mounted")
def test_fixtures_match_reference_instance_files():
    with open(os.path.join(GOLDEN, "instances_v1.json")) as f:
        fx = json.load(f)
    for name, obj in fx.items():
        with open(os.path.join(REFERENCE, "instances", name + ".json")) as f:
            assert json.load(f) == obj
