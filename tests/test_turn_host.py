"""Turn endgames, host side and CPU checker (no GPU).

The turn round is beyond the reference; its checker
(oracle/turn_oracle.py) composes the reference's own pieces.  Pinned here:
the game's structure, the checker's payoff blocks against the oracle's
referenceMatvec on an ordinary river instance, the adjoint identity of the
assembled products, and that the composed DCFR converges."""
import numpy as np
import pytest

import pyoracle as po
import turn_oracle as TO
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.turn import TurnGame


@pytest.fixture(scope="module")
def game():
    return TurnGame()


def test_turn_game_structure(game):
    assert game.m == 231 and len(game.rivers) == 22 and game.K == 18
    assert game.n_turn == (4, 4)
    # check-check, bet-call, check-bet-call; contributions from the S entries
    assert [(int(a), int(b), float(c)) for a, b, c in game.conts] == [(1, 1, 1875.0), (2, 4, 3750.0),
                                                                       (4, 2, 3750.0)]
    assert all(mb == 210 for mb in game.mb)
    for b, order in enumerate(game.order):  # each board keeps exactly the hands without its card
        assert sorted(order.tolist()) == [h for h in range(game.m) if game.rivers[b] not in game.hands[h]]
    assert game.size[0] == game.m * 4 + 3 * sum(game.mb) * 10


def test_block_formula_matches_reference_matvec():
    """The checker's block product Y = P X F^T + (P o W) X S^T equals the
    oracle's referenceMatvec(T) (kron.hpp:211-254) on an ordinary river."""
    from test_kron_host import kron_arrays
    p = H.builtin("river_full", seed=2, board="Kc9d7c4d2c", deck=26, tree=3)
    o = po.Instance.builtin("river_full", seed=2, board="Kc9d7c4d2c", deck=26, tree=3)
    k = kron_arrays(p)
    blk = TO.Block(dict(key=k["key"], cards=k["cards"], lam=k["lam"], F=k["F"], S=k["S"]))
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
    ax = blk.ax(x.reshape(p.m2, p.n2)).ravel()
    aty = blk.atx(y.reshape(p.m1, p.n1)).ravel()
    ex, ey = o.reference_matvec(x), o.reference_matvec_t(y)
    assert np.abs(ax - ex).max() <= 1e-12 * (1 + np.abs(ex).max())
    assert np.abs(aty - ey).max() <= 1e-12 * (1 + np.abs(ey).max())


def test_products_are_adjoint(game):
    o = TO.TurnOracle(game)
    rng = np.random.default_rng(2)
    x1, x2 = rng.standard_normal(game.size[0]), rng.standard_normal(game.size[1])
    lhs, rhs = x1 @ o.ax(x2), o.atx(x1) @ x2
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)


def test_composed_dcfr_converges(game):
    o = TO.TurnOracle(game)
    trace, (a1, a2) = o.dcfr(6, checkpoint_every=2)
    expl = [e for _, _, _, e in trace]
    assert all(e > 0 for e in expl) and expl[-1] < 0.5 * expl[0]
    # the averages are sequence-form strategies: the turn block of each hand
    # sums to one over the root node's actions
    assert np.allclose(a1[:game.m * 4].reshape(game.m, 4)[:, :2].sum(axis=1), 1.0)


def test_all_in_continuations_are_check_check_showdowns():
    g = TurnGame(turn_menu=(0.5, 1.0), turn_raise_cap=1, turn_all_in=True, stack=3000.0)
    allin = [t for t, (_, _, c) in enumerate(g.conts) if 3000.0 - (c - g.pot) <= 0]
    assert allin and all(g.n_river[t] == (1, 1) for t in allin)
    for t in allin:  # one forced check each, the showdown at the continuation's stakes
        pc = g.kron_pieces(t)[0]
        assert pc["S"].shape == (1, 1) and pc["S"][0, 0] == g.conts[t][2] and not pc["F"].any()


def test_checker_rules_keep_their_invariants(game):
    """The checker's CFR+ update leaves every regret non-negative (beta = -inf
    zeroes the negative part); PRM+ keeps the same regrets but plays the regret
    match of R + the last instantaneous regret (from R = 0 the two coincide,
    hence the random start)."""
    o = TO.TurnOracle(game)
    n1, n2 = game.size
    X2 = np.zeros(n2)
    o.update(1, np.zeros(n2), X2, None, mode1=False)
    grad = o.ax(X2)
    R0, X0 = np.random.default_rng(3).uniform(0, 50, n1), np.zeros(n1)
    o.update(0, R0, X0, None, mode1=False)
    R, X = R0.copy(), X0.copy()
    o.update(0, R, X, grad, rule=1, pos=1.0, neg=0.0)
    assert R.min() >= 0 and R.max() > 0
    Rp, Xp = R0.copy(), X0.copy()
    o.update(0, Rp, Xp, grad, rule=2, pos=1.0, neg=0.0)
    np.testing.assert_array_equal(Rp, R)  # same discounted regrets ...
    assert not np.allclose(Xp, X)  # ... different strategy (matches R + r)
