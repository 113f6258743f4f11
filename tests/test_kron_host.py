"""Host side of the implicit Kronecker engine (CPU, no GPU needed).

1. krh_instance_kron_view exposes exactly the instance the factored path
   uses: keys ascending (kron.hpp:74-83), cards matching the hand strings,
   lambdas equal to the instance vectors, F / S with the advertised sizes.
2. The prefix-scan / inclusion–exclusion restatement that k_kron_weights,
   k_kron_scan and k_kron_combine implement (kr_kron.cu header), written
   here in numpy as test infrastructure, reproduces the oracle's
   referenceMatvec / referenceMatvecT (kron.hpp:211-254) to 1e-12 normwise —
   so a GPU mismatch is a kernel bug, not a formula bug.
"""
import ctypes as C

import numpy as np
import pytest

import pyoracle as po
from paper_2112_03804_b200 import host as H

TOL = 1e-12
RANKS, SUITS = "23456789TJQKA", "cdhs"


def card_id(s):
    return RANKS.index(s[0]) * 4 + SUITS.index(s[1])


def csr(c, ncols):
    no = c.outer_size
    outer = np.ctypeslib.as_array(C.cast(c.outer, C.POINTER(C.c_int64)), (no + 1,)).copy()
    nnz = int(outer[-1])
    dense = np.zeros((no, ncols))
    if nnz:
        inner = np.ctypeslib.as_array(C.cast(c.inner, C.POINTER(C.c_int32)), (nnz,))
        val = np.ctypeslib.as_array(C.cast(c.val, C.POINTER(C.c_double)), (nnz,))
        for r in range(no):
            for e in range(outer[r], outer[r + 1]):
                dense[r, inner[e]] += val[e]
    return dense


def kron_arrays(inst):
    v = inst.kron_view()
    m = (v.m1, v.m2)
    out = {"m": m, "n": (v.n1, v.n2)}
    out["key"] = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint32)), (mm,)).copy()
                  for p, mm in ((v.key1, m[0]), (v.key2, m[1]))]
    out["cards"] = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), (2 * mm,)).reshape(mm, 2).copy()
                    for p, mm in ((v.cards1, m[0]), (v.cards2, m[1]))]
    out["lam"] = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), (mm,)).copy()
                  for p, mm in ((v.lambda1, m[0]), (v.lambda2, m[1]))]
    out["F"], out["S"] = csr(v.F, v.n2), csr(v.S, v.n2)
    return out


def implicit_product(k, vec, direction):
    """The three-kernel algorithm of kr_kron.cu, restated sequentially."""
    O, S = (0, 1) if direction == 0 else (1, 0)
    Fd, Sd = (k["F"], k["S"]) if direction == 0 else (k["F"].T, k["S"].T)
    mO, mS = k["m"][O], k["m"][S]
    nO, nS = k["n"][O], k["n"][S]
    sign = 1.0 if direction == 0 else -1.0
    V = vec.reshape(mS, nS)
    WF = k["lam"][S][:, None] * (V @ Fd.T)  # [j, a]
    WS = k["lam"][S][:, None] * (V @ Sd.T)
    PS = np.vstack([np.zeros((1, nO)), np.cumsum(WS, axis=0)])
    TF, TS = WF.sum(axis=0), WS.sum(axis=0)
    kS, cS = k["key"][S], k["cards"][S]
    lists = [np.flatnonzero((cS == c).any(axis=1)) for c in range(52)]
    out = np.zeros((mO, nO))
    for i in range(mO):
        key = k["key"][O][i]
        c1, c2 = k["cards"][O][i]
        lt, le = np.searchsorted(kS, key, "left"), np.searchsorted(kS, key, "right")
        fpart = TF.copy()
        lower, upper = PS[lt].copy(), TS - PS[le]
        for c in (c1, c2):
            L = lists[c]
            cps = np.vstack([np.zeros((1, nO)), np.cumsum(WS[L], axis=0)])
            fpart -= WF[L].sum(axis=0)
            a, b = np.searchsorted(kS[L], key, "left"), np.searchsorted(kS[L], key, "right")
            lower -= cps[a]
            upper -= cps[-1] - cps[b]
        dup = [j for j in lists[c1] if set(cS[j]) == {c1, c2}]
        if dup:
            fpart += WF[dup[0]]
        out[i] = k["lam"][O][i] * (fpart + sign * (lower - upper))
    return out.ravel()


CASES = [("golden", {}), ("twenty_card", {}), ("bluffing", {}), ("all_tie", {}),
         ("random_small", dict(seed=3)), ("random_small", dict(seed=5)),
         ("river_full", dict(seed=2, board="Kc9d7c4d2c", deck=26, tree=3))]


@pytest.mark.parametrize("name,kw", CASES)
def test_kron_view_matches_instance(name, kw):
    p = H.builtin(name, **kw)
    k = kron_arrays(p)
    assert k["m"] == (p.m1, p.m2) and k["n"] == (p.n1, p.n2)
    _, _, l1, l2 = p.vectors()
    assert np.array_equal(k["lam"][0], l1) and np.array_equal(k["lam"][1], l2)
    for pl in (0, 1):
        assert np.all(np.diff(k["key"][pl].astype(np.int64)) >= 0)
        hands = p.hands(pl)
        ids = np.array([[card_id(h[:2]), card_id(h[2:])] for h in hands])
        assert np.array_equal(np.sort(ids, axis=1), np.sort(k["cards"][pl], axis=1))
    assert np.count_nonzero(k["F"]) <= p.nnzF and np.count_nonzero(k["S"]) <= p.nnzS


@pytest.mark.parametrize("name,kw", CASES)
def test_implicit_algorithm_matches_reference_matvec(name, kw):
    p = H.builtin(name, **kw)
    o = po.Instance.builtin(name, **kw)
    k = kron_arrays(p)
    rng = np.random.default_rng(11)
    for _ in range(2):
        x, y = rng.standard_normal(p.cols), rng.standard_normal(p.rows)
        ax, ex = implicit_product(k, x, 0), o.reference_matvec(x)
        aty, ey = implicit_product(k, y, 1), o.reference_matvec_t(y)
        assert np.abs(ax - ex).max() <= TOL * (1 + np.abs(ex).max())
        assert np.abs(aty - ey).max() <= TOL * (1 + np.abs(ey).max())
