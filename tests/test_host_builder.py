"""The product's host side (libkrhost.so) against the CPU oracle: instance
loading, strength sorting, payoff pieces and the Technique A/B factor
structure must be bit-exact (north star: "sparsification structure (nnz
counts, index sets) bit-exact").  CPU only."""
import json
import os

import numpy as np
import pytest

import pyoracle as po
from conftest import bits_equal, factors_equal
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200._native import (ContractError, DegenerateBeliefsError, InvalidInputError, KrError,
                                           ParseError)

BUILTINS = ["golden", "twenty_card", "bluffing", "all_tie"]


def corpus():
    out = [(n, dict()) for n in BUILTINS]
    out += [("random_small", dict(seed=s)) for s in range(10)]
    out += [("random_small", dict(seed=s, hands=4)) for s in range(3)]
    out += [("bench", dict(seed=11, hands=50)), ("bench", dict(seed=5, hands=75, shared=4))]
    return out


def _pair(name, kw):
    return po.Instance.builtin(name, **kw), H.builtin(name, **kw)


@pytest.mark.parametrize("name,kw", corpus())
def test_instance_pieces_match(name, kw):
    o, p = _pair(name, kw)
    assert o.hands(0) == p.hands(0) and o.hands(1) == p.hands(1)
    assert bits_equal(o.beta, p.beta)
    for a, b in zip(o.vectors(), p.vectors()):
        assert bits_equal(a, b)
    assert (o.n1, o.n2, o.terminals, o.nnzF, o.nnzS) == (p.n1, p.n2, p.terminals, p.nnzF, p.nnzS)
    assert o.dense_nnz() == p.dense_nnz()
    for player in (0, 1):
        t = p.treeplex(player)
        flat = []
        for v in range(len(t.parent)):
            a0, a1 = t.action_ptr[v], t.action_ptr[v + 1]
            flat += [t.parent[v], a1 - a0, *t.action_seq[a0:a1]]
        assert list(o.treeplex(player)) == flat


@pytest.mark.parametrize("name,kw", corpus())
@pytest.mark.parametrize("technique", ["a", "b"])
@pytest.mark.parametrize("post", [False, True])
def test_factors_bit_exact(name, kw, technique, post):
    o, p = _pair(name, kw)
    fo = o.sparsify(technique, post).factors()
    fp = p.sparsify(technique, post)
    assert fp.technique == technique and fp.postprocessed == post
    assert factors_equal(fo, fp.factors())


def test_generic_postprocess_matches_closed_form():
    """Factors.postprocess() on techniqueB == the closed-form B-post builder."""
    for name, kw in corpus()[:10]:
        p = H.builtin(name, **kw)
        assert factors_equal(p.sparsify("b", False).postprocess().factors(), p.sparsify("b", True).factors())
        assert factors_equal(p.sparsify("a", False).postprocess().factors(), p.sparsify("a", True).factors())


# SURVEY.md §8(a) sizing table: (ahat, u, m, v) after postprocessing, dense nnz
SIZES = {("Kc9d7c4d2c", 26, "b"): ((229320, 11970, 12179, 301071), 2045246),
         ("Kc9d7c4d2c", 26, "a"): ((470455, 157057, 29028, 159957), 2045246),
         ("Ks7d4c2h9s", 52, "b"): ((2754388, 61617, 62697, 3390846), 60755142),
         ("AhKhQh7c7d", 52, "b"): ((2754388, 61617, 62697, 2049828), 53173092),
         ("Ks7d4c2h9s", 52, "a"): ((9666364, 795578, 29028, 795578), 60755142)}  # rank 1000 (peel cap)


@pytest.mark.parametrize("board,deck,tech", list(SIZES))
def test_synthetic_configs_bit_exact(board, deck, tech):
    """Configs 2 (dry and wet board) and 4: structure bit-exact against the
    oracle, and the sizes of SURVEY.md §8(a)."""
    o = po.Instance.builtin("river_full", seed=1, board=board, deck=deck, tree=3)
    p = H.builtin("river_full", seed=1, board=board, deck=deck, tree=3)
    assert o.hands(0) == p.hands(0)
    f = p.sparsify(tech, True).factors()
    assert factors_equal(o.sparsify(tech, True).factors(), f)
    nnz, dense = SIZES[(board, deck, tech)]
    assert tuple(int(f[k][0][-1]) for k in ("ahat", "u", "m", "v")) == nnz
    assert p.dense_nnz() == dense


def test_json_loader_matches_constructors(instance_fixtures, tmp_path):
    for name, obj in instance_fixtures.items():
        path = tmp_path / f"{name}.json"
        path.write_text(json.dumps(obj, indent=2))
        loaded, built = H.read_instance(str(path)), H.builtin(name)
        assert loaded.hands(0) == built.hands(0) and loaded.hands(1) == built.hands(1)
        assert bits_equal(loaded.beta, built.beta)
        assert factors_equal(loaded.sparsify("b").factors(), built.sparsify("b").factors())
        # the oracle's JSON path agrees too
        o = po.Instance.from_json(obj)
        assert o.hands(0) == loaded.hands(0)


def test_json_loader_errors(instance_fixtures, tmp_path):
    base = instance_fixtures["golden"]

    def load(obj):
        p = tmp_path / "bad.json"
        p.write_text(obj if isinstance(obj, str) else json.dumps(obj))
        return H.read_instance(str(p))

    with pytest.raises(ParseError):
        load("{not json")
    with pytest.raises(ParseError):
        load(dict(base, schema_version=2))
    with pytest.raises(ParseError):
        load({k: v for k, v in base.items() if k != "board"})
    bad = json.loads(json.dumps(base))
    bad["beliefs"][0]["AdAc"] = "x"
    with pytest.raises(ParseError):
        load(bad)
    bad = json.loads(json.dumps(base))
    bad["beliefs"][0]["AcAd"] = 0.1  # same hand as AdAc
    with pytest.raises(ParseError):
        load(bad)
    bad = json.loads(json.dumps(base))
    bad["betting"]["menus"][0]["bogus"] = [1.0]
    with pytest.raises(ParseError):
        load(bad)
    bad = json.loads(json.dumps(base))
    bad["beliefs"] = [{"AsAh": 1.0}, {"AsKd": 1.0}]  # only pair blocks
    with pytest.raises(ParseError):
        load(bad)
    with pytest.raises(KrError) as e:
        H.read_instance(str(tmp_path / "missing.json"))
    assert e.value.code == "IO"


def test_degenerate_and_invalid_inputs():
    with pytest.raises(InvalidInputError):
        H.builtin("river_full", board="KsKs4c2h9s", tree=3)
    with pytest.raises(InvalidInputError):
        H.builtin("nonexistent")


def test_bundle_round_trip_is_exact(tmp_path):
    p = H.builtin("twenty_card")
    for tech in ("a", "b"):
        f = p.sparsify(tech, True)
        d = tmp_path / tech
        f.write_bundle(str(d))
        g = H.Factors.read_bundle(str(d))
        assert g.technique == tech and g.postprocessed
        assert factors_equal(f.factors(), g.factors())
        hdr = json.loads((d / "header.json").read_text())
        assert hdr["k"] == f.k and hdr["nonzeros"]["v"] == f.nnz["v"]
    # writing twice is byte-identical (cli_pipeline.sh:12-14)
    f = p.sparsify("b", True)
    f.write_bundle(str(tmp_path / "x1"))
    f.write_bundle(str(tmp_path / "x2"))
    for n in ("header.json", "ahat.mtx", "u.mtx", "m.mtx", "v.mtx"):
        assert (tmp_path / "x1" / n).read_bytes() == (tmp_path / "x2" / n).read_bytes()


def test_bundle_rejects_corruption(tmp_path):
    f = H.builtin("golden").sparsify("b", True)
    d = tmp_path / "b"
    f.write_bundle(str(d))
    m = (d / "m.mtx").read_text().splitlines()
    # tamper the first diagonal entry of M (bundle_io.hpp:88-92 -> ParseError)
    for q, line in enumerate(m):
        if line.startswith("1 1 "):
            m[q] = "1 1 2"
    (d / "m.mtx").write_text("\n".join(m) + "\n")
    with pytest.raises(ParseError):
        H.Factors.read_bundle(str(d))
    f.write_bundle(str(d))
    lines = (d / "v.mtx").read_text().splitlines()
    (d / "v.mtx").write_text("\n".join(lines[:-3]) + "\n")  # truncated
    with pytest.raises(ParseError):
        H.Factors.read_bundle(str(d))


def test_from_arrays_validation():
    f = H.builtin("golden").sparsify("b", True)
    arr = f.factors()
    g = H.Factors.from_arrays(f.rows, f.cols, f.k, arr)
    g.validate()
    o, i, v = arr["m"]
    v2 = v.copy()
    v2[0] = 2.0
    bad = H.Factors.from_arrays(f.rows, f.cols, f.k, dict(arr, m=(o, i, v2)))
    with pytest.raises(ContractError):
        bad.validate()


def test_turn_instances_build():
    boards = H.turn_instances(nboards=3)
    assert len(boards) == 3
    for inst, f in boards:
        assert inst.m1 == 1081 and inst.n1 == 43 and f.postprocessed
