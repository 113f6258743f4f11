"""Write tests/golden/instances_v1.json: the reference's four bundled games
(golden, twenty_card, bluffing, all_tie) in instance schema v1, generated from
the constructor definitions of instances.hpp:33-101 (restated below), which
the reference locks its instance files to (test_instance_io.cpp:149-154).
tests/test_host_builder.py checks, when /root/reference is mounted, that the
reference's own instances/*.json parse to the same games."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CTX = ["first_action", "facing_check", "facing_bet", "after_one_raise", "after_multiple_raises"]


def menus(m1, m2):
    return [{c: list(m1.get(c, [])) for c in CTX}, {c: list(m2.get(c, [])) for c in CTX}]


def game(board, beliefs, stacks, pot, menu1, menu2, all_in, deck="standard52", raise_cap=None):
    return {"schema_version": 1, "deck": deck, "board": board, "stacks": stacks, "pot_contribution": pot,
            "beliefs": beliefs,
            "betting": {"all_in": all_in, "raise_cap": raise_cap, "menus": menus(menu1, menu2)}}


def canon(a, b):
    order = lambda c: ("23456789TJQKA".index(c[0]), "cdhs".index(c[1]))  # noqa: E731
    return a + b if order(a) > order(b) else b + a


def main():
    ref = {c: [0.75] for c in CTX}
    out = {}
    out["golden"] = game(["2c", "7d", "9h", "Jc", "3s"],
                         [{"AdAc": 0.5, "KdKc": 0.3, "5d5c": 0.2}, {"AsAh": 0.4, "QdQc": 0.4, "7h7c": 0.2}],
                         [18125.0, 18125.0], 1875.0, ref, ref, True)
    deck = [r + s for r in "23456" for s in "cdhs"]
    board = ["2c", "2d", "4h", "5s", "6c"]
    rest = [c for c in deck if c not in board]
    hands = {canon(rest[i], rest[j]): 1.0 for i in range(len(rest)) for j in range(i + 1, len(rest))}
    out["twenty_card"] = game(board, [hands, dict(hands)], [18125.0, 18125.0], 1875.0, ref, ref, True, deck=deck)
    out["bluffing"] = game(["2c", "2d", "2h", "3c", "3d"], [{"3s3h": 0.5, "5c4c": 0.5}, {"AdAc": 1.0}],
                           [40.0, 40.0], 10.0, {"first_action": [1.0]}, {}, False)
    out["all_tie"] = game(["As", "Ks", "Qs", "Js", "Ts"], [{"3c2c": 0.5, "5d4d": 0.5}, {"3h2h": 0.5, "5h4h": 0.5}],
                          [40.0, 40.0], 10.0, {"first_action": [1.0]}, {"facing_check": [1.0]}, False)
    path = os.path.join(ROOT, "tests", "golden", "instances_v1.json")
    with open(path, "w") as f:
        json.dump(out, f, sort_keys=True, separators=(",", ":"))
        f.write("\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
