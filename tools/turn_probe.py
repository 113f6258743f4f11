"""Turn endgame timing: the 52-card turn Ks7d4c2h (1,128 hands per side,
48 river boards), turn menus {0.5} without raises, river menus {0.5, 1.0}
with one raise: build time, DCFR iterations/s on the device."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2112_03804_b200.turn import TurnGame, TurnSolver  # noqa: E402

deck = 26 if "--small" in sys.argv else 52
turn = "Kc9d7c4d" if deck == 26 else "Ks7d4c2h"
t0 = time.time()
g = TurnGame(turn=turn, deck=deck)
build = time.time() - t0
t0 = time.time()
s = TurnSolver(g)
create = time.time() - t0
s.run(max_iters=3, checkpoint_every=3)
r = s.run(max_iters=200, checkpoint_every=50)
print(json.dumps({"deck": deck, "hands": g.m, "boards": len(g.rivers), "continuations": len(g.conts),
                  "n_turn": g.n_turn, "n_river": g.n_river[0], "vector_len": g.size, "build_s": round(build, 2),
                  "create_s": round(create, 2), "iters": r["iterations"], "device_s": r["seconds"],
                  "iters_per_s": r["iterations"] / r["seconds"], "exploitability": r["exploitability"],
                  "trace": [float(v) for v in r["trace_expl"]]}))
