"""Solver timing at config 3: DCFR iterations/s with the factored and the
implicit engine (checkpoint_every = 50), and the player-step kernel time."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

if "--config2" in sys.argv:
    inst = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    boards = [(inst, inst.sparsify("b", True))]
else:
    boards = H.turn_instances("Ks7d4c2h", 48, 3)
for implicit in (True, False):
    sv = solver_for(boards, implicit=implicit)
    sv.run(DcfrParams(max_iters=5, checkpoint_every=5))
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = sv.run(DcfrParams(max_iters=200, checkpoint_every=50), want_avg=False)
    dt = time.perf_counter() - t
    print(json.dumps({"implicit": implicit, "iters_per_s": 200 / dt, "iters_per_s_solver_clock": 200 / r.seconds,
                      "exploitability": r.exploitability}), flush=True)
