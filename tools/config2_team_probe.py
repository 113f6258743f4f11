"""Config-2 DCFR iterations/s (factored and K7, checkpointEvery=50, 400
iterations after a 10-iteration warm-up), as bench.py's config2 block times
them.  Run under different KR_TEAM / KR_TEAM_THREADS settings to compare
team-step shapes on the single-board engine."""
import json
import os
import sys

sys.path.insert(0, ".")
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

inst = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
f = inst.sparsify("b", True)
out = {"team": os.environ.get("KR_TEAM", "4"), "threads": os.environ.get("KR_TEAM_THREADS", "128")}
for name, implicit in (("factored", False), ("implicit", True)):
    sv = solver_for([(inst, f)], implicit=implicit)
    sv.run(DcfrParams(max_iters=10, checkpoint_every=10))
    r = sv.run(DcfrParams(max_iters=400, checkpoint_every=50), want_avg=False)
    out[name] = round(400 / r.seconds)
    out[name + "_expl"] = r.exploitability
print(json.dumps(out), flush=True)
