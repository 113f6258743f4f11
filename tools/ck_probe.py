"""Solver iterations/s where checkpoints weigh: config 1 (twenty_card, 1000
CFR+ iterations, a best response every iteration) and config 2 (one river
board) at checkpoint_every 1 and 10, factored and implicit engines.  Run with
and without KR_BR_SERIAL=1 to compare concurrent / serial best responses."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

out = {"serial": bool(os.environ.get("KR_BR_SERIAL"))}
p = H.builtin("twenty_card")
sv = solver_for([(p, p.sparsify("b", True))])
sv.run(DcfrParams.cfr_plus(max_iters=50, checkpoint_every=1))
r = sv.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1), want_avg=False)
out["config1_ck1"] = {"iters_per_s": 1000 / r.seconds, "expl": r.exploitability}
inst = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
boards = [(inst, inst.sparsify("b", True))]
for implicit in (False, True):
    sv = solver_for(boards, implicit=implicit)
    for ck in (1, 10):
        sv.run(DcfrParams(max_iters=20, checkpoint_every=ck))
        torch.cuda.synchronize()
        r = sv.run(DcfrParams(max_iters=400, checkpoint_every=ck), want_avg=False)
        out[f"config2_{'implicit' if implicit else 'factored'}_ck{ck}"] = {"iters_per_s": 400 / r.seconds,
                                                                          "expl": r.exploitability}
print(json.dumps(out))
