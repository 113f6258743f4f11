"""Config 1 (twenty_card, 1000 CFR+ iterations, a checkpoint every
iteration) through the factored engine (bitwise path) and through K7."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

p = H.builtin("twenty_card")
out = {}
for implicit in (False, True):
    sv = solver_for([(p, p.sparsify("b", True))], implicit=implicit)
    sv.run(DcfrParams.cfr_plus(max_iters=20, checkpoint_every=1))
    torch.cuda.synchronize()
    r = sv.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1), want_avg=False)
    out["implicit" if implicit else "factored"] = {"iters_per_s": 1000 / r.seconds, "expl": r.exploitability}
print(json.dumps(out))
