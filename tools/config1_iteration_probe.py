"""Config 1 (twenty_card, Technique B post, 1000 CFR+ iterations,
checkpointEvery = 1) DCFR iterations/s through the factored and the implicit
engines, best of three runs, under the caller's environment (step / team /
launch knobs).  Short runs (argv[1] = iterations) serve ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
inst = H.builtin("twenty_card")
f = inst.sparsify("b", True)
out = {}
for label, implicit in (("factored", False), ("implicit", True)):
    sv = solver_for([(inst, f)], implicit=implicit)
    sv.run(DcfrParams.cfr_plus(max_iters=3, checkpoint_every=1))
    best = 0.0
    for _ in range(3 if iters >= 100 else 1):
        r = sv.run(DcfrParams.cfr_plus(max_iters=iters, checkpoint_every=1))
        best = max(best, r.iterations / r.seconds)
    out[label] = round(best, 1)
    out[label + "_step"] = sv.step_kind(0)
print(os.environ.get("PROBE_LABEL", ""), out)
