import sys, os
sys.path.insert(0, os.getcwd())
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for
inst = H.builtin("twenty_card")
sv = solver_for([(inst, inst.sparsify("b", True))])
sv.run(DcfrParams.cfr_plus(max_iters=3, checkpoint_every=1))
r = sv.run(DcfrParams.cfr_plus(max_iters=10, checkpoint_every=1))
print("its", r.iterations / r.seconds)
