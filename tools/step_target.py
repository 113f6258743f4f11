"""ncu target: a few DCFR iterations at config 3 on the implicit engine."""
import sys

sys.path.insert(0, ".")
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

boards = H.turn_instances("Ks7d4c2h", 48, 3, factors=False)
sv = solver_for(boards, implicit=True)
r = sv.run(DcfrParams(max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 6, checkpoint_every=50))
print("iterations", r.iterations)
