"""Real-run kernel time breakdown of DCFR iterations (torch.profiler / CUPTI,
no replay): config 3, implicit or factored engine."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

implicit = "--factored" not in sys.argv
boards = H.turn_instances("Ks7d4c2h", 48, 3, factors=not implicit)
sv = solver_for(boards if not implicit else [b[0] for b in boards], implicit=implicit)
sv.run(DcfrParams(max_iters=5, checkpoint_every=5))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    r = sv.run(DcfrParams(max_iters=100, checkpoint_every=50))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
print("seconds", r.seconds)
