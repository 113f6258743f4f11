"""CUPTI trace (torch.profiler) of turn-solver iterations at the bench's turn
workload: in-situ kernel times (ncu's serialised cold-cache times overstate
the small latency-bound kernels).  Run with KR_NO_GRAPH=1 for per-launch
host timing as well."""
import re
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2112_03804_b200.turn import TurnGame, TurnSolver  # noqa: E402

g = TurnGame(turn="Ks7d4c2h", deck=52)
s = TurnSolver(g)
s.run(max_iters=3, checkpoint_every=3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    s.run(max_iters=10, checkpoint_every=10)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
t1 = max(e.time_range.end for e in ev)
tot = defaultdict(float)
cnt = defaultdict(int)
for e in ev:
    m = re.search(r"(k_\w+(<[^>]*>)?)", e.name)
    k = m.group(1) if m else e.name[:40]
    tot[k] += e.time_range.end - e.time_range.start
    cnt[k] += 1
print(f"span us {t1 - t0:.0f} for 10 iterations + 1 checkpoint; kernel sum {sum(tot.values()):.0f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:42s} n={cnt[k]:4d} total={v:8.1f} us  avg={v / cnt[k]:7.2f} us")
