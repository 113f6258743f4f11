import re, sys
sys.path.insert(0, ".")
from collections import defaultdict
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for
p = H.builtin("twenty_card")
sv = solver_for([(p, p.sparsify("b", True))])
sv.run(DcfrParams.cfr_plus(max_iters=20, checkpoint_every=1))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sv.run(DcfrParams.cfr_plus(max_iters=100, checkpoint_every=1))
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev); t1 = max(e.time_range.end for e in ev)
tot = defaultdict(float); cnt = defaultdict(int)
for e in ev:
    m = re.search(r"(k_\w+(<[^>]*>)?)", e.name); k = m.group(1) if m else e.name[:30]
    tot[k] += e.time_range.end - e.time_range.start; cnt[k] += 1
print(f"span {t1-t0:.0f} us / 100 it; kernels {sum(cnt.values())}; busy sum {sum(tot.values()):.0f}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]): print(f"{k:40s} n={cnt[k]:5d} avg={v/cnt[k]:6.2f} total={v:8.1f}")
