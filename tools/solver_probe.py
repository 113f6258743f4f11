"""DCFR iterations/s at config 3 (48 boards) through a chosen engine, and a
short run for ncu captures: python tools/solver_probe.py [kron|kfactored|factored] [iters]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import CudaSolver, DcfrParams  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "kron"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
nb = int(os.environ.get("BOARDS", "48"))
boards = H.turn_instances(nboards=nb, factors=kind == "factored")
insts = [i for i, _ in boards]
eng = {"kron": lambda: CudaEngine.kron(insts), "kfactored": lambda: CudaEngine.kfactored(insts),
       "factored": lambda: CudaEngine([f for _, f in boards])}[kind]()
i0 = insts[0]
s = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [i.m1 for i in insts], [i.m2 for i in insts], i0.pot)
s.run(DcfrParams(max_iters=5, checkpoint_every=5))
t = time.perf_counter()
r = s.run(DcfrParams(max_iters=iters, checkpoint_every=50), want_avg=False)
print(f"{kind} boards={nb} iters={iters} device {iters / r.seconds:.1f} it/s (wall {iters / (time.perf_counter() - t):.1f}) "
      f"expl={r.exploitability!r}")
