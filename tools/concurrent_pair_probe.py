"""Whole-pair time at config 3 (and config 2 with --config2): Ax then ATy on
one stream against kr_engine_pair_device (ATy forked onto a side stream),
checked bitwise; per-kernel timing off in both."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402

if "--config2" in sys.argv:
    inst = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    boards = [(inst, inst.sparsify("b", True))]
else:
    boards = H.turn_instances("Ks7d4c2h", 48, 3)
eng = CudaEngine([f for _, f in boards])
s = torch.cuda.ExternalStream(eng.stream)
x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
ax, atx = torch.empty(eng.rows, dtype=torch.float64, device="cuda"), torch.empty(eng.cols, dtype=torch.float64, device="cuda")
ax2, atx2 = torch.empty_like(ax), torch.empty_like(atx)


def serial():
    eng.ax_device(x.data_ptr(), ax.data_ptr())
    eng.atx_device(y.data_ptr(), atx.data_ptr())


def pair():
    eng.pair_device(x.data_ptr(), ax2.data_ptr(), y.data_ptr(), atx2.data_ptr())


def timeit(fn, n=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


out = {"prio": os.environ.get("KR_PAIR_PRIORITY", "0")}
for rep in range(3):
    out[f"serial_us_{rep}"] = timeit(serial)
    out[f"pair_us_{rep}"] = timeit(pair)
torch.cuda.synchronize()
out["bitwise"] = bool(torch.equal(ax, ax2) and torch.equal(atx, atx2))
print(json.dumps(out))
