import sys, json
sys.path.insert(0, ".")
import torch
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
boards = H.turn_instances("Ks7d4c2h", 48, 3)
eng = CudaEngine([f for _, f in boards])
s = torch.cuda.ExternalStream(eng.stream)
x = torch.randn(eng.cols, dtype=torch.float64, device="cuda"); y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda"); atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
def run(n, timing):
    eng.set_timing(timing)
    for _ in range(5):
        eng.ax_device(x.data_ptr(), ax.data_ptr()); eng.atx_device(y.data_ptr(), atx.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        eng.ax_device(x.data_ptr(), ax.data_ptr()); eng.atx_device(y.data_ptr(), atx.data_ptr())
    e1.record(s); e1.synchronize()
    eng.set_timing(False); eng.kernel_times()
    return e0.elapsed_time(e1) / n * 1e3
out = {}
for rep in range(3):
    for t in (False, True):
        out[f"{'timed' if t else 'plain'}_{rep}"] = round(run(800, t), 1)
print(json.dumps(out))
