import sys, json
sys.path.insert(0, ".")
import torch
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
boards = H.turn_instances("Ks7d4c2h", 48, 3)
for name, eng in (("device", CudaEngine.device_built([i for i, _ in boards])), ("host", CudaEngine([f for _, f in boards]))):
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda"); y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda"); atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    for _ in range(3): eng.ax_device(x.data_ptr(), ax.data_ptr()); eng.atx_device(y.data_ptr(), atx.data_ptr())
    torch.cuda.synchronize(); eng.kernel_times(); eng.set_timing(True)
    for _ in range(10): eng.ax_device(x.data_ptr(), ax.data_ptr()); eng.atx_device(y.data_ptr(), atx.data_ptr())
    torch.cuda.synchronize()
    kt = eng.kernel_times()
    print(name, {k: round(1e3 * v["ms"] / max(v["launches"], 1), 1) for k, v in kt.items()})
    eng.close(); torch.cuda.empty_cache()
