import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2112_03804_b200 import CudaEngine, host as H
def tp(eng, reps=200):
    s = torch.cuda.ExternalStream(eng.stream)
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda"); y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda"); atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(5):
        eng.ax_device(x.data_ptr(), ax.data_ptr()); eng.atx_device(y.data_ptr(), atx.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(reps):
        eng.ax_device(x.data_ptr(), ax.data_ptr()); eng.atx_device(y.data_ptr(), atx.data_ptr())
    e1.record(s); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for name, mk in [("config2", lambda: [H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)]),
                 ("config3", lambda: [i for i, _ in H.turn_instances("Ks7d4c2h", 48, 3)]),
                 ("turn91", lambda: [i for i, _ in H.turn_instances("Ks7d4c2h", 48, 91)])]:
    insts = mk()
    eng = CudaEngine.kron(insts)
    print(json.dumps({"point": name, "us_per_pair_implicit": tp(eng)}), flush=True)
