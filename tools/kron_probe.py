"""Implicit Kronecker engine timing: us per matvec pair (Ax + ATx) with CUDA
events on the engine stream, after warm-up.  --only NAME selects a point,
--reps N the number of timed pairs (use a small N under ncu)."""
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402


def tp(eng, reps=200):
    s = torch.cuda.ExternalStream(eng.stream)
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(min(reps, 5)):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


POINTS = {
    "config2": lambda: [H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)],
    "config3": lambda: [i for i, _ in H.turn_instances("Ks7d4c2h", 48, 3, factors=False)],
    "turn91": lambda: [i for i, _ in H.turn_instances("Ks7d4c2h", 48, 91, factors=False)],
}

if __name__ == "__main__":
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 200
    for name, mk in POINTS.items():
        if only and name != only:
            continue
        eng = CudaEngine.kron(mk())
        print(json.dumps({"point": name, "us_per_pair_implicit": tp(eng, reps)}), flush=True)
