"""CUPTI trace (torch.profiler) of host-buffer products at config 3: copy /
kernel timeline of one kr_engine_ax and one kr_engine_atx call, for the
factored (--factored) or implicit engine."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2112_03804_b200 import CudaEngine, _native as N  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402

fact = "--factored" in sys.argv
boards = H.turn_instances("Ks7d4c2h", 48, 3, factors=fact)
eng = CudaEngine([f for _, f in boards]) if fact else CudaEngine.kron([i for i, _ in boards])
L = N.cuda()
nx, ny = eng.cols, eng.rows
px, py, pax, patx = (L.kr_host_alloc(8 * n) for n in (nx, ny, ny, nx))
np.ctypeslib.as_array((C.c_double * nx).from_address(px))[:] = 1.0
np.ctypeslib.as_array((C.c_double * ny).from_address(py))[:] = 1.0
for _ in range(3):
    N.check(L.kr_engine_ax(eng.handle, px, nx, pax, ny))
    N.check(L.kr_engine_atx(eng.handle, py, ny, patx, nx))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    N.check(L.kr_engine_ax(eng.handle, px, nx, pax, ny))
    N.check(L.kr_engine_atx(eng.handle, py, ny, patx, nx))
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0):9.1f} {(e.time_range.end - t0):9.1f}  {e.name[:60]}")
cpu = [e for e in prof.events() if e.device_type.name == "CPU"]
print("cpu span us", max(e.time_range.end for e in cpu) - min(e.time_range.start for e in cpu))
if "--api" in sys.argv:  # runtime API calls on the host timeline (same origin)
    for e in sorted((e for e in cpu if e.name.startswith("cuda")), key=lambda e: e.time_range.start):
        print(f"API {(e.time_range.start - t0):9.1f} {(e.time_range.end - t0):9.1f}  {e.name[:40]}")
