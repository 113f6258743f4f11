"""Device vs end-to-end (host pinned buffers through kr_engine_ax/atx) matvec
pairs/s at config 3 for several board-group counts (KR_GROUPS), for the
factored and the implicit engine.  python tools/e2e_probe.py [G ...]"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine, _native as N  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402


def device_pairs(eng, reps):
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
    for _ in range(reps):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    e1.record(s)
    e1.synchronize()
    return reps / (e0.elapsed_time(e1) / 1e3)


def e2e_pairs(eng, reps):
    L = N.cuda()
    nx, ny = eng.cols, eng.rows
    px, py, pax, patx = (L.kr_host_alloc(8 * n) for n in (nx, ny, ny, nx))
    arr = lambda p, n: np.ctypeslib.as_array((C.c_double * n).from_address(p))  # noqa: E731
    arr(px, nx)[:] = np.random.default_rng(1).standard_normal(nx)
    arr(py, ny)[:] = np.random.default_rng(2).standard_normal(ny)
    for _ in range(2):
        N.check(L.kr_engine_ax(eng.handle, px, nx, pax, ny))
        N.check(L.kr_engine_atx(eng.handle, py, ny, patx, nx))
    t = time.perf_counter()
    for _ in range(reps):
        N.check(L.kr_engine_ax(eng.handle, px, nx, pax, ny))
        N.check(L.kr_engine_atx(eng.handle, py, ny, patx, nx))
    t = time.perf_counter() - t
    out = arr(pax, ny).copy()
    for p in (px, py, pax, patx):
        L.kr_host_free(p)
    return reps / t, out


if __name__ == "__main__":
    groups = [int(g) for g in sys.argv[1:] if g.isdigit()] or [1, 2, 4, 8]
    boards = H.turn_instances("Ks7d4c2h", 48, 3)
    ref = None
    for G in groups:
        os.environ["KR_GROUPS"] = str(G)
        eng = CudaEngine([f for _, f in boards])
        d = device_pairs(eng, 100)
        e, out = e2e_pairs(eng, 30)
        ref = out if ref is None else ref
        print(json.dumps({"engine": "factored", "groups": G, "device_pairs_s": d, "e2e_pairs_s": e,
                          "same_as_first": bool(np.array_equal(out, ref))}), flush=True)
        eng.close()
    for G in groups if "--factored" not in sys.argv else []:
        os.environ["KR_GROUPS"] = str(G)
        eng = CudaEngine.kron([i for i, _ in boards])
        d = device_pairs(eng, 300)
        e, _ = e2e_pairs(eng, 50)
        print(json.dumps({"engine": "implicit", "groups": G, "device_pairs_s": d, "e2e_pairs_s": e}), flush=True)
