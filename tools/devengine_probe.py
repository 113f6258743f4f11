"""Factored engine creation: host path (libkrhost factors, 16 threads, then
the host-built SELL layout) vs kr_engine_create_device_b (everything on the
device), and matvec pairs through each, at config 3 and at the sweep's top
point (2 turns x 48 rivers, 91-sequence tree, 1.25e9 stored nonzeros)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402


def pair_us(eng, reps=20):
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
    return e0.elapsed_time(e1) / reps * 1e3


# warm the device path (context, module loads, allocator) outside the timings
CudaEngine.device_built(H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)).close()

points = {"config3": (["Ks7d4c2h"], 3), "config5_top": (["Ks7d4c2h", "Ah8c5d3s"], 91)}
only = sys.argv[1] if len(sys.argv) > 1 else None
for name, (turns, tree) in points.items():
    if only and name != only:
        continue
    insts = []
    for t in turns:
        insts += [i for i, _ in H.turn_instances(t, 48, tree, factors=False)]
    t0 = time.perf_counter()
    eng_d = CudaEngine.device_built(insts)
    torch.cuda.synchronize()
    dev_s = time.perf_counter() - t0
    us_d = pair_us(eng_d)
    nnz = sum(eng_d.nnz.values())
    eng_d.close()
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(16) as ex:
        facs = list(ex.map(lambda i: i.sparsify("b", True), insts))
    build_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    eng_h = CudaEngine(facs)
    create_s = time.perf_counter() - t0
    us_h = pair_us(eng_h)
    eng_h.close()
    del facs
    torch.cuda.empty_cache()
    print(json.dumps({"point": name, "nnz": nnz, "device_create_s": round(dev_s, 3),
                      "host_factors_s": round(build_s, 3), "host_engine_create_s": round(create_s, 3),
                      "us_per_pair_device_built": us_d, "us_per_pair_host_built": us_h}), flush=True)
