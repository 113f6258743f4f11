"""Kronecker-factored engine probe: per-direction and pair times (CUDA events,
device pointers) at config 2 and config 3, bitwise against the device-built
factored engine on the same inputs.  Prints one JSON line per config."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402


def time_it(fn, stream, reps):
    s = torch.cuda.ExternalStream(stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    s.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def run(name, insts, reps):
    t0 = time.time()
    kf = CudaEngine.kfactored(insts)
    tkf = time.time() - t0
    db = CudaEngine.device_built(insts)
    x = torch.randn(kf.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(kf.rows, dtype=torch.float64, device="cuda")
    outs = {k: torch.empty(n, dtype=torch.float64, device="cuda") for k, n in
            (("a1", kf.rows), ("t1", kf.cols), ("a2", kf.rows), ("t2", kf.cols))}
    torch.cuda.synchronize()
    db.ax_device(x.data_ptr(), outs["a1"].data_ptr())
    db.atx_device(y.data_ptr(), outs["t1"].data_ptr())
    kf.ax_device(x.data_ptr(), outs["a2"].data_ptr())
    kf.atx_device(y.data_ptr(), outs["t2"].data_ptr())
    torch.cuda.synchronize()
    torch.cuda.ExternalStream(db.stream).synchronize()
    torch.cuda.ExternalStream(kf.stream).synchronize()
    eq = bool(torch.equal(outs["a1"], outs["a2"]) and torch.equal(outs["t1"], outs["t2"]))
    res = dict(config=name, boards=len(insts), bitwise_vs_device_built=eq, create_s=round(tkf, 3),
               nnz=kf.nnz)
    res["kf_ax_us"] = time_it(lambda: kf.ax_device(x.data_ptr(), outs["a2"].data_ptr()), kf.stream, reps)
    res["kf_atx_us"] = time_it(lambda: kf.atx_device(y.data_ptr(), outs["t2"].data_ptr()), kf.stream, reps)
    res["kf_pair_us"] = time_it(lambda: kf.pair_device(x.data_ptr(), outs["a2"].data_ptr(), y.data_ptr(),
                                                       outs["t2"].data_ptr()), kf.stream, reps)
    res["db_pair_us"] = time_it(lambda: db.pair_device(x.data_ptr(), outs["a1"].data_ptr(), y.data_ptr(),
                                                       outs["t1"].data_ptr()), db.stream, max(3, reps // 4))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["2", "3"]
    if "2" in which:
        run("config2", [H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)], 200)
    if "3" in which:
        run("config3", [i for i, _ in H.turn_instances(nboards=48, factors=False)], 50)
