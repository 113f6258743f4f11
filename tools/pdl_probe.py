"""Config 2 DCFR (factored and K7, checkpoint every 50), config 2 serial
pair and config 1 (factored): the programmatic-dependent-launch settings
(KR_PDL / KR_PDL_MAXGRID) are read per launch, so one process sweeps them."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

inst = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
f = inst.sparsify("b", True)
tw = H.builtin("twenty_card")
twf = tw.sparsify("b", True)
settings = sys.argv[1:] or ["off", "64", "512", "2000"]
out = {}
for st in settings:
    os.environ.pop("KR_PDL", None)
    os.environ.pop("KR_PDL_MAXGRID", None)
    if st == "off":
        os.environ["KR_PDL"] = "0"
    else:
        os.environ["KR_PDL_MAXGRID"] = st
    row = {}
    for name, implicit in (("c2_factored", False), ("c2_implicit", True)):
        sv = solver_for([(inst, f)], implicit=implicit)
        sv.run(DcfrParams(max_iters=10, checkpoint_every=10))
        r = sv.run(DcfrParams(max_iters=400, checkpoint_every=50), want_avg=False)
        row[name] = round(400 / r.seconds)
    sv = solver_for([(tw, twf)])
    sv.run(DcfrParams.cfr_plus(max_iters=20, checkpoint_every=1))
    r = sv.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1), want_avg=False)
    row["c1_factored"] = round(1000 / r.seconds)
    eng = CudaEngine(f)
    s = torch.cuda.ExternalStream(eng.stream)
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    for _ in range(5):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(300):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    e1.record(s)
    e1.synchronize()
    row["c2_pair_us"] = round(e0.elapsed_time(e1) / 300 * 1e3, 1)
    out[st] = row
print(json.dumps(out))
