"""A short run of the small-engine product paths for an ncu capture: config 1
(twenty_card) DCFR iterations (deep-batch SELL kernels, per-matrix long-row
threshold, graph-replayed three-launch products), then stream-launched
products of the golden game (the fused cluster product k_tiny_product)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402

inst = H.builtin("twenty_card")
sv = solver_for([(inst, inst.sparsify("b", True))])
sv.run(DcfrParams.cfr_plus(max_iters=4, checkpoint_every=1))
g = H.builtin("golden")
e = CudaEngine(g.sparsify("b", True))
dev = torch.device("cuda", 0)
x = torch.randn(e.cols, dtype=torch.float64, device=dev)
y = torch.randn(e.rows, dtype=torch.float64, device=dev)
a = torch.empty(e.rows, dtype=torch.float64, device=dev)
b = torch.empty(e.cols, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
for _ in range(3):
    e.ax_device(x.data_ptr(), a.data_ptr())
    e.atx_device(y.data_ptr(), b.data_ptr())
torch.cuda.synchronize()
print("ok")
