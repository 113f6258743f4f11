"""Profile target (development tool): builds config 2 (or the first N boards
of the config-3 turn with --turn N) with the product's host builder and runs
a few matvec pairs on the device so ncu can capture the engine kernels.
Per pair the launch order is: k_seq_major, k_spmv[VT], k_chain_forward,
k_spmv[UA], k_spmv[UT], k_chain_backward, k_spmv[AV]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402


def main():
    nb = int(sys.argv[sys.argv.index("--turn") + 1]) if "--turn" in sys.argv else 0
    pairs = int(sys.argv[sys.argv.index("--pairs") + 1]) if "--pairs" in sys.argv else 4
    if nb:
        eng = CudaEngine([f for _, f in H.turn_instances(nboards=nb)])
    else:
        eng = CudaEngine(H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3).sparsify("b", True))
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(pairs):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    torch.cuda.synchronize()
    print("ok", eng.rows, eng.cols, eng.k, eng.bytes_per_product(), float(ax.abs().sum()), float(atx.abs().sum()))


if __name__ == "__main__":
    main()
