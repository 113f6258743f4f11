"""Profile target (development tool): builds config 2 (or the 48-board
config 3 with --turn) with the CPU oracle's builder and runs a few products
on the device so ncu can capture the engine kernels."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402


def turn_boards(turn="Ks7d4c2h", nboards=48):
    used = {turn[i:i + 2] for i in range(0, 8, 2)}
    ranks, suits = "23456789TJQKA", "cdhs"
    cards = [r + s for r in ranks for s in suits if r + s not in used][:nboards]
    out = []
    for c in cards:
        cid = ranks.index(c[0]) * 4 + suits.index(c[1])
        I = po.Instance.builtin("river_full", seed=1000 + cid, board=turn + c, tree=3)
        out.append(I.sparsify("b", True))
    return out


def main():
    nb = int(sys.argv[sys.argv.index("--turn") + 1]) if "--turn" in sys.argv else 0
    if nb:
        eng = CudaEngine(turn_boards(nboards=nb))
    else:
        I = po.Instance.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
        eng = CudaEngine(I.sparsify("b", True))
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(4):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    torch.cuda.synchronize()
    print("ok", eng.rows, eng.cols, eng.k, float(ax.abs().sum()), float(atx.abs().sum()))


if __name__ == "__main__":
    main()
