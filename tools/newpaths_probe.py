"""Small workloads over the round's newer kernels and paths, checked by
assertions (compute-sanitizer is closed on the GPU pool): compressed slots
(KR_SELL_COMP), the host pipeline
(graph capture on pinned buffers), kr_engine_pair_device, the DCFR solver
(graph replay, PDL, concurrent best responses, fused normalise), K7, and the
turn solver (fused gather / scale, continuations side by side)."""
import ctypes
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("KR_SELL_COMP", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine, _native as N  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402
from paper_2112_03804_b200.solver import DcfrParams, solver_for  # noqa: E402
from paper_2112_03804_b200.turn import TurnGame, TurnSolver  # noqa: E402

boards = [H.builtin("river_full", seed=10 + k, board=b, deck=26, tree=3)
          for k, b in enumerate(["Kc9d7c4d2c", "Ac8d6c3d2d", "QcJd9c5d3c"])]
pairs = [(p, p.sparsify("b", True)) for p in boards]
eng = CudaEngine([f for _, f in pairs])
rng = np.random.default_rng(1)
x, y = rng.standard_normal(eng.cols), rng.standard_normal(eng.rows)
ax, aty = eng.Ax(x), eng.ATx(y)
L = N.cuda()
px, py = L.kr_host_alloc(8 * eng.cols), L.kr_host_alloc(8 * eng.rows)
np.ctypeslib.as_array((ctypes.c_double * eng.cols).from_address(px))[:] = x
for _ in range(3):  # enqueue, capture, replay
    N.check(L.kr_engine_ax(eng.handle, px, eng.cols, py, eng.rows))
assert np.array_equal(np.ctypeslib.as_array((ctypes.c_double * eng.rows).from_address(py)), ax)
L.kr_host_free(px)
L.kr_host_free(py)
dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
o1, o2 = torch.empty(eng.rows, dtype=torch.float64, device="cuda"), torch.empty(eng.cols, dtype=torch.float64,
                                                                                   device="cuda")
torch.cuda.synchronize()
eng.pair_device(dx.data_ptr(), o1.data_ptr(), dy.data_ptr(), o2.data_ptr())
torch.cuda.ExternalStream(eng.stream).synchronize()
assert np.array_equal(o1.cpu().numpy(), ax) and np.array_equal(o2.cpu().numpy(), aty)
sv = solver_for(pairs)
r = sv.run(DcfrParams(max_iters=12, checkpoint_every=4))
sk = solver_for(pairs, implicit=True)
rk = sk.run(DcfrParams.cfr_plus(max_iters=8, checkpoint_every=2))
g = TurnGame(boards=list(range(4)))
t = TurnSolver(g).run(max_iters=4, checkpoint_every=2, rule=2)
print("ok", r.exploitability, rk.exploitability, t["exploitability"])
