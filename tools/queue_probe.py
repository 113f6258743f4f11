"""kr_engine_pair_queue at config 3 on the K7 and Kronecker-factored engines:
pairs/s against the queue length and the number of distinct pinned buffer
sets the inputs cycle through.  One JSON line per point."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import _native as N  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402

insts = [i for i, _ in H.turn_instances("Ks7d4c2h", 48, factors=False)]
L = N.cuda()
for kind in ("implicit", "kfactored"):
    eng = CudaEngine.kron(insts) if kind == "implicit" else CudaEngine.kfactored(insts)
    nx, ny = eng.cols, eng.rows
    sets = [[L.kr_host_alloc(8 * n) for n in (nx, ny, ny, nx)] for _ in range(4)]
    rng = np.random.default_rng(3)
    for b in sets:
        np.ctypeslib.as_array((ctypes.c_double * nx).from_address(b[0]))[:] = rng.standard_normal(nx)
        np.ctypeslib.as_array((ctypes.c_double * ny).from_address(b[1]))[:] = rng.standard_normal(ny)
    for ring in (1, 2, 4):
        for q in (8, 50):
            order = [i % ring for i in range(q)]
            P = ctypes.c_void_p * q
            col = [P(*[sets[o][j] for o in order]) for j in range(4)]
            fn = lambda: N.check(L.kr_engine_pair_queue(eng.handle, q, col[0], nx, col[2], ny, col[1], ny,  # noqa
                                                        col[3], nx))
            fn()
            t = time.perf_counter()
            for _ in range(3):
                fn()
            dt = (time.perf_counter() - t) / 3
            print(json.dumps({"engine": kind, "ring": ring, "queue": q, "pairs_per_s": q / dt}), flush=True)
    for b in sets:
        for p in b:
            L.kr_host_free(p)
    del eng
