"""Host-buffer pair pipeline at config 3: where does kr_engine_pair's time go?

1. Copy-only emulations of the pair's transfer schedule (no kernels; G board
   groups per direction, each output chunk copied back once its input chunk
   has landed), on pinned buffers of the config-3 sizes:
     per_dir  : each direction its own H2D and D2H streams (kr_engine_pair)
     shared_i : one H2D and one D2H stream, directions interleaved per group
     shared_s : one H2D and one D2H stream, direction 1 first, then direction 0
2. kr_engine_pair on the K7 engine for several board-group counts (KR_GROUPS
   is read at engine creation).
Prints one JSON line per measurement."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

N = 2_231_184  # config-3 vector length (48 boards x 43 sequences x 1,081 hands)


def emulate(kind, G, reps=30):
    """The schedule captured into one CUDA graph (no host enqueue cost, like
    the engine's replayed pair graph), timed with events around `reps`
    replays.  kind "duplex": no dependencies at all (all H2D on one stream,
    all D2H on another): the bus floor."""
    h_in = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]
    h_out = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(2)]
    d_in = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(2)]
    d_out = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(2)]
    cut = [N * g // G for g in range(G + 1)]
    side = [torch.cuda.Stream() for _ in range(4)]
    if kind == "per_dir":
        cin, cout = side[0:2], side[2:4]
    else:
        cin, cout = [side[0], side[0]], [side[2], side[2]]
    order = ([(d, g) for g in range(G) for d in (1, 0)] if kind != "shared_s"
             else [(d, g) for d in (1, 0) for g in range(G)])

    def once():
        main = torch.cuda.current_stream()
        for q in side:
            q.wait_stream(main)
        for d, g in order:
            a, b = cut[g], cut[g + 1]
            with torch.cuda.stream(cin[d]):
                d_in[d][a:b].copy_(h_in[d][a:b], non_blocking=True)
            if kind != "duplex":
                cout[d].wait_stream(cin[d])
            with torch.cuda.stream(cout[d]):
                h_out[d][a:b].copy_(d_out[d][a:b], non_blocking=True)
        for q in side:
            main.wait_stream(q)

    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):
        once()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        once()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    e1.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / reps
    return {"emulate": kind, "groups": G, "us_per_pair": dt * 1e6, "pairs_per_s": 1 / dt}


def engine_pairs(groups):
    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import _native as NN
    from paper_2112_03804_b200 import host as H
    import ctypes
    insts = [i for i, _ in H.turn_instances("Ks7d4c2h", 48, factors=False)]
    L = NN.cuda()
    out = []
    for G in groups:
        os.environ["KR_GROUPS"] = str(G)
        eng = CudaEngine.kron(insts)
        nx, ny = eng.cols, eng.rows
        px, py, pax, patx = (L.kr_host_alloc(8 * n) for n in (nx, ny, ny, nx))
        rng = np.random.default_rng(1)
        np.ctypeslib.as_array((ctypes.c_double * nx).from_address(px))[:] = rng.standard_normal(nx)
        np.ctypeslib.as_array((ctypes.c_double * ny).from_address(py))[:] = rng.standard_normal(ny)
        fn = lambda: NN.check(L.kr_engine_pair(eng.handle, px, nx, pax, ny, py, ny, patx, nx))  # noqa: E731
        for _ in range(5):
            fn()
        t = time.perf_counter()
        for _ in range(50):
            fn()
        dt = (time.perf_counter() - t) / 50
        out.append({"engine": "implicit", "groups": G, "us_per_pair": dt * 1e6, "pairs_per_s": 1 / dt})
        for p in (px, py, pax, patx):
            L.kr_host_free(p)
        del eng
    return out


if __name__ == "__main__":
    for kind in ("duplex", "per_dir", "shared_i", "shared_s"):
        for G in (1, 2, 4, 8, 16, 48):
            print(json.dumps(emulate(kind, G)), flush=True)
    for r in engine_pairs([int(g) for g in (sys.argv[1:] or ["4", "8", "16", "24", "48"])]):
        print(json.dumps(r), flush=True)
