"""Host<->device copy bandwidth on the box: H2D alone, D2H alone, both at
once (separate streams), for pinned buffers of the config-3 vector size."""
import json
import sys
import time

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 17_849_472 // 8 * 8
h_in = torch.empty(n // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(n // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(n // 8, dtype=torch.float64, device="cuda")
d_out = torch.randn(n // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=50):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    return (int(h2d) + int(d2h)) * n / dt / 1e9


print(json.dumps({"bytes": n, "h2d_gbs": run(1, 0), "d2h_gbs": run(0, 1), "both_total_gbs": run(1, 1)}))


def split_h2d(k, reps=50):
    ss = [torch.cuda.Stream() for _ in range(k)]
    m = (n // 8) // k
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for i, st in enumerate(ss):
            with torch.cuda.stream(st):
                d_in[i * m:(i + 1) * m].copy_(h_in[i * m:(i + 1) * m], non_blocking=True)
    torch.cuda.synchronize()
    return k * m * 8 / ((time.perf_counter() - t) / reps) / 1e9


print(json.dumps({f"h2d_{k}_streams_gbs": split_h2d(k) for k in (1, 2, 4, 8)}))
