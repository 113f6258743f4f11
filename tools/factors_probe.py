"""Technique B post factor construction: host builder (libkrhost, one board
per thread) vs the device builder (kr_factors_build_device, boards one after
another, device seconds incl. download) at config 2 and config 3."""
import json
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
from paper_2112_03804_b200 import host as H  # noqa: E402

insts = [i for i, _ in H.turn_instances("Ks7d4c2h", 48, 3, factors=False)]
one = insts[0]
t0 = time.perf_counter()
one.sparsify("b", True)
host1 = time.perf_counter() - t0
one.sparsify_device()  # warm (context, modules)
t0 = time.perf_counter()
d = one.sparsify_device()
dev1_wall = time.perf_counter() - t0
t0 = time.perf_counter()
with ThreadPoolExecutor(16) as ex:
    list(ex.map(lambda i: i.sparsify("b", True), insts))
host48 = time.perf_counter() - t0
t0 = time.perf_counter()
ds = [i.sparsify_device() for i in insts]
dev48_wall = time.perf_counter() - t0
print(json.dumps({"config2_host_s": host1, "config2_device_s": d.seconds, "config2_device_wall_s": dev1_wall,
                  "config3_host_16threads_s": host48, "config3_device_s": sum(x.seconds for x in ds),
                  "config3_device_wall_s": dev48_wall, "nnz_config3": sum(x.size() for x in ds)}))
