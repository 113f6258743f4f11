"""Small-engine product settings (the fused product k_tiny_product, the
deep-batch SELL kernels): config-1 CFR+ iterations/s (twenty_card,
checkpointEvery = 1), config-2 / config-4 and a few corpus engines' pair and
product times and DCFR it/s, per environment setting (default: the KR_TINY /
KR_TINY_CLUSTER sweep; argv[1]: a JSON list of [label, env] pairs).
Each setting runs in its own process (the engine reads the knobs per
product, but the solver's captured graph keeps the launches it captured)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, time
sys.path.insert(0, ROOT)
import torch
from paper_2112_03804_b200 import CudaEngine
from paper_2112_03804_b200 import host as H
from paper_2112_03804_b200.solver import DcfrParams, solver_for
dev = torch.device("cuda", 0)
out = {}
inst = H.builtin("twenty_card")
f = inst.sparsify("b", True)
sv = solver_for([(inst, f)])
sv.run(DcfrParams.cfr_plus(max_iters=5, checkpoint_every=1))
best = None
for _ in range(3):
    r = sv.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1))
    its = r.iterations / r.seconds
    best = its if best is None else max(best, its)
out["config1_its"] = best
r = sv.run(DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=50))
out["config1_its_ck50"] = r.iterations / r.seconds

def dir_us(e, reps=2000):
    st = torch.cuda.ExternalStream(e.stream)
    x = torch.randn(e.cols, dtype=torch.float64, device=dev)
    y = torch.randn(e.rows, dtype=torch.float64, device=dev)
    a = torch.empty(e.rows, dtype=torch.float64, device=dev)
    b = torch.empty(e.cols, dtype=torch.float64, device=dev)
    res = []
    for f, i, o in ((e.ax_device, x, a), (e.atx_device, y, b)):
        for _ in range(20):
            f(i.data_ptr(), o.data_ptr())
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            f(i.data_ptr(), o.data_ptr())
        e1.record(st)
        torch.cuda.synchronize(dev)
        res.append(e0.elapsed_time(e1) * 1e3 / reps)
    return res

def pair_us(e, reps=2000):
    st = torch.cuda.ExternalStream(e.stream)
    g = torch.Generator(device="cpu").manual_seed(4)
    x = torch.randn(e.cols, dtype=torch.float64, generator=g).to(dev)
    y = torch.randn(e.rows, dtype=torch.float64, generator=g).to(dev)
    a = torch.empty(e.rows, dtype=torch.float64, device=dev)
    b = torch.empty(e.cols, dtype=torch.float64, device=dev)
    for _ in range(20):
        e.pair_device(x.data_ptr(), a.data_ptr(), y.data_ptr(), b.data_ptr())
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        e.pair_device(x.data_ptr(), a.data_ptr(), y.data_ptr(), b.data_ptr())
    e1.record(st)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) * 1e3 / reps

for name, kw in [("twenty_card", {}), ("bench", dict(seed=2, hands=100)), ("golden", {}),
                 ("random_small", dict(seed=3)),
                 ("river_full", dict(seed=1, board="Kc9d7c4d2c", deck=26, tree=3))]:
    p = H.builtin(name, **kw)
    e = CudaEngine(p.sparsify("b", True))
    out[name + "_pair_us"] = pair_us(e)
    out[name + "_ax_atx_us"] = dir_us(e)
    if name != "river_full":
        sv = solver_for([(p, p.sparsify("b", True))])
        sv.run(DcfrParams(max_iters=5, checkpoint_every=1))
        r = sv.run(DcfrParams(max_iters=1000, checkpoint_every=1))
        out[name + "_dcfr_its_ck1"] = r.iterations / r.seconds
inst2 = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
e2 = CudaEngine(inst2.sparsify("b", True))
out["config2_factored_pair_us"] = pair_us(e2, reps=500)
out["config2_factored_ax_atx_us"] = dir_us(e2, reps=500)
s2 = solver_for([(inst2, inst2.sparsify("b", True))])
s2.run(DcfrParams(max_iters=5, checkpoint_every=50))
r = s2.run(DcfrParams(max_iters=400, checkpoint_every=50))
out["config2_factored_dcfr_its"] = r.iterations / r.seconds
inst4 = H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
s4 = solver_for([(inst4, inst4.sparsify("b", True))])
s4.run(DcfrParams(max_iters=5, checkpoint_every=50))
r = s4.run(DcfrParams(max_iters=400, checkpoint_every=50))
out["config4_dcfr_its"] = r.iterations / r.seconds
print("RESULT " + json.dumps(out))
'''


def run(env):
    e = dict(os.environ, **env)
    code = CHILD.replace("ROOT", repr(ROOT), 1)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
    for ln in r.stdout.splitlines():
        if ln.startswith("RESULT "):
            return json.loads(ln[7:])
    return {"error": (r.stderr or r.stdout)[-800:]}


def main():
    if len(sys.argv) > 1:   # JSON list of [label, env] pairs
        for label, env in json.loads(sys.argv[1]):
            print(json.dumps({"setting": label, "env": env, **run(env)}), flush=True)
        return
    settings = [("three launches", {"KR_TINY": "0"}),
                ("fused, default size", {}),
                ("fused, all engines, default size", {"KR_TINY": "1000000000"})]
    settings += [(f"fused, all engines, cluster {c}", {"KR_TINY": "1000000000", "KR_TINY_CLUSTER": str(c)})
                 for c in (4, 8, 16)]
    for label, env in settings:
        print(json.dumps({"setting": label, "env": env, **run(env)}), flush=True)


if __name__ == "__main__":
    main()
