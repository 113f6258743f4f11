"""Scratch probe (development tool, not the bench): engine parity vs the CPU
oracle on the small corpus and config 2, plus device timings of the
products at config 2 and the 48-board turn (config 3).  Uses the oracle to
build factors, so it is NOT a product path; bench.py is."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as po  # noqa: E402
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402


def bits_equal(a, b):
    return np.array_equal(np.asarray(a).view(np.int64), np.asarray(b).view(np.int64))


def parity(name, inst, sp, rng):
    eng = CudaEngine(sp)
    ok = True
    for _ in range(3):
        x = rng.standard_normal(inst.cols)
        y = rng.standard_normal(inst.rows)
        a, b = eng.Ax(x), sp.matvec(x)
        c, d = eng.ATx(y), sp.matvec_t(y)
        ok &= bits_equal(a, b) and bits_equal(c, d)
        if not ok:
            print("  MISMATCH", name, np.abs(a - b).max(), np.abs(c - d).max())
            break
    print(f"{name:40s} rows={inst.rows} k={sp.k} bitwise={'yes' if ok else 'NO'} flops={eng.last_flops()}"
          f"/{sp.flops_per_matvec()}")
    return ok


def time_products(eng, reps=20):
    s = torch.cuda.ExternalStream(eng.stream)
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(3):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    out = {}
    for name, fn in (("Ax", lambda: eng.ax_device(x.data_ptr(), ax.data_ptr())),
                     ("ATx", lambda: eng.atx_device(y.data_ptr(), atx.data_ptr()))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        e1.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    B = eng.bytes_per_product()
    print(f"  Ax {out['Ax']*1e3:.1f} us  ATx {out['ATx']*1e3:.1f} us   bytes/product {B/1e6:.1f} MB  "
          f"-> Ax {B/out['Ax']/1e6:.0f} GB/s  ATx {B/out['ATx']/1e6:.0f} GB/s  (peak 6552)")
    return out


def main():
    rng = np.random.default_rng(7)
    ok = True
    for nm in ("twenty_card", "golden", "bluffing", "all_tie"):
        I = po.Instance.builtin(nm)
        for tech in ("a", "b"):
            for post in (False, True):
                ok &= parity(f"{nm} {tech} post={post}", I, I.sparsify(tech, post), rng)
    for seed in range(6):
        I = po.Instance.builtin("random_small", seed=seed)
        for tech in ("a", "b"):
            ok &= parity(f"random_small[{seed}] {tech}", I, I.sparsify(tech, True), rng)
    t = time.time()
    I2 = po.Instance.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    S2 = I2.sparsify("b", True)
    print(f"config2 build {time.time()-t:.1f}s")
    ok &= parity("config2 Ks7d4c2h9s B-post", I2, S2, rng)
    e2 = CudaEngine(S2)
    time_products(e2)
    # config 3: 48 river boards under the turn Ks7d4c2h
    turn = "Ks7d4c2h"
    used = {turn[i:i + 2] for i in range(0, 8, 2)}
    ranks, suits = "23456789TJQKA", "cdhs"
    cards = [r + s for r in ranks for s in suits if r + s not in used]
    t = time.time()
    boards = []
    for cid, c in enumerate(cards):
        card_id = ranks.index(c[0]) * 4 + suits.index(c[1])
        Ib = po.Instance.builtin("river_full", seed=1000 + card_id, board=turn + c, tree=3)
        boards.append((Ib, Ib.sparsify("b", True)))
    print(f"config3 oracle build {time.time()-t:.1f}s, total nnz {sum(s.size_total() for _, s in boards)/1e6:.1f}M")
    t = time.time()
    e3 = CudaEngine([s for _, s in boards])
    print(f"config3 engine create {time.time()-t:.1f}s")
    time_products(e3)
    # spot-check parity on the stacked engine (first and last boards)
    x = rng.standard_normal(e3.cols)
    ax = e3.Ax(x)
    ro = co = 0
    good = True
    for b, (Ib, Sb) in enumerate(boards):
        if b in (0, 17, len(boards) - 1):
            good &= bits_equal(ax[ro:ro + Ib.rows], Sb.matvec(x[co:co + Ib.cols]))
        ro += Ib.rows
        co += Ib.cols
    print("config3 stacked bitwise:", good)
    ok &= good
    ok &= solver_probe()
    print("ALL OK" if ok else "FAILURES")
    return 0 if ok else 1


def solver_probe():
    from paper_2112_03804_b200.solver import CudaSolver, DcfrParams, Treeplex
    ok = True

    def mk(I, sps, hands1, hands2):
        eng = CudaEngine(sps)
        t1 = Treeplex.from_flat(I.n1, I.treeplex(0))
        t2 = Treeplex.from_flat(I.n2, I.treeplex(1))
        return eng, CudaSolver(eng, t1, t2, hands1, hands2, 2 * 1875.0)

    I = po.Instance.builtin("twenty_card")
    S = I.sparsify("b", True)
    eng, sol = mk(I, S, [I.m1], [I.m2])
    r = sol.run(DcfrParams(max_iters=600))
    o = po.dcfr(I, S, max_iters=600)
    good = r.exploitability == o["exploitability"] and r.gradient_flops == o["gradient_flops"] == 67228200
    good &= bits_equal(r.avg1, o["avg1"]) and bits_equal(r.avg2, o["avg2"])
    print(f"twenty_card 600 it: gpu expl {r.exploitability!r} oracle {o['exploitability']!r} flops {r.gradient_flops}"
          f" bitwise={good} ({r.seconds*1e3:.1f} ms, {r.launches} launches)")
    ok &= good
    r = sol.run(DcfrParams(max_iters=300, checkpoint_every=1))
    o = po.dcfr(I, S, max_iters=300, checkpoint_every=1)
    good = bits_equal(r.trace_expl, o["trace_expl"]) and bits_equal(r.trace_br1, o["trace_br1"])
    print(f"twenty_card 300 it every-iteration trace bitwise={good}  ({r.seconds*1e3:.1f} ms)")
    ok &= good
    for nm in ("bluffing", "all_tie", "golden"):
        Ib = po.Instance.builtin(nm)
        Sb = Ib.sparsify("b", True)
        e_b, s_b = mk(Ib, Sb, [Ib.m1], [Ib.m2])
        s_b = CudaSolver(e_b, Treeplex.from_flat(Ib.n1, Ib.treeplex(0)), Treeplex.from_flat(Ib.n2, Ib.treeplex(1)),
                         [Ib.m1], [Ib.m2], 20.0 if nm != "golden" else 3750.0)
        r = s_b.run(DcfrParams(max_iters=400, checkpoint_every=1))
        o = po.dcfr(Ib, Sb, max_iters=400, checkpoint_every=1)
        good = bits_equal(r.trace_br1, o["trace_br1"]) and bits_equal(r.trace_br2, o["trace_br2"])
        print(f"{nm} 400 it trace bitwise={good} final expl {r.exploitability!r} vs {o['exploitability']!r}")
        ok &= good
    I2 = po.Instance.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    S2 = I2.sparsify("b", True)
    e2, s2 = mk(I2, S2, [I2.m1], [I2.m2])
    r = s2.run(DcfrParams(max_iters=60, checkpoint_every=10))
    t = time.time()
    o = po.dcfr(I2, S2, max_iters=60, checkpoint_every=10)
    tcpu = time.time() - t
    good = bits_equal(r.trace_br1, o["trace_br1"]) and bits_equal(r.trace_br2, o["trace_br2"])
    print(f"config2 60 it (ckpt 10) trace bitwise={good} gpu {r.seconds*1e3:.1f} ms cpu {tcpu*1e3:.0f} ms")
    ok &= good
    r = s2.run(DcfrParams(max_iters=500, checkpoint_every=50))
    print(f"config2 500 it: {500/r.seconds:.0f} it/s  expl {r.exploitability:.6g}")
    return ok


if __name__ == "__main__":
    sys.exit(main())
