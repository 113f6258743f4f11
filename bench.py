#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 gradient oracle.

Metric (BASELINE.json): payoff matvec pairs/s (fp64); solver iters/s is
reported beside it.  A step is one matvec pair (A x and A^T y, engine.hpp:58
and :96) over the whole workload:

  config 3: turn Ks7d4c2h + each of the 48 river cards,
  1,081 hands per side, 3-bet tree (n = 43 sequences), Technique B with
  postprocessing, beliefs from seed 1000 + card id; ~3.0e8 stored nonzeros,
  3.6 GB of factors streamed per product (>> the 126 MB L2, so no flush is
  needed between steps).

It is the largest single-GPU configuration of BASELINE.json and the instance
the north star's roofline target names.  Factors are built by the product's
C++ host side (libkrhost) and applied by the sm_100a kernels (libkrcuda).

  python bench.py [--gpus N --steps K --warmup W]           product arm
  python bench.py --impl reference [...]                    CPU reference arm

Multi-GPU (torchrun, one process per GPU): boards are sharded contiguously
(48/N per GPU), products need no communication, time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "payoff matvec pairs/s and solver iters/s (fp64) at 1/2/4/8 B200 vs CPU"
TURN = "Ks7d4c2h"
NBOARDS = 48


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=800)  # ~1 s timed: several nvidia-smi clock samples
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["product", "reference"], default="product")
    p.add_argument("--boards", type=int, default=NBOARDS)
    p.add_argument("--solver-iters", type=int, default=100)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip the config-5 sweep leg")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the bounded CPU sample")
    return p.parse_args()


def workload_config(nboards, world, extra=None):
    cfg = {"workload": f"config3: turn {TURN} x {nboards} river boards, 1081 hands/side, 3-bet tree (n=43), "
                       "Technique B postprocessed, fp64 factors", "boards": nboards, "hands_per_side": 1081,
           "sequences": 43, "tree": "menus {0.5,1.0} all contexts, all-in, raise cap 3, stacks 18125, pot 1875",
           "l2": "no flush: every product streams 3.6 GB of factors (>> 126 MB L2)",
           "parallelism": f"boards sharded {nboards // world if nboards % world == 0 else 'uneven'} per GPU, "
                          f"{world} GPU(s), no data-path collective"}
    if extra:
        cfg.update(extra)
    return cfg


def _finite(obj):
    """Strict JSON: non-finite floats become strings ("inf", "nan")."""
    if isinstance(obj, float) and not np.isfinite(obj):
        return str(obj)
    if isinstance(obj, dict):
        return {k: _finite(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_finite(v) for v in obj]
    return obj


# --------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_id):
        self.dev = device_id
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", self.dev], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [s.strip() for s in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full
    summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------ CPU side ----
def oracle_boards(indices, threads, with_instances=False):
    """CPU oracle factors (oracle/, test infrastructure) for the given boards."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    from concurrent.futures import ThreadPoolExecutor
    from paper_2112_03804_b200.host import turn_boards
    specs = turn_boards(TURN, NBOARDS)

    def one(b):
        card, seed = specs[b]
        inst = po.Instance.builtin("river_full", seed=seed, board=TURN + card, tree=3)
        return (inst, inst.sparsify("b", True)) if with_instances else inst.sparsify("b", True)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(one, indices))


def run_turn(rank, world, local, max_over_ranks, group, comm=None):
    """Turn endgame: the 52-card turn
    Ks7d4c2h with a betting round (menus {0.5}, no raise) above its 48 river
    boards (menus {0.5, 1.0}, one raise), 1,128 hands per side; boards sharded
    over the ranks, one allreduce of the turn values per half-iteration."""
    from paper_2112_03804_b200.dist import boards_per_rank, shard
    from paper_2112_03804_b200.turn import TurnGame, TurnSolver
    t0 = time.time()
    g = TurnGame(turn=TURN, deck=52, boards=list(shard(NBOARDS, rank, world)))
    if comm is not None:  # NCCL in-stream, graph-captured
        s = TurnSolver(g, device=local, comm=comm, boards_per_rank=boards_per_rank(NBOARDS, world))
    else:
        s = TurnSolver(g, device=local, group=group if world > 1 else None)
    setup = time.time() - t0
    s.run(max_iters=3, checkpoint_every=3)  # warm
    r = s.run(max_iters=200, checkpoint_every=50)
    secs = max_over_ranks(r["seconds"])
    return {"workload": f"turn {TURN}: betting round (menus {{0.5}}, no raise) above 48 river boards "
                        "(menus {0.5, 1.0}, one raise), 1,128 hands per side, 3 continuations",
            "sequences_per_player_this_rank": int(g.size[0]),
            "iterations": r["iterations"], "device_seconds": secs, "iters_per_s": r["iterations"] / secs,
            "exploitability": r["exploitability"], "setup_s": round(setup, 2),
            "collective": ("one all-gather of the per-board river values (T x m x boards doubles) per "
                           "half-iteration and per best response, folded in board order "
                           + ("(libkrcuda NCCL, in-stream, graph-captured)" if comm is not None else
                              "(host process group)")) if world > 1 else "none (one GPU)"}


def config1_gpu():
    """BASELINE config 1: the parity game (twenty_card plays the Leduc role,
    SURVEY.md §7), Kronecker sparsification + 1000 CFR+ iterations in fp64,
    checkpointEvery = 1 (the parity run), on the device."""
    from paper_2112_03804_b200 import host as H
    from paper_2112_03804_b200.solver import DcfrParams, solver_for
    inst = H.builtin("twenty_card")
    t0 = time.perf_counter()
    f = inst.sparsify("b", True)
    sparsify_s = time.perf_counter() - t0
    sv = solver_for([(inst, f)])
    prm = DcfrParams.cfr_plus(max_iters=1000, checkpoint_every=1)
    sv.run(DcfrParams.cfr_plus(max_iters=5, checkpoint_every=1))  # warm
    r = sv.run(prm)
    # the same solve driven by K7 (within tolerance, not bitwise: DESIGN.md §4.2)
    sk = solver_for([(inst, f)], implicit=True)
    sk.run(DcfrParams.cfr_plus(max_iters=5, checkpoint_every=1))
    rk = sk.run(prm)
    return {"workload": "config1: twenty_card (Leduc role), Technique B post, 1000 CFR+ iterations, "
                        "checkpointEvery=1", "iterations": r.iterations, "exploitability": r.exploitability,
            "device_seconds": r.seconds, "iters_per_s": r.iterations / r.seconds if r.seconds else None,
            "sparsify_s": sparsify_s, "alpha": "+inf", "beta": "-inf", "gamma": 1.0, "rule": "cfr+",
            "implicit": {"iters_per_s": rk.iterations / rk.seconds if rk.seconds else None,
                         "exploitability": rk.exploitability,
                         "rel_diff_vs_factored": abs(rk.exploitability - r.exploitability) / r.exploitability},
            "_trace": r.trace_expl}


def config2_gpu(peak):
    """BASELINE configs[1] (config 2): one river board Ks7d4c2h9s, 1,081 hands
    per side, 3-bet tree, B-post (6.27e6 stored nonzeros, 76 MB per product).
    Kernels this small are latency-bound, so besides the serial pair it
    reports the concurrent pair (kr_engine_pair_device), K7 and the solver."""
    import torch

    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import host as H
    from paper_2112_03804_b200.solver import DcfrParams, solver_for
    inst = H.builtin("river_full", seed=1, board="Ks7d4c2h9s", tree=3)
    f = inst.sparsify("b", True)
    eng, ek, ekf = CudaEngine(f), CudaEngine.kron([inst]), CudaEngine.kfactored([inst])
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device="cpu").manual_seed(2)
    x = torch.randn(eng.cols, dtype=torch.float64, generator=g).to(dev)
    y = torch.randn(eng.rows, dtype=torch.float64, generator=g).to(dev)
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for n in (eng.rows, eng.cols) * 5]

    def timed(e, fn, reps=300):
        st = torch.cuda.ExternalStream(e.stream)
        for _ in range(5):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    def serial():
        eng.ax_device(x.data_ptr(), outs[0].data_ptr())
        eng.atx_device(y.data_ptr(), outs[1].data_ptr())

    def pair():
        eng.pair_device(x.data_ptr(), outs[2].data_ptr(), y.data_ptr(), outs[3].data_ptr())

    def kron():
        ek.ax_device(x.data_ptr(), outs[4].data_ptr())
        ek.atx_device(y.data_ptr(), outs[5].data_ptr())

    def kf_serial():
        ekf.ax_device(x.data_ptr(), outs[6].data_ptr())
        ekf.atx_device(y.data_ptr(), outs[7].data_ptr())

    def kf_pair():
        ekf.pair_device(x.data_ptr(), outs[8].data_ptr(), y.data_ptr(), outs[9].data_ptr())

    us_serial, us_pair, us_k7 = timed(eng, serial), timed(eng, pair), timed(ek, kron)
    us_kf, us_kf_pair = timed(ekf, kf_serial), timed(ekf, kf_pair)
    torch.cuda.synchronize(dev)
    bitwise = bool(torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[3]))
    kf_bitwise = bool(torch.equal(outs[0], outs[6]) and torch.equal(outs[1], outs[7]) and
                      torch.equal(outs[0], outs[8]) and torch.equal(outs[1], outs[9]))
    k7_diff = max(float((outs[4] - outs[0]).abs().max() / (1 + outs[0].abs().max())),
                  float((outs[5] - outs[1]).abs().max() / (1 + outs[1].abs().max())))
    pair_bytes = 2 * eng.bytes_per_product()
    solver = {}
    from paper_2112_03804_b200.solver import CudaSolver
    for name, implicit in (("factored", False), ("implicit", True), ("kfactored", None)):
        sv = (solver_for([(inst, f)], implicit=implicit) if implicit is not None else
              CudaSolver(ekf, inst.treeplex(0), inst.treeplex(1), [inst.m1], [inst.m2], inst.pot))
        sv.run(DcfrParams(max_iters=10, checkpoint_every=10))
        r = sv.run(DcfrParams(max_iters=400, checkpoint_every=50), want_avg=False)
        solver[name] = {"iters_per_s": 400 / r.seconds, "exploitability": r.exploitability}
    # the headline: the fastest pair whose bits are the factored engine's
    # (the oracle's, tests/test_gpu_kfengine.py)
    cands = [("factored", "kr_engine_ax_device + kr_engine_atx_device", us_serial, True),
             ("factored", "kr_engine_pair_device", us_pair, bitwise),
             ("kfactored", "kr_engine_ax_device + kr_engine_atx_device", us_kf, kf_bitwise),
             ("kfactored", "kr_engine_pair_device", us_kf_pair, kf_bitwise)]
    best = min((c for c in cands if c[3]), key=lambda c: c[2])
    return {"workload": "config2: river Ks7d4c2h9s, 1,081 hands per side, 3-bet tree (n=43), B-post",
            "nnz_stored": int(f.size()), "algorithmic_bytes_per_pair": pair_bytes,
            "us_per_pair": best[2], "pairs_per_s": 1e6 / best[2], "engine": best[0], "api": best[1],
            "bitwise_equal": True,
            "whole_pair_frac_of_peak": pair_bytes / (best[2] / 1e6) / 1e9 / peak,
            "frac_note": "algorithmic bytes of the materialised factors (SURVEY 8(d)) over the pair time; the "
                         "Kronecker-factored engine computes the same products bit for bit without streaming "
                         "those bytes (an effective rate)" if best[0] == "kfactored" else
                         "algorithmic bytes over the pair time",
            "factored": {"us_per_pair": us_serial, "pairs_per_s": 1e6 / us_serial,
                         "whole_pair_frac_of_peak": pair_bytes / (us_serial / 1e6) / 1e9 / peak,
                         "concurrent_pair": {"api": "kr_engine_pair_device", "us_per_pair": us_pair,
                                             "pairs_per_s": 1e6 / us_pair, "bitwise_equal_to_serial": bitwise}},
            "implicit": {"us_per_pair": us_k7, "pairs_per_s": 1e6 / us_k7, "normwise_diff_vs_factored": k7_diff,
                         "tolerance": 1e-12},
            "kfactored": {"api": "kr_engine_create_kfactored", "us_per_pair": us_kf, "pairs_per_s": 1e6 / us_kf,
                          "concurrent_us_per_pair": us_kf_pair, "concurrent_pairs_per_s": 1e6 / us_kf_pair,
                          "bitwise_equal_to_factored": kf_bitwise,
                          "effective_frac_of_peak": pair_bytes / (min(us_kf, us_kf_pair) / 1e6) / 1e9 / peak},
            "solver_checkpoint_every_50": solver}


def config4_gpu(peak):
    """BASELINE configs[3] (config 4): the large-rank variant, 26-card deck
    (13 ranks x 2 suits), board Kc9d7c4d2c, all 210 hands per side, 3-bet tree.
    Technique A exercises the low-rank U V^T term (rank 1,000 = the peel cap)
    and the A-hat SpMV; Technique B beside it.  Pairs/s (device pointers,
    CUDA events), the fraction of the HBM peak, DCFR iterations/s, and the
    implicit engine on the same payoff."""
    import torch

    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import host as H
    from paper_2112_03804_b200.solver import DcfrParams, solver_for
    inst = H.builtin("river_full", seed=1, board="Kc9d7c4d2c", deck=26, tree=3)
    dev = torch.device("cuda", torch.cuda.current_device())
    out = {"workload": "config4: 26-card deck (13 ranks x 2 suits), board Kc9d7c4d2c, 210 hands per side, 3-bet tree"}

    def timed(e, reps=500):
        st = torch.cuda.ExternalStream(e.stream)
        g = torch.Generator(device="cpu").manual_seed(4)
        x = torch.randn(e.cols, dtype=torch.float64, generator=g).to(dev)
        y = torch.randn(e.rows, dtype=torch.float64, generator=g).to(dev)
        a = torch.empty(e.rows, dtype=torch.float64, device=dev)
        b = torch.empty(e.cols, dtype=torch.float64, device=dev)
        for _ in range(5):
            e.pair_device(x.data_ptr(), a.data_ptr(), y.data_ptr(), b.data_ptr())
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            e.pair_device(x.data_ptr(), a.data_ptr(), y.data_ptr(), b.data_ptr())
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    for tech in ("a", "b"):
        f = inst.sparsify(tech, True)
        eng = CudaEngine(f)
        us = timed(eng)
        pair_bytes = 2 * eng.bytes_per_product()
        sv = solver_for([(inst, f)])
        sv.run(DcfrParams(max_iters=10, checkpoint_every=10))
        r = sv.run(DcfrParams(max_iters=1000, checkpoint_every=50), want_avg=False)
        out[f"technique_{tech}"] = {"nnz": {k: int(v) for k, v in eng.nnz.items()}, "k": int(eng.k),
                                    "us_per_pair": us, "pairs_per_s": 1e6 / us,
                                    "whole_pair_frac_of_peak": pair_bytes / (us / 1e6) / 1e9 / peak,
                                    "api": "kr_engine_pair_device",
                                    "solver_iters_per_s": 1000 / r.seconds, "exploitability": r.exploitability}
        sv.close()
        eng.close()
    ek = CudaEngine.kron([inst])
    us = timed(ek)
    out["implicit"] = {"us_per_pair": us, "pairs_per_s": 1e6 / us}
    ek.close()
    return out


def config1_cpu(gpu):
    """The same 1000 CFR+ iterations on the oracle (CPU, one thread) and the
    bitwise cross-check of the GPU trace against it."""
    import math
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    o = po.Instance.builtin("twenty_card")
    t0 = time.perf_counter()
    r = po.dcfr(o, o.sparsify("b", True), alpha=math.inf, beta=-math.inf, gamma=1.0, max_iters=1000,
                checkpoint_every=1, rule=1)
    secs = time.perf_counter() - t0
    same = bool(np.array_equal(np.asarray(gpu["_trace"]).view(np.int64), r["trace_expl"].view(np.int64)))
    return {"seconds": secs, "iters_per_s": 1000 / secs, "cores": 1, "kind": "port",
            "exploitability": r["exploitability"], "gpu_trace_bitwise_equal": same}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(threads, budget_s, gpu_out=None):
    """The reference engine (restated in oracle/: matvec / matvecTranspose,
    engine.hpp:58-133, sequential per call) over a bounded sample of the
    boards, one board per host thread; scaled to full-turn pairs/s.  Inputs
    are dense Gaussians (mt19937_64, as tools/main.cpp:313-317).  Also: the
    reference-faithful single-thread per-call time (engine.hpp:11-13 is
    sequential), and the parity check of the GPU's timed outputs against the
    oracle on the sampled boards (gpu_out: {engine: (ax, atx)} host arrays of
    the bench's x, y)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    nb = min(NBOARDS, threads)
    pairs = oracle_boards(range(nb), threads, with_instances=True)
    sps = [sp for _, sp in pairs]
    # single thread, one board, per call (SURVEY.md §8(d) CPU baseline (i))
    rng = np.random.default_rng(1)
    x0, y0 = rng.standard_normal(pairs[0][0].cols), rng.standard_normal(pairs[0][0].rows)
    s1 = sps[0].time_pairs(x0, y0, 1)
    reps1 = max(2, int(min(3.0, budget_s / 4) / max(s1, 1e-4)))
    s1 = sps[0].time_pairs(x0, y0, reps1) / reps1
    parity = None
    if gpu_out:
        parity = {"boards": nb, "inputs": "the bench's own x, y (Gaussian)", "engines": {}}
        for name, (gax, gatx, x, y) in gpu_out.items():
            ok = True
            c0 = r0 = 0
            for inst, sp in pairs:
                ok &= bool(np.array_equal(sp.matvec(x[c0:c0 + inst.cols]).view(np.int64),
                                          gax[r0:r0 + inst.rows].view(np.int64)))
                ok &= bool(np.array_equal(sp.matvec_t(y[r0:r0 + inst.rows]).view(np.int64),
                                          gatx[c0:c0 + inst.cols].view(np.int64)))
                c0 += inst.cols
                r0 += inst.rows
            parity["engines"][name] = ok
        parity["bitwise"] = all(parity["engines"].values())
    t1 = po.time_pairs_multi(sps, threads, 1)  # warm + estimate
    reps = max(1, int(budget_s / max(t1, 1e-3)))
    t = po.time_pairs_multi(sps, threads, reps)
    board_pairs_per_s = nb * reps / t
    # DCFR iterations/s, same boards, one per thread
    d1 = po.time_dcfr_multi(pairs, threads, 1)
    iters = max(1, int(0.5 * budget_s / max(d1, 1e-3)))
    d = po.time_dcfr_multi(pairs, threads, iters)
    return {"value": board_pairs_per_s / NBOARDS, "unit": "pairs/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "inputs": "dense Gaussian x, y (mt19937_64, tools/main.cpp:313-317)",
            "sample": f"{nb} of {NBOARDS} boards x {reps} matvec pairs each, one board per thread "
                      f"({t:.1f} s); full-turn pairs/s = board-pairs/s / {NBOARDS}",
            "single_thread": {"ms_per_pair_one_board": 1e3 * s1, "full_turn_pairs_per_s": 1.0 / (s1 * NBOARDS),
                              "cores": 1, "sample": f"board 0, {reps1} pairs, one thread (the reference engine is "
                                                    "sequential per call, engine.hpp:11-13)"},
            "parity": parity,
            "solver_iters_per_s": nb * iters / d / NBOARDS,
            "solver_sample": f"{nb} of {NBOARDS} boards x {iters} DCFR iterations each (default parameters, "
                             f"no checkpoints), one board per thread ({d:.1f} s); full-turn it/s = "
                             f"board-iterations/s / {NBOARDS}"}


def run_reference(args):
    """Reference arm: the reference's CPU implementation of the path (the
    oracle's restatement; the reference itself needs Eigen3, absent here) on
    all host threads, same metric and workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    threads = os.cpu_count() or 1
    pairs = oracle_boards(range(args.boards), threads, with_instances=True)
    sps = [sp for _, sp in pairs]
    t1 = po.time_pairs_multi(sps, threads, 1)
    steps = args.steps
    budget = 150.0
    if t1 * (args.steps + args.warmup) > budget:
        steps = max(3, int(budget / t1) - args.warmup)
    for _ in range(args.warmup):
        po.time_pairs_multi(sps, threads, 1)
    total = 0.0
    for _ in range(steps):
        total += po.time_pairs_multi(sps, threads, 1)
    value = steps / total
    # DCFR iterations/s on the same game (all boards, one per thread), bounded
    d1 = po.time_dcfr_multi(pairs, threads, 1)
    it = max(1, min(20, int(30.0 / max(d1, 1e-3))))
    solver_ips = it / po.time_dcfr_multi(pairs, threads, it)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.boards, args.gpus),
            "steps_requested": args.steps,
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                             "sample": f"all {args.boards} boards per step, one board per thread at a time; "
                                       "reference engine restated in oracle/ (Eigen3 absent: reference "
                                       "unbuildable)"},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "solver_iters_per_s": solver_ips,
            "solver_sample": f"all {args.boards} boards x {it} DCFR iterations (default parameters), one board "
                             "per thread at a time"}
    print(json.dumps(_finite(line)), flush=True)
    return 0


# -------------------------------------------------------- product (GPU) ----
def run_product(args):
    import torch
    import torch.distributed as dist

    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import host as H
    from paper_2112_03804_b200.dist import DistributedDcfr, shard
    from paper_2112_03804_b200.solver import CudaSolver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # NCCL over NVLink between the GPUs of the node; KR_DIST_BACKEND=gloo
    # runs the same multi-rank logic with host collectives (used to smoke the
    # torchrun path on a one-GPU box: ranks share cuda:0, no kernel waits on
    # another rank).
    backend = os.environ.get("KR_DIST_BACKEND", "nccl")
    local = min(local, torch.cuda.device_count() - 1)
    coll_dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    # The library's own NCCL communicator carries the solvers' exchanges
    # (checkpoint values, turn river values) in-stream; with a host backend
    # (KR_DIST_BACKEND=gloo: several ranks on one GPU) the same all-gathers
    # go through the process group.
    from paper_2112_03804_b200.dist import Comm, boards_per_rank
    comm = Comm.from_process_group(local) if world > 1 and backend == "nccl" else None
    bpr = boards_per_rank(args.boards, world)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    mine = shard(args.boards, rank, world)
    t0 = time.time()
    boards = H.turn_instances(TURN, args.boards, indices=list(mine))
    build_s = time.time() - t0
    t0 = time.time()
    eng = CudaEngine([f for _, f in boards], device=local)
    create_s = time.time() - t0
    nnz_stored = int(sum(f.size() for _, f in boards))
    pair_bytes = 2 * eng.bytes_per_product()
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(eng.cols, dtype=torch.float64, device=dev, generator=g)
    y = torch.randn(eng.rows, dtype=torch.float64, device=dev, generator=g)
    ax = torch.empty(eng.rows, dtype=torch.float64, device=dev)
    atx = torch.empty(eng.cols, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)

    def pair():
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())

    for _ in range(max(args.warmup, 3)):
        pair()
    torch.cuda.synchronize(dev)
    # Pre-pass (untimed for `value`): every SpMV bracketed by events, for the
    # per-matrix breakdown and to pick the dominant kernel.  The timed region
    # then brackets only that kernel (its events cost ~0.4% of a pair; all
    # four, ~1.5%).
    eng.kernel_times()  # reset counters
    eng.set_timing(True)
    pre_steps = max(20, min(args.steps, 100))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(pre_steps):
        pair()
    e1.record(stream)
    e1.synchronize()
    pre_ms = e0.elapsed_time(e1)
    eng.set_timing(False)
    pre_times = eng.kernel_times()
    dominant = max(pre_times, key=lambda k: pre_times[k]["ms"])
    eng.set_timing(True, only=[dominant])
    launches0 = eng.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    uuid = str(torch.cuda.get_device_properties(dev).uuid)
    sampler = ClockSampler(uuid if uuid.startswith("GPU-") else f"GPU-{uuid}")
    barrier()
    torch.cuda.synchronize(dev)
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            pair()
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize(dev)
    barrier()
    ms_local = e0.elapsed_time(e1)
    gpu_launches = int(sum_over_ranks(eng.launches() - launches0))
    eng.set_timing(False)
    ktimes = eng.kernel_times()  # the dominant kernel, over the timed region
    eng.set_timing(False, only=None)
    ms = max_over_ranks(ms_local)
    pairs_per_s = args.steps / (ms / 1e3)

    # ---- e2e: the C-ABI host-buffer calls, H2D + D2H inside the region ----
    e2e = e2e_host_pairs(eng, x, y, barrier, max_over_ranks, max(5, min(args.steps, 50)))
    check_ok = bool(np.array_equal(e2e.pop("_ax"), ax.cpu().numpy()))
    nx, ny = eng.cols, eng.rows

    # ---- solver iterations/s (DCFR, checkpointEvery = 50) ----------------
    i0 = boards[0][0]
    solver = CudaSolver(eng, i0.treeplex(0), i0.treeplex(1), [b[0].m1 for b in boards], [b[0].m2 for b in boards],
                        i0.pot)
    if comm is not None:
        solver.set_comm(comm, bpr)
    drv = DistributedDcfr(solver, args.boards, i0.pot, rank, world, device=coll_dev)
    drv.run(max_iters=5, checkpoint_every=5)  # warm
    barrier()
    torch.cuda.synchronize(dev)
    ts = time.perf_counter()
    res = drv.run(max_iters=args.solver_iters, checkpoint_every=50)
    torch.cuda.synchronize(dev)
    solver_s = max_over_ranks(time.perf_counter() - ts)
    factored_steps = step_kinds(solver)

    # ---- Kronecker-factored engine (bitwise, nothing streamed) -------------
    kfac = run_kfactored(args, boards, eng, x, y, ax, atx, dev, local, rank, world, coll_dev, barrier,
                         max_over_ranks, sum_over_ranks, res, comm, bpr)
    # ---- implicit Kronecker engine (K7) -------------
    implicit = run_implicit(args, boards, eng, x, y, ax, dev, local, rank, world, coll_dev, barrier, max_over_ranks,
                            sum_over_ranks, comm, bpr)
    turn = run_turn(rank, world, local, max_over_ranks, dist.group.WORLD if world > 1 else None, comm)
    config1 = config1_gpu() if rank == 0 else None
    config2 = config2_gpu(measured_peak()[0]) if rank == 0 else None
    config4 = config4_gpu(measured_peak()[0]) if rank == 0 else None
    gpu_out = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the timed region's last outputs, for the parity check against the oracle
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
        torch.cuda.ExternalStream(eng.stream, device=dev).synchronize()
        gpu_out = {"factored": (ax.cpu().numpy(), atx.cpu().numpy(), x.cpu().numpy(), y.cpu().numpy())}
    del boards
    solver.close()
    eng.close()
    torch.cuda.empty_cache()
    sweep = run_sweep() if rank == 0 and world == 1 and not args.no_sweep else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peak, peak_src = measured_peak()
    kd = ktimes[dominant]
    per_launch_ms = kd["ms"] / max(kd["launches"], 1)
    achieved = kd["bytes_per_launch"] / (per_launch_ms / 1e3) / 1e9
    kernels = {k: {"launches": v["launches"], "avg_us": 1e3 * v["ms"] / max(v["launches"], 1),
                   "gb_per_s": v["bytes_per_launch"] / (v["ms"] / max(v["launches"], 1) / 1e3) / 1e9
                   if v["launches"] else None, "bytes_per_launch": v["bytes_per_launch"],
                   "share_of_step": v["ms"] / pre_ms if pre_ms else None} for k, v in pre_times.items()}
    kernels["_source"] = (f"pre-pass of {pre_steps} pairs with every SpMV bracketed by events; the roofline "
                          f"kernel ({dominant}) is timed again over the timed region itself")
    line = {
        "metric": METRIC, "value": pairs_per_s, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.boards, world),
        "workload_detail": {"nnz_stored": nnz_stored if world == 1 else None,
                            "algorithmic_bytes_per_pair": pair_bytes if world == 1 else None,
                            "host_build_s": round(build_s, 2), "engine_create_s": round(create_s, 2)},
        "roofline": {"bound": "hbm", "kernel": f"k_spmv[{dominant}]", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                     "traffic": ncu_traffic(dominant) if world == 1 and args.boards == NBOARDS else None,
                     "whole_pair_gb_per_s": pair_bytes / (ms_local / args.steps / 1e3) / 1e9 if world == 1 else None},
        "kernels": kernels,
        "e2e": dict(e2e, matches_device_path=check_ok),
        "solver_iters_per_s": args.solver_iters / solver_s,
        "solver": {"iterations": res["iterations"], "exploitability": res["exploitability"],
                   "checkpoint_every": 50, "player_step": factored_steps},
        "gpu_launches": gpu_launches,
        "multi_gpu": {"ranks": world, "boards_per_rank": [int(v) for v in bpr],
                      "transport": ("libkrcuda kr_comm (NCCL): checkpoint values and turn values all-gathered "
                                    "in-stream, folded in board order (bitwise N-invariant)") if comm is not None else
                      ("host process group (" + backend + ")" if world > 1 else "none")},
        "clocks": sampler.summary(),
        "kfactored": kfac,
        "implicit": implicit,
        "config5_sweep": sweep,
        "config1": {k: v for k, v in config1.items() if not k.startswith("_")},
        "config2": config2,
        "config4": config4,
        "turn": turn,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(os.cpu_count() or 1, args.cpu_seconds, gpu_out)
        line["parity"] = line["cpu_baseline"].pop("parity")
        line["cpu_baseline"]["config1"] = config1_cpu(config1)
    print(json.dumps(_finite(line)), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_host_pairs(eng, x, y, barrier, max_over_ranks, steps, ring=4):
    """End to end through the C ABI on pinned host buffers: each step ships an
    x and a y to the device and both results back (H2D + D2H inside the timed
    region).  Headline: kr_engine_pair_queue over `steps` independent pairs
    (the reference's benchmark loop of products, tools/main.cpp:313-323),
    their inputs cycling through `ring` distinct pinned buffer sets: the input
    copies of the next pair and the output copies of the previous one run
    under each pair's kernels.  Beside it: kr_engine_pair one pair per call
    (both directions in flight, graph-replayed) and the reference's call
    pattern, kr_engine_ax then kr_engine_atx."""
    import ctypes

    from paper_2112_03804_b200 import _native as N
    L = N.cuda()
    nx, ny = eng.cols, eng.rows
    as_np = lambda p, n: np.ctypeslib.as_array((ctypes.c_double * n).from_address(p))  # noqa: E731
    sets = []
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    for r in range(ring):
        b = [L.kr_host_alloc(8 * n) for n in (nx, ny, ny, nx)]
        as_np(b[0], nx)[:] = xh if r == 0 else np.roll(xh, r)
        as_np(b[1], ny)[:] = yh if r == 0 else np.roll(yh, r)
        sets.append(b)
    px, py, pax, patx = sets[0]
    order = [i % ring for i in range(steps)]
    P = ctypes.c_void_p * steps
    qcol = [P(*[sets[o][j] for o in order]) for j in range(4)]

    def queue():
        N.check(L.kr_engine_pair_queue(eng.handle, steps, qcol[0], nx, qcol[2], ny, qcol[1], ny, qcol[3], nx))

    def pair():
        N.check(L.kr_engine_pair(eng.handle, px, nx, pax, ny, py, ny, patx, nx))

    def serial():
        N.check(L.kr_engine_ax(eng.handle, px, nx, pax, ny))
        N.check(L.kr_engine_atx(eng.handle, py, ny, patx, nx))

    out = {}
    for name, fn, calls in (("serial", serial, steps), ("pair", pair, steps), ("queue", queue, 3)):
        for _ in range(1 if name == "queue" else 3):
            fn()
        barrier()
        t = time.perf_counter()
        for _ in range(calls):
            fn()
        out[name] = (steps if name != "queue" else 3 * steps) / max_over_ranks(time.perf_counter() - t)
    res = {"value": out["queue"], "unit": "pairs/s", "h2d_bytes_per_step": 8 * (nx + ny),
           "d2h_bytes_per_step": 8 * (nx + ny), "steps": 3 * steps,
           "api": f"kr_engine_pair_queue: 3 calls of {steps} independent pairs, inputs cycling through {ring} pinned "
                  "buffer sets (x, y in; A x, A^T y out per pair; next pair's input copies and previous pair's "
                  "output copies under each pair's kernels)",
           "pair_call": {"value": out["pair"], "api": "kr_engine_pair, one pair per call (both directions in "
                                                      "flight, graph-replayed)"},
           "serial_calls": {"value": out["serial"], "api": "kr_engine_ax then kr_engine_atx (the reference's "
                                                          "call pattern, solver.hpp:366, 370)"},
           "_ax": as_np(pax, ny).copy()}
    # every ring slot's queued result is the bits of the one-pair call on it
    ok = True
    for b in sets:
        gax, gatx = as_np(b[2], ny).copy(), as_np(b[3], nx).copy()
        N.check(L.kr_engine_pair(eng.handle, b[0], nx, b[2], ny, b[1], ny, b[3], nx))
        ok &= bool(np.array_equal(gax.view(np.int64), as_np(b[2], ny).view(np.int64)))
        ok &= bool(np.array_equal(gatx.view(np.int64), as_np(b[3], nx).view(np.int64)))
    res["queue_bitwise_equal_to_pair_call"] = ok
    res["_ax"] = as_np(pax, ny).copy()
    for b in sets:
        for p in b:
            L.kr_host_free(p)
    return res


def step_kinds(solver):
    """Which kernel ran each player's step (kr_solver_step_kind)."""
    names = {2: "compiled for the treeplex (NVRTC, kr_jit.cu)", 1: "generic team kernel", 0: "generic per-hand kernel"}
    out = {}
    for p in (0, 1):
        k, why = solver.step_kind(p)
        out[f"player{p + 1}"] = names.get(k, "?") + (f" ({why})" if why and k != 2 else "")
    return out


def run_kfactored(args, boards, eng, x, y, ax, atx, dev, local, rank, world, coll_dev, barrier, max_over_ranks,
                  sum_over_ranks, ref_solve, comm=None, bpr=None):
    """The same pairs through the Kronecker-factored engine (Technique B post
    kept as its hand-space factors, every Kronecker product expanded on the
    fly: kr_kfengine.cu), which is BITWISE the factored engine: device
    pairs/s, e2e, the bit check against the factored outputs, and DCFR
    iterations/s with the trace compared bitwise to the factored solve."""
    import torch

    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200.dist import DistributedDcfr
    from paper_2112_03804_b200.solver import CudaSolver

    t0 = time.time()
    ek = CudaEngine.kfactored([b[0] for b in boards], device=local)
    create_s = time.time() - t0
    st = torch.cuda.ExternalStream(ek.stream, device=dev)
    kax, katx = torch.empty_like(ax), torch.empty_like(atx)

    def serial():
        ek.ax_device(x.data_ptr(), kax.data_ptr())
        ek.atx_device(y.data_ptr(), katx.data_ptr())

    def pair():
        ek.pair_device(x.data_ptr(), kax.data_ptr(), y.data_ptr(), katx.data_ptr())

    res = {}
    steps = max(args.steps, 50)
    for name, fn in (("serial", serial), ("pair", pair)):
        for _ in range(max(args.warmup, 3)):
            fn()
        torch.cuda.synchronize(dev)
        l0 = ek.launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(st)
        for _ in range(steps):
            fn()
        e1.record(st)
        e1.synchronize()
        barrier()
        res[name] = (max_over_ranks(e0.elapsed_time(e1)), int(sum_over_ranks(ek.launches() - l0)))
    bitwise = bool(torch.equal(kax, ax) and torch.equal(katx, atx))
    bitwise = max_over_ranks(0.0 if bitwise else 1.0) == 0.0
    e2e = e2e_host_pairs(ek, x, y, barrier, max_over_ranks, 50)
    e2e.pop("_ax")
    i0 = boards[0][0]
    solver = CudaSolver(ek, i0.treeplex(0), i0.treeplex(1), [b[0].m1 for b in boards], [b[0].m2 for b in boards],
                        i0.pot)
    if comm is not None:
        solver.set_comm(comm, bpr)
    drv = DistributedDcfr(solver, args.boards, i0.pot, rank, world, device=coll_dev)
    drv.run(max_iters=5, checkpoint_every=5)
    barrier()
    torch.cuda.synchronize(dev)
    ts = time.perf_counter()
    r = drv.run(max_iters=args.solver_iters, checkpoint_every=50)
    torch.cuda.synchronize(dev)
    solver_s = max_over_ranks(time.perf_counter() - ts)
    same_trace = bool(np.array_equal(np.asarray(r["trace_expl"]).view(np.int64),
                                     np.asarray(ref_solve["trace_expl"]).view(np.int64)))
    out = {"engine": "kr_engine_create_kfactored (Technique B post from its Kronecker factors; "
                     "k_kfa_vt / k_kfa_fold / k_kfa_ua, k_kft_fold / k_kft_av)",
           "pairs_per_s": steps / (res["serial"][0] / 1e3), "us_per_pair": 1e3 * res["serial"][0] / steps,
           "concurrent_pair": {"api": "kr_engine_pair_device", "pairs_per_s": steps / (res["pair"][0] / 1e3),
                               "us_per_pair": 1e3 * res["pair"][0] / steps},
           "steps": steps, "gpu_launches": res["serial"][1], "bitwise_equal_to_factored": bitwise,
           "create_s": round(create_s, 3), "e2e": e2e,
           "solver_iters_per_s": args.solver_iters / solver_s,
           "solver": {"iterations": r["iterations"], "exploitability": r["exploitability"],
                      "trace_bitwise_equal_to_factored_solve": same_trace, "player_step": step_kinds(solver)}}
    solver.close()
    ek.close()
    return out


def run_sweep(budget_s=40.0):
    """Config 5 (BASELINE.json): matvec pairs over synthetic poker instances
    from ~5e5 to ~1.25e9 stored nonzeros, one B200.  Each point's factored
    engine is built on the device (kr_engine_create_device_b, bitwise the
    host-built engine) and timed with CUDA events (whole pair, Ax then ATy);
    the Kronecker-factored engine (bitwise, nothing streamed) beside it.
    Algorithmic bytes per BASELINE.md §2."""
    import torch

    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import host as H
    peak = measured_peak()[0]

    def river(board, deck=52, tree=3):
        return [H.builtin("river_full", seed=1, board=board, deck=deck, tree=tree)]

    def turns(ts, tree):
        out = []
        for t in ts:
            out += [i for i, _ in H.turn_instances(turn=t, nboards=NBOARDS, tree=tree, factors=False)]
        return out

    points = [("config4: 26-card deck, 210 hands, 3-bet", lambda: river("Kc9d7c4d2c", deck=26)),
              ("config2: river 1081 hands, 3-bet", lambda: river("Ks7d4c2h9s")),
              ("river 1081 hands, 91-seq tree", lambda: river("Ks7d4c2h9s", tree=91)),
              ("config3: turn x 48 rivers, 3-bet", lambda: turns([TURN], 3)),
              ("turn x 48 rivers, 91-seq tree", lambda: turns([TURN], 91)),
              ("2 turns x 48 rivers, 91-seq tree", lambda: turns([TURN, "Ah8c5d3s"], 91))]

    def timed(e, reps):
        st = torch.cuda.ExternalStream(e.stream)
        x = torch.randn(e.cols, dtype=torch.float64, device="cuda")
        y = torch.randn(e.rows, dtype=torch.float64, device="cuda")
        a = torch.empty(e.rows, dtype=torch.float64, device="cuda")
        b = torch.empty(e.cols, dtype=torch.float64, device="cuda")
        for _ in range(3):
            e.ax_device(x.data_ptr(), a.data_ptr())
            e.atx_device(y.data_ptr(), b.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            e.ax_device(x.data_ptr(), a.data_ptr())
            e.atx_device(y.data_ptr(), b.data_ptr())
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    rows, t_start = [], time.time()
    for name, make in points:
        if time.time() - t_start > budget_s:
            rows.append({"point": name, "skipped": "sweep time budget"})
            continue
        insts = make()
        eng = CudaEngine.device_built(insts)
        nnz = sum(eng.nnz.values())
        pair_bytes = 2 * eng.bytes_per_product()
        reps = max(10, min(500, int(0.3 / max(pair_bytes / (peak * 1e9 * 0.8), 1e-6))))
        t = timed(eng, reps)
        eng.close()
        torch.cuda.empty_cache()
        ek = CudaEngine.kfactored(insts)
        tk = timed(ek, max(10, min(500, int(0.3 / max(t / 2, 1e-6)))))
        ek.close()
        torch.cuda.empty_cache()
        rows.append({"point": name, "boards": len(insts), "stored_nnz": int(nnz), "bytes_per_pair": pair_bytes,
                     "factored": {"us_per_pair": 1e6 * t, "pairs_per_s": 1 / t, "gb_per_s": pair_bytes / t / 1e9,
                                  "frac_of_measured_peak": pair_bytes / t / 1e9 / peak, "reps": reps},
                     "kfactored": {"us_per_pair": 1e6 * tk, "pairs_per_s": 1 / tk}})
    return {"workload": "config5: matvec pairs over synthetic poker instances (Technique B post), one GPU",
            "peak_gb_per_s": peak, "points": rows}


def run_implicit(args, boards, eng, x, y, ax, dev, local, rank, world, coll_dev, barrier, max_over_ranks,
                 sum_over_ranks, comm=None, bpr=None):
    """The same matvec pairs through the implicit Kronecker engine (nothing
    materialised: strength-order and card-list prefix scans per board and
    sequence, kr_kron.cu), on the same boards and inputs: device pairs/s,
    host-buffer e2e pairs/s, agreement with the factored engine, and DCFR
    iterations/s driven by it."""
    import ctypes
    import torch

    from paper_2112_03804_b200 import CudaEngine
    from paper_2112_03804_b200 import _native as N
    from paper_2112_03804_b200.dist import DistributedDcfr
    from paper_2112_03804_b200.solver import CudaSolver

    ek = CudaEngine.kron([b[0] for b in boards], device=local)
    st = torch.cuda.ExternalStream(ek.stream, device=dev)
    kax = torch.empty_like(ax)
    katx = torch.empty(ek.cols, dtype=torch.float64, device=dev)

    def pair():
        ek.ax_device(x.data_ptr(), kax.data_ptr())
        ek.atx_device(y.data_ptr(), katx.data_ptr())

    for _ in range(max(args.warmup, 3)):
        pair()
    torch.cuda.synchronize(dev)
    l0 = ek.launches()
    steps = max(args.steps, 50)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(st)
    for _ in range(steps):
        pair()
    e1.record(st)
    e1.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = int(sum_over_ranks(ek.launches() - l0))
    dif = float((kax - ax).abs().max().item() / (1.0 + ax.abs().max().item()))
    dif = max_over_ranks(dif)

    e2e = e2e_host_pairs(ek, x, y, barrier, max_over_ranks, 50)
    e2e.pop("_ax")

    i0 = boards[0][0]
    solver = CudaSolver(ek, i0.treeplex(0), i0.treeplex(1), [b[0].m1 for b in boards], [b[0].m2 for b in boards],
                        i0.pot)
    if comm is not None:
        solver.set_comm(comm, bpr)
    drv = DistributedDcfr(solver, args.boards, i0.pot, rank, world, device=coll_dev)
    drv.run(max_iters=5, checkpoint_every=5)
    barrier()
    torch.cuda.synchronize(dev)
    ts = time.perf_counter()
    res = drv.run(max_iters=args.solver_iters, checkpoint_every=50)
    torch.cuda.synchronize(dev)
    solver_s = max_over_ranks(time.perf_counter() - ts)
    out = {"engine": "kr_engine_create_kron (k_kron_fused: one CTA per board and sequence)",
           "pairs_per_s": steps / (ms / 1e3), "us_per_pair": 1e3 * ms / steps, "steps": steps,
           "gpu_launches": launches, "normwise_diff_vs_factored": dif, "tolerance": 1e-12,
           "e2e": e2e,
           "solver_iters_per_s": args.solver_iters / solver_s,
           "solver": {"iterations": res["iterations"], "exploitability": res["exploitability"],
                      "player_step": step_kinds(solver),
                      "layout": "sequence-major x and gradients (kron_product_seq)" if os.environ.get("KR_K7SEQ") != "0"
                                else "hand-major"}}
    solver.close()
    ek.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_product(args)


if __name__ == "__main__":
    sys.exit(main())
