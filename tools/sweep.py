"""Config 5 (BASELINE.json): matvec bandwidth sweep over synthetic poker
instances from ~1e6 to ~1e9 stored nonzeros on one B200.

Each point builds the factors with the product's host side (libkrhost,
Technique B postprocessed), creates one engine (boards stacked), and times
matvec pairs with CUDA events on the engine stream (warm-up first).  Reports
pairs/s, algorithmic GB/s of the whole pair (BASELINE.md §2 byte formula)
and the fraction of the measured HBM peak.  Writes JSON lines to stdout and
a markdown table to profiles/<tag>_sweep.md.

usage: python tools/sweep.py [--tag r01] [--max-nnz 1.4e9]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2112_03804_b200 import CudaEngine  # noqa: E402
from paper_2112_03804_b200 import host as H  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6552.3


def river(board, deck=52, tree=3, seed=1):
    inst = H.builtin("river_full", seed=seed, board=board, deck=deck, tree=tree)
    return [(inst, inst.sparsify("b", True))]


def turns(turn_list, tree):
    out = []
    for t in turn_list:
        out += H.turn_instances(turn=t, nboards=48, tree=tree)
    return out


POINTS = [
    ("config4: 26-card deck, 210 hands, 3-bet", lambda: river("Kc9d7c4d2c", deck=26)),
    ("config2a: river 1081 hands, reference tree", lambda: river("Ks7d4c2h9s", tree=1)),
    ("config2: river 1081 hands, 3-bet tree", lambda: river("Ks7d4c2h9s")),
    ("river 1081 hands, 91-seq tree", lambda: river("Ks7d4c2h9s", tree=91)),
    ("config3: turn Ks7d4c2h x 48 rivers, 3-bet", lambda: turns(["Ks7d4c2h"], 3)),
    ("turn x 48 rivers, 91-seq tree", lambda: turns(["Ks7d4c2h"], 91)),
    ("config5 top: 2 turns x 48 rivers, 91-seq tree", lambda: turns(["Ks7d4c2h", "Ah8c5d3s"], 91)),
]


def time_pairs(eng, reps, concurrent=False):
    """Seconds per pair: Ax then ATy on the engine stream, or both in flight
    together (kr_engine_pair_device) with concurrent=True."""
    s = torch.cuda.ExternalStream(eng.stream)
    x = torch.randn(eng.cols, dtype=torch.float64, device="cuda")
    y = torch.randn(eng.rows, dtype=torch.float64, device="cuda")
    ax = torch.empty(eng.rows, dtype=torch.float64, device="cuda")
    atx = torch.empty(eng.cols, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    for _ in range(3):
        eng.ax_device(x.data_ptr(), ax.data_ptr())
        eng.atx_device(y.data_ptr(), atx.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        if concurrent:
            eng.pair_device(x.data_ptr(), ax.data_ptr(), y.data_ptr(), atx.data_ptr())
        else:
            eng.ax_device(x.data_ptr(), ax.data_ptr())
            eng.atx_device(y.data_ptr(), atx.data_ptr())
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    tag = sys.argv[sys.argv.index("--tag") + 1] if "--tag" in sys.argv else "r01"
    max_nnz = float(sys.argv[sys.argv.index("--max-nnz") + 1]) if "--max-nnz" in sys.argv else 1.4e9
    rows = []
    for name, make in POINTS:
        t0 = time.time()
        boards = make()
        nnz = sum(f.size() for _, f in boards)
        if nnz > max_nnz:
            print(json.dumps({"point": name, "skipped": f"nnz {nnz} > max {max_nnz}"}), flush=True)
            continue
        build_s = time.time() - t0
        t0 = time.time()
        eng = CudaEngine([f for _, f in boards])
        create_s = time.time() - t0
        pair_bytes = 2 * eng.bytes_per_product()
        est = pair_bytes / (PEAK * 1e9 * 0.8)
        reps = max(10, min(2000, int(2.0 / max(est, 1e-6))))
        t = time_pairs(eng, reps)
        tc = time_pairs(eng, reps, concurrent=True)
        gbs = pair_bytes / t / 1e9
        eng.close()
        torch.cuda.empty_cache()
        # the same pairs through the implicit engine (K7, nothing materialised)
        t0 = time.time()
        ek = CudaEngine.kron([i for i, _ in boards])
        kron_create_s = time.time() - t0
        tk = time_pairs(ek, max(50, min(2000, int(0.5 / max(t / 8, 1e-6)))))
        ek.close()
        row = {"point": name, "nnz": nnz, "bytes_per_pair": pair_bytes, "pairs_per_s": 1 / t,
               "us_per_pair": t * 1e6, "gb_per_s": gbs, "frac_of_measured_peak": gbs / PEAK,
               "concurrent_us_per_pair": tc * 1e6, "concurrent_frac_of_measured_peak": pair_bytes / tc / 1e9 / PEAK,
               "reps": reps, "host_build_s": round(build_s, 2), "engine_create_s": round(create_s, 2),
               "implicit_us_per_pair": tk * 1e6, "implicit_pairs_per_s": 1 / tk,
               "implicit_create_s": round(kron_create_s, 2)}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del boards
        torch.cuda.empty_cache()
    lines = [f"# Matvec bandwidth sweep ({tag}), one B200, fp64, Technique B postprocessed", "",
             f"Whole matvec pair (Ax + ATx); algorithmic bytes per BASELINE.md §2; peak {PEAK} GB/s (measured).", "",
             "The concurrent columns put both products of a pair in flight together (kr_engine_pair_device). "
             "The implicit columns time the same pairs through K7 (kr_engine_create_kron), which streams no factors.",
             "",
             "| point | stored nnz | MB / pair | us / pair | pairs/s | GB/s | % of peak | concurrent us / pair "
             "| concurrent % of peak | K7 us / pair | K7 pairs/s |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['point']} | {r['nnz']:,} | {r['bytes_per_pair']/1e6:,.1f} | {r['us_per_pair']:,.1f} | "
                     f"{r['pairs_per_s']:,.1f} | {r['gb_per_s']:,.0f} | {100*r['frac_of_measured_peak']:.1f} | "
                     f"{r['concurrent_us_per_pair']:,.1f} | {100*r['concurrent_frac_of_measured_peak']:.1f} | "
                     f"{r['implicit_us_per_pair']:,.1f} | {r['implicit_pairs_per_s']:,.0f} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_sweep.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
