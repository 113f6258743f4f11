"""Summarise an ncu capture of the engine kernels into profiles/ (tracked).

usage: python tools/summarize_ncu.py <report.ncu-rep> <launches.csv> <tag>

Writes profiles/<tag>_ncu_summary.md (per-kernel DRAM bytes / throughput /
occupancy from the --set full capture, and the per-launch share of one
matvec pair from the launch list) and updates profiles/ncu_traffic.json,
which bench.py reads for roofline.traffic (dram bytes per launch of the four
SpMV matrices, captured as VT, UA, UT, AV in that order)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORDER = ["VT", "UA", "UT", "AV"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
         "us": 1e-6, "ms": 1e-3, "ns": 1e-9}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki].split("(")[0].split("::")[-1], float(r[vi])) for r in rows[hdr + 1:]
            if len(r) > vi and "::k_" in r[ki]]


def main():
    report, lcsv, tag = sys.argv[1:4]
    h, units, rows = raw(report)
    # the capture may include the other kernels of a pair (seq_major, chain
    # solves): the four SpMV launches, in pair order, are VT, UA, UT, AV
    kn = h.index("Kernel Name")
    others = [r for r in rows if "k_spmv" not in r[kn]]
    rows = [r for r in rows if "k_spmv" in r[kn]]
    lines = [f"# ncu summary `{tag}`", "", f"report: `{os.path.basename(report)}` (ncu --set full, --clock-control none);"
             " launch list: `" + os.path.basename(lcsv) + "`", "", "## SpMV kernels (one matvec pair)", "",
             "| matrix | time us | dram read MB | dram write MB | dram % peak | L2 hit % | L1 hit % | warps active % | regs |",
             "|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for name, r in zip(ORDER, rows):
        v = {}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    v[m] = float(r[i]) * SCALE.get(units[i], 1.0)
                except ValueError:
                    v[m] = None
        rd, wr = v["dram__bytes_read.sum"], v["dram__bytes_write.sum"]
        traffic[name] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                         "duration_s_ncu": v["gpu__time_duration.sum"], "capture": tag}
        lines.append(f"| {name} | {v['gpu__time_duration.sum']*1e6:.1f} | {rd/1e6:.1f} | {wr/1e6:.2f} | "
                     f"{v['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                     f"{v['lts__t_sector_hit_rate.pct']:.1f} | {v['l1tex__t_sector_hit_rate.pct']:.1f} | "
                     f"{v['sm__warps_active.avg.pct_of_peak_sustained_active']:.1f} | "
                     f"{v['launch__registers_per_thread']:.0f} |")
    if others:
        lines += ["", "Other kernels in the capture:", "", "| kernel | time us | dram read MB | dram write MB |",
                  "|---|---|---|---|"]
        for r in others:
            def val(m):
                i = h.index(m)
                return float(r[i]) * SCALE.get(units[i], 1.0)
            lines.append(f"| {r[kn].split('(')[0].split('::')[-1]} | {val('gpu__time_duration.sum') * 1e6:.1f} | "
                         f"{val('dram__bytes_read.sum') / 1e6:.1f} | {val('dram__bytes_write.sum') / 1e6:.2f} |")
    ks = launches(lcsv)
    # the first whole-range pair: [seq_major,] VT, chain, UA, UT, chain^T, AV
    # (seq_major only with KR_XSEQ=1): from the first kernel to the 4th SpMV
    first = next((i for i, (n, _) in enumerate(ks) if n.startswith("k_seq_major") or n.startswith("k_spmv")), 0)
    end, spmvs = first, 0
    while end < len(ks) and spmvs < 4:
        spmvs += ks[end][0].startswith("k_spmv")
        end += 1
    pair = ks[first:end]
    tot = sum(t for _, t in pair)
    lines += ["", "## One matvec pair, launch list (cold-cache, serialised: compare shares)", "",
              "| kernel | ns | share |", "|---|---|---|"]
    for n, t in pair:
        lines.append(f"| {n} | {t:.0f} | {t/tot:.1%} |")
    lines.append(f"| **pair** | {tot:.0f} | 100% |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
