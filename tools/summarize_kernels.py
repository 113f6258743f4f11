"""Generic ncu --set full summary into profiles/ (tracked): one row per
captured launch (duration, DRAM bytes, L1/L2/DRAM throughput, issue slots,
occupancy, registers), plus the top source lines by warp-stall samples for
each kernel name.

usage: python tools/summarize_kernels.py <report.ncu-rep> <tag> "<title>" <source.cu> [<launches.csv>]"""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = [("Duration", "gpu__time_duration.sum"), ("DRAM read", "dram__bytes_read.sum"),
        ("DRAM write", "dram__bytes_write.sum"),
        ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
        ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("issue busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread"), ("grid", "launch__grid_size")]


def short(name):
    return name.split("(")[0].split("::")[-1]


def main():
    rep, tag, title, src = sys.argv[1:5]
    launches = sys.argv[5] if len(sys.argv) > 5 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# {title}", "", f"Source: `{os.path.basename(rep)}` (ncu --set full, --clock-control none; "
             "per-launch numbers are cold-cache and serialised).", "",
             "| launch | kernel | " + " | ".join(c for c, _ in COLS) + " |",
             "|---|---|" + "---|" * len(COLS)]
    for r in data:
        cells = []
        for _, m in COLS:
            if m in idx:
                v, u = r[idx[m]], units[idx[m]]
                cells.append(f"{v} {u}".strip())
            else:
                cells.append("n/a")
        lines.append(f"| {r[idx['ID']]} | {short(r[idx['Kernel Name']])} | " + " | ".join(cells) + " |")
    # stall lines
    lines += ["", "## Top source lines by warp-stall samples (all captured launches)", "", "```"]
    sl = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, src, "16"],
                        capture_output=True, text=True)
    lines += sl.stdout.rstrip().split("\n") + ["```"]
    if launches:
        agg = collections.defaultdict(list)
        h2 = None
        for r in csv.reader(open(launches)):
            if r and r[0] == "ID":
                h2 = r
                continue
            if h2 and len(r) == len(h2):
                d = dict(zip(h2, r))
                agg[short(d["Kernel Name"])].append(float(d["Metric Value"]))
        tot = sum(sum(v) for v in agg.values()) or 1
        lines += ["", f"## Launch list (`{os.path.basename(launches)}`, gpu__time_duration.sum)", "",
                  "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    path = os.path.join(ROOT, "profiles", f"{tag}.md")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(path)


if __name__ == "__main__":
    main()
