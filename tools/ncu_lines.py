"""Aggregate an ncu report's per-instruction warp-stall samples by CUDA
source line: python tools/ncu_lines.py report.ncu-rep source.cu [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, srcfile = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, cur = None, None
agg, inst = collections.Counter(), collections.Counter()
stalls = collections.defaultdict(collections.Counter)
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or cur is None or not cur.endswith(srcfile.split("/")[-1]):
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(d["Line No"])
    except ValueError:
        continue
    agg[ln] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    inst[ln] += int(d["Instructions Executed"] or 0)
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls[ln][k[6:]] += int(d[k] or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
src = open(srcfile).read().split("\n")
for ln, s in agg.most_common(top):
    why = ", ".join(f"{k}={v}" for k, v in stalls[ln].most_common(3))
    text = src[ln - 1].strip()[:72] if ln - 1 < len(src) else "?"
    print(f"{ln:5d} {100 * s / tot:5.1f}% inst={inst[ln]:9d}  {text} | {why}")
