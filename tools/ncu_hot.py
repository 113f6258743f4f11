"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report:
python tools/ncu_hot.py report.ncu-rep [kernel-substring] [top]"""
import csv
import io
import subprocess
import sys

rep, sub, top = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else ""), int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
blocks = out.split('"Kernel Name",')
for blk in blocks[1:]:
    name = blk.split("\n", 1)[0]
    if sub not in name:
        continue
    rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
    h = rows[0]
    si, ii, ci = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    wi = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
    data = [r for r in rows[1:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in data) or 1
    print(name[:100], "total samples", tot)
    for r in sorted(data, key=lambda r: -int(r[si]))[:top]:
        print(f"{100*int(r[si])/tot:5.1f}%  inst={r[ci]:>10s}  smwf={r[wi] if wi else '-':>10s}  {r[ii].strip()[:90]}")
    break
