"""Print an ncu --csv metrics launch list compactly: one line per launch."""
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
    cur = None
    print(f)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        if r[ii] != cur:
            if cur is not None:
                print()
            cur = r[ii]
            print(f"{r[ii]:>3} {r[ki].split('(')[0].split('::')[-1][:18]:18s} {r[h.index('Grid Size')]:>14s}", end=' ')
        name = r[mi].replace('gpu__time_duration.sum', 'ns').replace('sm__warps_active.avg.pct_of_peak_sustained_active', 'warps%')
        name = name.replace('smsp__inst_executed.sum', 'inst').replace('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smwf')
        name = name.replace('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smconf')
        print(f"{name}={r[vi]}", end=' ')
    print()
