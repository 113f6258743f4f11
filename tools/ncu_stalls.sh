# key metrics + stall breakdown of an ncu report: bash tools/ncu_stalls.sh report.ncu-rep
python tools/ncu_brief.py $1 | grep -v '^\['
ncu -i $1 --page raw --csv 2>/dev/null > /tmp/raw_$$.csv
python3 - /tmp/raw_$$.csv <<'PY'
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[0]
for r in rows[2:]:
    for n,v in zip(h,r):
        if ('smsp__average_warps_issue_stalled' in n) and n.endswith('_per_issue_active.ratio'):
            try:
                if float(v)>0.3: print("   stall",n.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''),v)
            except: pass
        if n in ('smsp__inst_executed.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','lts__t_sectors_srcunit_tex_op_read.sum'):
            print("  ",n,v)
PY
rm -f /tmp/raw_$$.csv
