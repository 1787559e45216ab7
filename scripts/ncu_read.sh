#!/bin/bash
# usage: ncu_read.sh rep.ncu-rep [kernel-regex]
REP=$1
ncu -i $REP --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]
for row in r[2:]:
    name=row[h.index('Kernel Name')][:40]
    out=[]
    for i,k in enumerate(h):
        if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
            try: v=float(row[i])
            except: continue
            if v>0.05: out.append((round(v,2),k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')))
    print(name, sorted(out,reverse=True)[:7])
    for k in ['gpu__time_duration.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__inst_executed.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sectors_srcunit_tex_op_read.sum','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','launch__grid_size','launch__block_size']:
        if k in h: print('   ',k, row[h.index(k)])
"
