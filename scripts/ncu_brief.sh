#!/bin/bash
# brief summary of an ncu report: key throughput/occupancy lines + stall ratios
R=$1
ncu -i $R --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=csv.reader(sys.stdin); h=next(r)
for row in r:
    d=dict(zip(h,row))
    print(d['Section Name'][:28].ljust(28), d['Metric Name'][:50].ljust(50), d['Metric Value'], d['Metric Unit'])
" | grep -E "Duration|DRAM Throughput|Executed Ipc A|Issue Slots|No Eligible|Active Warps Per|Registers Per|Achieved Occ|Executed Instructions  |L2 Hit|Warp Cycles Per Issued|Mem Busy|Max Bandwidth"
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for k,x in zip(h,v):
    if ('warps_issue_stalled' in k and 'per_issue_active' in k):
        try:
            if float(x.replace(',',''))>0.1: print(k.replace('smsp__average_warps_issue_stalled_',''),x)
        except: pass
"
