#!/bin/bash
# Key metrics + per-line hot spots of an ncu report: tools/ncu_brief.sh <report> [lines]
ncu -i "$1" --page details --csv 2>/dev/null | python -c "
import csv,sys
keep=('Duration','DRAM Throughput','Registers Per Thread','Achieved Occupancy','Theoretical Occupancy','Issue Slots Busy','Grid Size','Block Limit Shared Mem','Block Limit Registers','L2 Hit Rate','No Eligible','Eligible Warps Per Scheduler','Executed Instructions','Local Memory Spilling Requests')
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[12] in keep: print('  ', r[12], r[14], r[13])
"
python profiles/ncu_lines.py "$1" ${2:-14}
