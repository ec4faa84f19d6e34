#!/bin/bash
# tools/ncu_digest.sh rep.ncu-rep : headline metrics of every kernel in a report
ncu -i "$1" --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=['Duration','DRAM Throughput','Memory Throughput','Compute (SM) Throughput','Executed Ipc Active','Issue Slots Busy','L1/TEX Hit Rate','L2 Hit Rate','Eligible Warps Per Scheduler','No Eligible','Warp Cycles Per Issued Instruction','Executed Instructions','Registers Per Thread','Achieved Occupancy','Theoretical Occupancy','Branch Efficiency','dram__bytes_read.sum','dram__bytes_write.sum']
seen=set()
for row in r[1:]:
    d=dict(zip(h,row)); n=d.get('Metric Name','')
    if n in keep and (d['Kernel Name'][:40],n) not in seen:
        seen.add((d['Kernel Name'][:40],n)); print(d['Kernel Name'][:40],'|',n,'=',d['Metric Value'],d['Metric Unit'])
"
