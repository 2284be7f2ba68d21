#!/bin/bash
# ncu --set full of pass 2 (gather_kernel) on cfg2 object 0 and cfg4, HDDA skip
TAG=$1
mkdir -p gpurun_out
for C in cfg2 cfg4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gather" -s 1 -c 1 -o /tmp/${TAG}_$C python tools/prof_step.py $C hdda_skip 0 > gpurun_out/${TAG}_ncu_$C.log 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_$C.ncu-rep > gpurun_out/${TAG}_ncu_gather_$C.txt 2>&1
  ncu -i /tmp/${TAG}_$C.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_gather_sass_$C.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$C.ncu-rep --page raw --csv > gpurun_out/${TAG}_gather_raw_$C.csv 2>/dev/null
done
