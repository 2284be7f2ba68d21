#!/bin/bash
# ncu --set full of one cfg2 count+write pass (object $OBJ, variant $V) -> summaries in gpurun_out/
set -u
TAG=${TAG:-r2}
OBJ=${OBJ:-0}
mkdir -p gpurun_out
for V in ${VARS:-hdda_skip}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_|gather_|tail_|scan_" -s 4 -c 4 \
     -o /tmp/${TAG}_full_$V python tools/prof_step.py ${CFG:-cfg2} $V $OBJ > gpurun_out/${TAG}_prof_$V.log 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_full_$V.ncu-rep > gpurun_out/${TAG}_ncu_${CFG:-cfg2}_$V.txt 2>&1
  ncu -i /tmp/${TAG}_full_$V.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_raw_${CFG:-cfg2}_$V.csv 2>/dev/null
  ncu -i /tmp/${TAG}_full_$V.ncu-rep --page source --csv -k regex:gather_ > gpurun_out/${TAG}_src_gather_$V.csv 2>/dev/null
done
