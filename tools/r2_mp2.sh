#!/bin/bash
# A/B main vs variants on cfg2/cfg1/cfg4 + ncu --set full of pass 2 (cfg2 object 0, cfg4)
#   bash tools/r2_mp2.sh TAG variant...
TAG=$1; shift
mkdir -p gpurun_out
export VARIANTS=hdda_skip,dda_branch,cd_skip
TAG=${TAG} CFG=cfg2 bash tools/r2_ab.sh "$@" > /dev/null 2>&1
TAG=${TAG}c1 CFG=cfg1 bash tools/r2_ab.sh "$@" > /dev/null 2>&1
TAG=${TAG}c4 CFG=cfg4 STEPS=5 bash tools/r2_ab.sh "$@" > /dev/null 2>&1
for C in cfg2 cfg4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gather" -s 1 -c 1 -o /tmp/${TAG}_$C python tools/prof_step.py $C hdda_skip 0 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_$C.ncu-rep > gpurun_out/${TAG}_ncu_gather_$C.txt 2>&1
  ncu -i /tmp/${TAG}_$C.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_gather_sass_$C.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$C.ncu-rep --page raw --csv > gpurun_out/${TAG}_gather_raw_$C.csv 2>/dev/null
done
