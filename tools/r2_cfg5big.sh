#!/bin/bash
# cfg5 large-launch probe: 16M-64M rays on the grids whose 32M/64M rows fell off the flat line
# in the s4 sweep, with per-pass split, all reps, free memory, and nvidia-smi sampled alongside.
#   TAG=b1 bash tools/r2_cfg5big.sh
TAG=${TAG:-big}
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,memory.used,clocks_throttle_reasons.active \
   --format=csv -lms 500 > gpurun_out/${TAG}_smi.csv 2>&1 &
SMI=$!
timeout 900 python tools/sweep_cfg5.py --out gpurun_out/${TAG}_a --log2-min 24 --reps 5 \
   --families random --fractions 0.005,0.1 > gpurun_out/${TAG}_a.log 2>&1
timeout 900 python tools/sweep_cfg5.py --out gpurun_out/${TAG}_b --log2-min 24 --reps 5 \
   --families blocky --fractions 0.01,0.1 > gpurun_out/${TAG}_b.log 2>&1
kill $SMI
