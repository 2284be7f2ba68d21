# ncu --set full with source counters for one object's pass 1 + pass 2; exports per-SASS-line stalls.
#   bash tools/ncu_src.sh TAG [cfg] [variant] [object]
TAG=$1; CFG=${2:-cfg2}; VAR=${3:-hdda_skip}; OBJ=${4:-0}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_|gather_|tail_" -s 3 -c 3 -o /tmp/${TAG} python tools/prof_step.py $CFG $VAR $OBJ > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py /tmp/${TAG}.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
for K in count_kernel gather_kernel tail_kernel; do
  ncu -i /tmp/${TAG}.ncu-rep -k regex:$K --page source --csv --print-source sass > gpurun_out/${TAG}_${K}_sass.csv 2>/dev/null
done
# (the .ncu-rep stays on the box: gpurun_out is capped at 64 MiB)
