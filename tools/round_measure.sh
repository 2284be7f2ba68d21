# One GPU call: bench (default cfg2 + CPU baseline), reference arm, launch list, ncu captures.
set -x
TAG=${1:-r1}
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
for c in cfg1 cfg3 cfg4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for V in hdda_skip dda_branch; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"count_|write_|scan_" -s 3 -c 3 -o /tmp/${TAG}_full_$V python tools/prof_step.py cfg1 $V > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_full_$V.ncu-rep > gpurun_out/${TAG}_ncu_cfg1_$V.txt
done
nproc > gpurun_out/${TAG}_host_cores.txt; lscpu | head -20 >> gpurun_out/${TAG}_host_cores.txt
