#!/bin/bash
# Round-2 measurement pass (one GPU call): tests, smoke, bench cfg2 (default) + cfg1/3/4, reference
# arm, launch list, ncu full of pass 1 + pass 2 (cfg2 object 0), issue counts, cfg5 sweep.
#   TAG=s1 bash tools/r2_measure.sh
set -x
TAG=${TAG:-r2m}
mkdir -p gpurun_out
nproc > gpurun_out/${TAG}_host_cores.txt; lscpu | head -20 >> gpurun_out/${TAG}_host_cores.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
for c in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-render > /dev/null 2>&1
for V in hdda_skip dda_branch; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_|gather_|tail_|scan_" -s 4 -c 4 \
     -o /tmp/${TAG}_full_$V python tools/prof_step.py cfg2 $V 0 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_full_$V.ncu-rep > gpurun_out/${TAG}_ncu_cfg2_$V.txt 2>&1
  ncu -i /tmp/${TAG}_full_$V.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_raw_cfg2_$V.csv 2>/dev/null
done
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:count_kernel --csv \
     --log-file gpurun_out/${TAG}_issue_$c.csv python tools/issue_probe.py run $c > /dev/null 2>&1
done
timeout 1800 python tools/sweep_cfg5.py --out gpurun_out/${TAG}_cfg5 > gpurun_out/${TAG}_cfg5.log 2>&1
tools/r2_e.sh > gpurun_out/${TAG}_e2e_sweep.txt 2>&1
