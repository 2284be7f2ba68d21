#!/bin/bash
# Final pass on the final build (no cfg5 / e2e sweeps): the driver's own commands (pytest -m gpu,
# smoke, bench --steps 20 --warmup 5, reference arm), bench cfg1/3/4, cfg2 launch list, ncu of
# pass 1 + pass 2, pass-1 issue counts.   TAG=s6 bash tools/r2_final.sh
set -x
TAG=${TAG:-fin}
mkdir -p gpurun_out
nproc > gpurun_out/${TAG}_host_cores.txt
timeout 1800 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
for c in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-render > /dev/null 2>&1
for V in hdda_skip dda_branch; do
  rm -f /tmp/${TAG}_full_$V.ncu-rep
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_|gather_|tail_|scan_" -s 4 -c 4 \
     -o /tmp/${TAG}_full_$V python tools/prof_step.py cfg2 $V 0 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_full_$V.ncu-rep > gpurun_out/${TAG}_ncu_cfg2_$V.txt 2>&1
done
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:count_kernel --csv \
     --log-file gpurun_out/${TAG}_issue_$c.csv python tools/issue_probe.py run $c > /dev/null 2>&1
done
