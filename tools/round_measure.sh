# One GPU call: bench (default cfg2 + e2e + CPU baseline), reference arm, cfg1/3/4, launch list,
# ncu --set full of pass 1 + pass 2 (dram bytes for roofline.traffic).   bash tools/round_measure.sh TAG
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nproc > gpurun_out/${TAG}_host_cores.txt; lscpu | head -20 >> gpurun_out/${TAG}_host_cores.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
for c in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for V in hdda_skip dda_branch; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_|gather_|tail_|scan_" -s 4 -c 4 -o /tmp/${TAG}_full_$V python tools/prof_step.py cfg2 $V 0 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_full_$V.ncu-rep > gpurun_out/${TAG}_ncu_cfg2_$V.txt 2>&1
  ncu -i /tmp/${TAG}_full_$V.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_raw_cfg2_$V.csv 2>/dev/null
done
bash tools/issue_all.sh > gpurun_out/${TAG}_issue.txt 2>&1
