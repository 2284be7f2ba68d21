# One GPU call: gpu tests, smoke, default bench, launch list and one ncu --set full of the step kernels.
set -x
TAG=${1:-s2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --variants hdda_skip > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_|write_|expand_|scan_" -s 3 -c 3 -o /tmp/${TAG}_full python tools/prof_step.py cfg2 hdda_skip > /dev/null 2>&1
python tools/ncu_summary.py /tmp/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_cfg2_hdda_skip.txt 2>&1
ncu -i /tmp/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_raw.csv 2>/dev/null
