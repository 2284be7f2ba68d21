# Quick GPU iteration: gpu tests, bench cfg2 (no CPU leg), per-kernel ncu summary of one cfg2 object.
set -x
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"count_|write_|expand_|tail_|scan_" -s 4 -c 4 -o /tmp/${TAG}_full python tools/prof_step.py cfg2 hdda_skip > /dev/null 2>&1
python tools/ncu_summary.py /tmp/${TAG}_full.ncu-rep > gpurun_out/${TAG}_ncu_cfg2_hdda_skip.txt 2>&1
cp /tmp/${TAG}_full.ncu-rep gpurun_out/ 2>/dev/null
