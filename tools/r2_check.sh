#!/bin/bash
# One GPU call: the -m gpu suite (per-file logs) and a short default bench run.
set -u
TAG=${TAG:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.txt
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
fi
tail -5 gpurun_out/${TAG}_pytest_gpu.txt
