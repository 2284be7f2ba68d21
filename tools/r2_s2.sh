#!/bin/bash
# second pass: full gpu tests, cfg4/cfg1/cfg2 bench lines, pass-1 register A/B, e2e sweep cfg1
set -x
TAG=${TAG:-s2}
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
for c in cfg4 cfg1 cfg2; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
TAG=${TAG}ab tools/r2_ab.sh minb7
