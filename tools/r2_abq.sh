#!/bin/bash
# Quick A/B: parity tests on the default build, then bench kernel timing vs _ab variants per config.
#   TAG=x CFGS="cfg2 cfg1" TESTS="tests/test_gpu_parity.py ..." bash tools/r2_abq.sh variant...
set -u
TAG=${TAG:-abq}
mkdir -p gpurun_out
timeout 1200 python -m pytest ${TESTS:-tests -m gpu} -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
tail -2 gpurun_out/${TAG}_pytest_gpu.txt
for CFG in ${CFGS:-cfg2 cfg1 cfg4 cfg3}; do
  TAG=${TAG}_$CFG CFG=$CFG STEPS=${STEPS:-20} bash tools/r2_ab.sh "$@"
done
