#!/bin/bash
# pass-2 output-parallel batches: parity (full GPU suite) + A/B of the long-run threshold
#   bash tools/r2_mp.sh TAG variant...
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1
export VARIANTS=hdda_skip,dda_branch,cd_skip
TAG=${TAG} CFG=cfg2 bash tools/r2_ab.sh "$@" > /dev/null 2>&1
TAG=${TAG}c1 CFG=cfg1 bash tools/r2_ab.sh "$@" > /dev/null 2>&1
TAG=${TAG}c4 CFG=cfg4 STEPS=5 bash tools/r2_ab.sh "$@" > /dev/null 2>&1
