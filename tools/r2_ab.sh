#!/bin/bash
# A/B of library variants on one config: bench kernel timing only (no e2e/render/cpu legs).
#   TAG=x CFG=cfg2 tools/r2_ab.sh variant...   (main build first, then each _ab/<variant>)
set -u
TAG=${TAG:-ab}; CFG=${CFG:-cfg2}; VARS=${VARIANTS:-hdda_skip,dda_branch}
mkdir -p gpurun_out
for V in main "$@"; do
  if [ "$V" = main ]; then L=""; else L=$PWD/_ab/$V/libsogk.so; fi
  for rep in 1 2; do
    SOGK_LIB=$L timeout 600 python bench.py --config $CFG --steps ${STEPS:-20} --no-e2e --no-cpu-baseline --no-render \
      --variants $VARS > gpurun_out/${TAG}_${V}_${CFG}_$rep.json 2> gpurun_out/${TAG}_${V}_${CFG}_$rep.err
  done
done
python tools/ab_show.py gpurun_out/${TAG}_*_${CFG}_*.json > gpurun_out/${TAG}_summary.txt 2>&1
cat gpurun_out/${TAG}_summary.txt
