#!/bin/bash
# cfg5 subset for A/B: main build and each _ab/<variant>
for V in main "$@"; do
  if [ "$V" = main ]; then L=""; else L=$PWD/_ab/$V/libsogk.so; fi
  SOGK_LIB=$L timeout 900 python tools/sweep_cfg5.py --log2-min 22 --log2-max 22 --fractions ${FRACS:-0.005,0.02,0.2} \
     --families ${FAMS:-random,blocky} --out gpurun_out/${TAG:-c5}_$V > gpurun_out/${TAG:-c5}_$V.txt 2>&1
done
