#!/bin/bash
# ncu (full + sass source) of count_kernel on one grid for the main build and each _ab/<variant>
for V in main "$@"; do
  if [ "$V" = main ]; then L=""; else L=$PWD/_ab/$V/libsogk.so; fi
  SOGK_LIB=$L timeout 600 ncu --set full --import-source on --clock-control none -k regex:count_kernel -s 1 -c 1 \
     -o /tmp/${TAG}_$V python tools/prof_grid.py ${FAM:-random} ${FRAC:-0.02} > gpurun_out/${TAG}_$V.log 2>&1
  python tools/ncu_summary.py /tmp/${TAG}_$V.ncu-rep > gpurun_out/${TAG}_${V}_summary.txt 2>&1
  ncu -i /tmp/${TAG}_$V.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${V}_sass.csv 2>/dev/null
done
