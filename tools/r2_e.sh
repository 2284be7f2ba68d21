#!/bin/bash
# e2e host-path sweep (workers x host threads x expansion)
for w in 1 2 4; do
  for th in 2 4 8 16; do SOGK_HOST_THREADS=$th python tools/e2e_sweep.py $w; done
  SOGK_HOST_EXPAND=0 python tools/e2e_sweep.py $w
done
