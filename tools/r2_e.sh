#!/bin/bash
# e2e host-path sweep: expansion mode x host threads x workers
for w in 2 4; do
  for m in all ri t 0; do
    for th in 4 8; do SOGK_HOST_EXPAND=$m SOGK_HOST_THREADS=$th python tools/e2e_sweep.py $w; done
  done
done
