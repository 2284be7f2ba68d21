# ncu both launch modes of one variant on cfg1 (pass-1 and pass-2 kernels); summaries only
V=${1:-hdda_skip}
CFG=${2:-cfg1}
for M in 0 1; do
  SOGK_PERSISTENT=$M ncu --set full --clock-control none --import-source on -k regex:"count_|write_" -s 2 -c 2 -o /tmp/pm${M}_$V python tools/prof_step.py $CFG $V > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/pm${M}_$V.ncu-rep > gpurun_out/pm${M}_${V}_${CFG}.txt
  ncu -i /tmp/pm${M}_$V.ncu-rep --page source --csv --print-source sass > gpurun_out/pm${M}_${V}_${CFG}_sass.csv 2>/dev/null
done
