# Pass-1 issue-ceiling captures for every config (profiles/issue_<cfg>.json).   bash tools/issue_all.sh
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none \
      -k regex:count_kernel --csv --log-file gpurun_out/issue_$c.csv python tools/issue_probe.py run $c > /dev/null 2>&1
  python tools/issue_probe.py parse $c gpurun_out/issue_$c.csv
  cp profiles/issue_$c.json gpurun_out/
done
