# Bench every config (kernel timing only) with the main build: bash tools/all_cfgs.sh TAG
TAG=$1
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${c}.json 2> gpurun_out/${TAG}_${c}.err
done
