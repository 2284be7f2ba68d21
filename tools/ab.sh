# A/B: bench cfg2 (kernel timing only) for the main build and each _ab/<variant>.
#   bash tools/ab.sh TAG [cfg] [variant ...]
TAG=$1; CFG=${2:-cfg2}; shift 2
mkdir -p gpurun_out
timeout 600 python bench.py --config $CFG --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_main_${CFG}.json 2>&1
for V in "$@"; do
  SOGK_LIB=$PWD/_ab/$V/libsogk.so timeout 600 python bench.py --config $CFG --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${V}_${CFG}.json 2>&1
done
