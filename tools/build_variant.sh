# Build an A/B variant of libsogk.so into /root/repo/_ab/<name>/ (use with SOGK_LIB=...).
#   tools/build_variant.sh minb8 "-DSOGK_COUNT_MINB=8"
set -e
NAME=$1; shift
OUT=$(cd "$(dirname "$0")/.." && pwd)/_ab/$NAME
mkdir -p $OUT/obj
make -s -j8 -C $(dirname "$0")/../paper_2404_10272_b200/csrc OUT=$OUT OBJ=$OUT/obj EXTRA_NVFLAGS="$*"
echo built $OUT/libsogk.so
