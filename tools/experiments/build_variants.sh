# build experiment variants of libiabn.so into tools/libiabn_<name>.so, then restore the default
# usage: bash tools/build_variants.sh name1 "defines1" name2 "defines2" ...
set -e
while [ $# -ge 2 ]; do
  IABN_NVCC_EXTRA="$2" python paper_1712_02616_b200/build.py --force > /dev/null
  cp paper_1712_02616_b200/libiabn.so tools/libiabn_$1.so
  echo "built $1: $2"
  shift 2
done
python paper_1712_02616_b200/build.py --force > /dev/null
